// capi.cu — extern "C" entry points of libitertrace_cuda.so (include/itertrace_cuda.h) and the
// analyze_trace orchestration (pipeline.hpp:34-134) on the device.
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <atomic>
#include <new>
#include <set>

#include "ingest.cuh"
#include "pipeline.cuh"

using namespace itt;

// onesweep tile shape (radix.cuh kCfgBlock/kCfgItems); ITT_RADIX_CFG overrides for tuning sweeps.
// Default 256 x 12 at 5 CTAs per SM (C3 radix passes 2.84 -> 2.71 ms/step against 512 x 8).
int itt::radix::config_index() {
  static int cfg = [] {
    const char* e = std::getenv("ITT_RADIX_CFG");
    const int v = e ? std::atoi(e) : 9;
    return (v >= 0 && v < 10) ? v : 9;
  }();
  return cfg;
}

// struct itt_ctx { itt::Ctx c; } lives in pipeline.cuh (dist_driver.cu shares it)

// why an itt_analyze_opts.sa_provider call failed (set by providers on the calling thread)
static thread_local std::string tl_provider_error;

namespace {

template <typename F>
int guarded(itt_ctx* ctx, F&& f) {
  if (!ctx) return ITT_E_INVALID_ARGUMENT;
  Ctx* c = &ctx->c;
  try {
    ITT_CUDA(cudaSetDevice(c->device));
    c->arena_top = 0;  // the previous call synchronized: its small buffers are dead
    c->upload_top = 0;  // ... and its pinned uploads have completed
    f(c);
    c->sync();
    c->last_error.clear();
    return ITT_OK;
  } catch (const Error& e) {
    c->last_error = e.what();
    cudaStreamSynchronize(c->stream);
    c->pending.clear();
    return e.status;
  } catch (const std::bad_alloc&) {
    c->last_error = "host allocation failed";
    return ITT_E_CUDA;
  } catch (const std::exception& e) {
    c->last_error = e.what();
    return ITT_E_CUDA;
  }
}

template <typename T>
T* host_alloc(size_t n) {
  T* p = static_cast<T*>(std::calloc(n ? n : 1, sizeof(T)));
  if (!p) throw std::bad_alloc();
  return p;
}
// for outputs the device overwrites completely: no zeroing, so recycled heap pages stay warm
template <typename T>
T* host_alloc_uninit(size_t n) {
  T* p = static_cast<T*>(std::malloc((n ? n : 1) * sizeof(T)));
  if (!p) throw std::bad_alloc();
  return p;
}

void check_records(const itt_records* r) {
  if (!r) fail(ITT_E_INVALID_ARGUMENT, "records: null");
  if (r->n && (!r->start_ns || !r->duration_ns || !r->size_bytes || !r->flags || !r->stream || !r->name_off || !r->name_bytes))
    fail(ITT_E_INVALID_ARGUMENT, "records: missing column");
  if (r->n >= 0xFFFFFFFFull) fail(ITT_E_INVALID_ARGUMENT, "records: more than 2^32-1 rows per trace");
}

// records -> dictionary -> census (optionally device-filtered)
void prepare(Ctx* c, TraceState& t, const itt_records* r, bool device_filter, bool allow_late_dur = false) {
  check_records(r);
  t.c = c;
  {
    StageTimer st(c, "upload");
    upload_records(c, r, t.rec, allow_late_dur);
  }
  {
    StageTimer st(c, "order");
    order_launch(t);  // the dictionary does not depend on the order: its verdict is read after it
  }
  {
    StageTimer st(c, "dictionary");
    build_dictionary(t);
  }
  {
    StageTimer st(c, "order-finish");
    order_finish(t);
  }
  if (!device_filter) {
    t.filtering = false;
    t.kept = t.rec.n;
  }
  StageTimer st(c, "census");
  stream_census(t);
}

uint64_t stream_total(const itt_stream_summary& s) {
  return s.counts[0] + s.counts[1] + s.counts[2] + s.counts[3] + s.counts[4] + s.counts[5];
}

void fill_census(const TraceState& t, itt_census* out) {
  out->n_streams = static_cast<uint32_t>(t.streams.size());
  out->streams = host_alloc<itt_stream_summary>(t.streams.size());
  std::memcpy(out->streams, t.streams.data(), t.streams.size() * sizeof(itt_stream_summary));
  out->n_devices = t.n_devices;
  out->majority_device = t.majority;
  out->dropped_records = t.filtering ? t.rec.n - t.kept : 0;
  out->n_records = t.kept;
}

// select_main_stream (streams.hpp:113-145)
uint32_t select_main(const std::vector<itt_stream_summary>& ss, uint32_t* n_main) {
  const itt_stream_summary* best = nullptr;
  uint32_t cnt = 0;
  for (const auto& s : ss) {
    if (s.cls != ITT_CLASS_MAIN) continue;
    ++cnt;
    if (!best || s.counts[0] > best->counts[0] || (s.counts[0] == best->counts[0] && s.stream < best->stream)) best = &s;
  }
  if (n_main) *n_main = cnt;
  if (!best) fail(ITT_E_NO_MAIN_STREAM, "stream-classify: no stream contains kernel operations");
  return best->stream;
}

// Mining reads repeats of length <= L_max = (n-1)/iterations only (mine.hpp:64-67), so suffixes need
// ordering by their first max(L_max) + 1 symbols (sa.cu: capped suffix array / LCP).
uint32_t mining_cap(uint64_t n, const std::vector<itt_mining_cfg>& cfgs) {
  int64_t lmax = 0;
  for (const auto& l : cfgs)
    if (l.iterations >= 1 && n >= 1) lmax = std::max<int64_t>(lmax, (static_cast<int64_t>(n) - 1) / l.iterations);
  return static_cast<uint32_t>(std::min<int64_t>(lmax, 0xFFFFFFFEll) + 1);
}

void tokens_to_device(Ctx* c, const int32_t* tokens, uint64_t n, DBuf<int32_t>& d) {
  d.alloc(c, n + 1);
  h2d(c, d.p, tokens, n);
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes pa{};
  if (cudaPointerGetAttributes(&pa, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return pa.type == cudaMemoryTypeDevice || pa.type == cudaMemoryTypeManaged;
}

// itt_suffix_array{,_capped}: inputs and outputs in host or device memory
void suffix_array_any(Ctx* c, const int32_t* tokens, uint64_t n, int32_t term, uint32_t cap, uint32_t* sa,
                      uint32_t* lcp) {
  DBuf<int32_t> dt;
  const int32_t* tok = tokens;
  if (n && !is_device_ptr(tokens)) {
    tokens_to_device(c, tokens, n, dt);
    tok = dt.p;
  }
  SuffixState s;
  s.keep_levels = lcp != nullptr;
  radix::Scratch rs;
  ScanScratch sc;
  build_suffix_array(c, tok, n, term, s, lcp != nullptr, rs, sc, cap);
  ITT_CUDA(cudaMemcpyAsync(sa, s.sa.p, (n + 1) * 4, cudaMemcpyDefault, c->stream));
  if (lcp) ITT_CUDA(cudaMemcpyAsync(lcp, s.lcp.p, (n + 1) * 4, cudaMemcpyDefault, c->stream));
  c->sync();
}

}  // namespace

extern "C" {

int itt_abi_version(void) { return ITT_ABI_VERSION; }

int itt_ctx_create(int device, itt_ctx** out) {
  if (!out) return ITT_E_INVALID_ARGUMENT;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0 || device < 0 || device >= ndev) return ITT_E_CUDA;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return ITT_E_CUDA;
  if (prop.major < 10) return ITT_E_CUDA;  // sm_100a kernels only
  itt_ctx* x = new (std::nothrow) itt_ctx;
  if (!x) return ITT_E_CUDA;
  Ctx* c = &x->c;
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete x;
    return ITT_E_CUDA;
  }
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = device;
  if (cudaMemPoolCreate(&c->pool, &props) != cudaSuccess) {
    cudaStreamDestroy(c->stream);
    delete x;
    return ITT_E_CUDA;
  }
  uint64_t thr = UINT64_MAX;  // keep freed blocks for reuse across calls
  cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &thr);
  *out = x;
  return ITT_OK;
}

int itt_ctx_destroy(itt_ctx* ctx) {
  if (!ctx) return ITT_OK;
  Ctx* c = &ctx->c;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (auto& p : c->pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : c->event_pool) cudaEventDestroy(e);
  if (c->sync_event) cudaEventDestroy(c->sync_event);
  for (auto& kv : c->out_live) cudaFreeHost(kv.first);  // outputs must be released before this
  for (auto& kv : c->out_free) cudaFreeHost(kv.second);
  for (auto& kv : c->big_cap) cudaFree(kv.first);  // cached large blocks (live ones are the caller's bug)
  if (c->pinned) cudaFreeHost(c->pinned);
  if (c->deferred) cudaFreeHost(c->deferred);
  if (c->deferred_ev) cudaEventDestroy(c->deferred_ev);
  if (c->upload) cudaFreeHost(c->upload);
  if (c->copy_stream) {
    cudaStreamSynchronize(c->copy_stream);
    cudaStreamDestroy(c->copy_stream);
  }
  for (auto w : c->win)
    if (w) cudaFree(w);
  if (c->arena) cudaFree(c->arena);
  for (auto b : c->bounce)
    if (b) cudaFreeHost(b);
  if (c->pool) cudaMemPoolDestroy(c->pool);
  cudaStreamDestroy(c->stream);
  delete ctx;
  return ITT_OK;
}

const char* itt_last_error(itt_ctx* ctx) { return ctx ? ctx->c.last_error.c_str() : "null context"; }

// error text for the host-only entry points (report.cu)
extern "C" __attribute__((visibility("hidden"))) int itt_ctx_set_error_(itt_ctx* ctx, const char* msg) {
  if (ctx) ctx->c.last_error = msg ? msg : "";
  return 0;
}

int itt_free(itt_ctx* ctx, void* p) {
  if (!p) return ITT_OK;
  if (ctx && ctx->c.out_release(p)) return ITT_OK;  // pinned output block: back to the context
  std::free(p);
  return ITT_OK;
}

int itt_ctx_set_profiling(itt_ctx* ctx, int enabled) {
  return guarded(ctx, [&](Ctx* c) { c->profiling = enabled != 0; });
}
int itt_ctx_reset_stats(itt_ctx* ctx) {
  return guarded(ctx, [&](Ctx* c) { c->stats.clear(); });
}
int itt_ctx_kernel_stats(itt_ctx* ctx, itt_kernel_stat* out, uint32_t cap, uint32_t* n_out) {
  return guarded(ctx, [&](Ctx* c) {
    uint32_t i = 0;
    for (const auto& kv : c->stats) {
      if (i < cap && out) {
        std::memset(&out[i], 0, sizeof(out[i]));
        std::strncpy(out[i].name, kv.first.c_str(), sizeof(out[i].name) - 1);
        out[i].launches = kv.second.launches;
        out[i].total_ms = kv.second.total_ms;
        out[i].bytes = kv.second.bytes;
      }
      ++i;
    }
    if (n_out) *n_out = i;
  });
}
int itt_ctx_mem_stats(itt_ctx* ctx, uint64_t* used, uint64_t* used_high, int reset) {
  return guarded(ctx, [&](Ctx* c) {
    c->sync();
    uint64_t u = 0, h = 0, r = 0;
    ITT_CUDA(cudaMemPoolGetAttribute(c->pool, cudaMemPoolAttrUsedMemCurrent, &u));
    ITT_CUDA(cudaMemPoolGetAttribute(c->pool, cudaMemPoolAttrUsedMemHigh, &h));
    ITT_CUDA(cudaMemPoolGetAttribute(c->pool, cudaMemPoolAttrReservedMemCurrent, &r));
    // large blocks live outside the pool (Ctx::big_take): added to both figures
    u += c->big_live;
    h += c->big_high;
    if (std::getenv("ITT_TRACE")) std::fprintf(stderr, "[itt] pool used %.2f GB high %.2f GB reserved %.2f GB\n", u / 1e9, h / 1e9, r / 1e9);
    if (used) *used = u;
    if (used_high) *used_high = h;
    if (reset) {
      uint64_t z = 0;
      ITT_CUDA(cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrUsedMemHigh, &z));
      c->big_high = c->big_live;
    }
  });
}

int itt_ctx_launch_count(itt_ctx* ctx, uint64_t* out) {
  if (!ctx || !out) return ITT_E_INVALID_ARGUMENT;
  *out = ctx->c.launches;
  return ITT_OK;
}
int itt_device_alloc(itt_ctx* ctx, uint64_t bytes, void** out) {
  return guarded(ctx, [&](Ctx* c) {
    ITT_CUDA(cudaMalloc(out, bytes + 16));
    (void)c;
  });
}
int itt_device_free(itt_ctx* ctx, void* p) {
  return guarded(ctx, [&](Ctx*) { ITT_CUDA(cudaFree(p)); });
}
int itt_memcpy_h2d(itt_ctx* ctx, void* dst, const void* src, uint64_t bytes) {
  return guarded(ctx, [&](Ctx* c) { ITT_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream)); });
}
int itt_memcpy_d2h(itt_ctx* ctx, void* dst, const void* src, uint64_t bytes) {
  return guarded(ctx, [&](Ctx* c) { ITT_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream)); });
}
int itt_memcpy(itt_ctx* ctx, void* dst, const void* src, uint64_t bytes) {
  return guarded(ctx, [&](Ctx* c) {
    if (bytes) ITT_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->stream));
  });
}
int itt_host_register(itt_ctx* ctx, void* p, uint64_t bytes) {
  return guarded(ctx, [&](Ctx*) { ITT_CUDA(cudaHostRegister(p, bytes, cudaHostRegisterDefault)); });
}
int itt_host_unregister(itt_ctx* ctx, void* p) {
  return guarded(ctx, [&](Ctx*) { ITT_CUDA(cudaHostUnregister(p)); });
}
int itt_ctx_stream(itt_ctx* ctx, void** stream) {
  if (!ctx || !stream) return ITT_E_INVALID_ARGUMENT;
  *stream = ctx->c.stream;
  return ITT_OK;
}
int itt_ctx_synchronize(itt_ctx* ctx) {
  return guarded(ctx, [&](Ctx*) {});
}

// ------------------------------------------------------------------ streams
int itt_summarize_streams(itt_ctx* ctx, const itt_records* recs, int filter_device, itt_census* out) {
  if (!out) return ITT_E_INVALID_ARGUMENT;
  std::memset(out, 0, sizeof(*out));
  return guarded(ctx, [&](Ctx* c) {
    if (!recs || recs->n == 0) fail(ITT_E_EMPTY_TRACE, "stream-classify: trace has no records");
    TraceState t;
    prepare(c, t, recs, filter_device != 0);
    fill_census(t, out);
  });
}

int itt_select_main_stream(itt_ctx* ctx, const itt_census* census, uint32_t* main_stream, uint32_t* n_main_streams) {
  return guarded(ctx, [&](Ctx*) {
    if (!census || !main_stream) fail(ITT_E_INVALID_ARGUMENT, "select_main_stream: null argument");
    std::vector<itt_stream_summary> ss(census->streams, census->streams + census->n_streams);
    *main_stream = select_main(ss, n_main_streams);
  });
}

int itt_build_token_sequence(itt_ctx* ctx, const itt_records* recs, uint32_t main_stream, itt_tokens** out) {
  if (!out) return ITT_E_INVALID_ARGUMENT;
  *out = nullptr;
  return guarded(ctx, [&](Ctx* c) {
    TraceState t;
    if (!recs || recs->n == 0)
      fail(ITT_E_EMPTY_MAIN_STREAM, "stream-classify: stream " + std::to_string(main_stream) + " has no records");
    prepare(c, t, recs, false);
    uint64_t n_main = 0;
    for (const auto& s : t.streams)
      if (s.stream == main_stream) n_main = stream_total(s);
    if (n_main == 0)
      fail(ITT_E_EMPTY_MAIN_STREAM, "stream-classify: stream " + std::to_string(main_stream) + " has no records");
    compact_main(t, main_stream, true);
    renumber_tokens(t);
    itt_tokens* o = host_alloc<itt_tokens>(1);
    o->n = t.n_tok;
    o->tokens = host_alloc<int32_t>(t.n_tok);
    o->record_index = host_alloc<uint64_t>(t.n_tok);
    o->n_names = t.n_names;
    o->name_row = host_alloc<uint64_t>(t.n_names);
    d2h(c, o->tokens, t.tokens.p, t.n_tok);
    d2h(c, o->record_index, t.tok_record.p, t.n_tok);
    std::memcpy(o->name_row, t.name_row.data(), t.n_names * sizeof(uint64_t));
    c->sync();
    *out = o;
  });
}

int itt_count_interval_overlaps(itt_ctx* ctx, const itt_records* recs, uint32_t stream, int64_t* out) {
  if (!out) return ITT_E_INVALID_ARGUMENT;
  *out = 0;
  return guarded(ctx, [&](Ctx* c) {
    if (!recs || recs->n == 0) return;
    TraceState t;
    prepare(c, t, recs, false);
    compact_main(t, stream, false);
    *out = count_overlaps(t);
  });
}

// ------------------------------------------------------------------ primitives
int itt_radix_sort_pairs_u32(itt_ctx* ctx, uint32_t* keys, uint32_t* vals, uint64_t n, int begin_bit, int end_bit,
                             int mem) {
  return guarded(ctx, [&](Ctx* c) {
    if (n == 0) return;
    if (!keys || !vals || begin_bit < 0 || end_bit > 32 || begin_bit >= end_bit)
      fail(ITT_E_INVALID_ARGUMENT, "radix_sort: bad arguments");
    DBuf<uint32_t> k0, v0, k1(c, n), v1(c, n);
    uint32_t* kp = keys;
    uint32_t* vp = vals;
    if (mem != ITT_MEM_DEVICE) {
      k0.alloc(c, n);
      v0.alloc(c, n);
      h2d(c, k0.p, keys, n);
      h2d(c, v0.p, vals, n);
      kp = k0.p;
      vp = v0.p;
    }
    radix::Scratch rs;
    const bool alt = radix_sort_pairs<uint32_t>(c, kp, vp, k1.p, v1.p, n, begin_bit, end_bit, rs);
    const uint32_t* rk = alt ? k1.p : kp;
    const uint32_t* rv = alt ? v1.p : vp;
    const cudaMemcpyKind kind = mem == ITT_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (rk != keys) ITT_CUDA(cudaMemcpyAsync(keys, rk, n * 4, kind, c->stream));
    if (rv != vals) ITT_CUDA(cudaMemcpyAsync(vals, rv, n * 4, kind, c->stream));
  });
}

// ------------------------------------------------------------------ mining
int itt_suffix_array(itt_ctx* ctx, const int32_t* tokens, uint64_t n, int32_t term, uint32_t* sa, uint32_t* lcp) {
  return guarded(ctx, [&](Ctx* c) {
    if (!sa || (n && !tokens)) fail(ITT_E_INVALID_ARGUMENT, "suffix_array: null argument");
    suffix_array_any(c, tokens, n, term, 0xFFFFFFFFu, sa, lcp);
  });
}

int itt_suffix_array_capped(itt_ctx* ctx, const int32_t* tokens, uint64_t n, int32_t term, uint32_t cap, uint32_t* sa,
                            uint32_t* lcp) {
  return guarded(ctx, [&](Ctx* c) {
    if (!sa || (n && !tokens)) fail(ITT_E_INVALID_ARGUMENT, "suffix_array: null argument");
    if (cap == 0) fail(ITT_E_INVALID_ARGUMENT, "suffix_array: cap must be positive");
    suffix_array_any(c, tokens, n, term, cap, sa, lcp);
  });
}

namespace {
__global__ void k_collect_repeats(const uint32_t* __restrict__ lcp, const uint32_t* __restrict__ cnt,
                                  const uint32_t* __restrict__ par, const uint32_t* __restrict__ lb,
                                  const uint32_t* __restrict__ sa, uint64_t np, int64_t min_count, int64_t max_len,
                                  itt_repeat* out, unsigned int* n_out) {
  const uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= np || cnt[k] == 0) return;
  const int64_t c = cnt[k];
  if (c < min_count) return;
  const int64_t len = imin64(static_cast<int64_t>(lcp[k]), max_len);
  if (len <= static_cast<int64_t>(par[k])) return;
  uint32_t m = 0xFFFFFFFFu;
  for (uint32_t q = 0; q < c; ++q) m = min(m, sa[lb[k] + q]);
  const unsigned i = atomicAdd(n_out, 1u);
  out[i].start = static_cast<int32_t>(m);
  out[i].length = static_cast<int32_t>(len);
  out[i].count = c;
}
}  // namespace

int itt_enumerate_repeats(itt_ctx* ctx, const int32_t* tokens, uint64_t n, int32_t term, int64_t min_count, int64_t max_len,
                          itt_repeat** out, uint64_t* n_out) {
  if (!out || !n_out) return ITT_E_INVALID_ARGUMENT;
  *out = nullptr;
  *n_out = 0;
  return guarded(ctx, [&](Ctx* c) {
    itt_repeat* res = nullptr;
    uint64_t cnt = 0;
    if (max_len >= 1 && n > 0) {  // mine.hpp:50
      DBuf<int32_t> dt;
      tokens_to_device(c, tokens, n, dt);
      SuffixState s;
      radix::Scratch rs;
      ScanScratch sc;
      // repeats longer than max_len are cut to max_len: groups by max_len + 1 symbols suffice
      const uint32_t cap = static_cast<uint32_t>(std::min<int64_t>(max_len, 0xFFFFFFFEll) + 1);
      build_suffix_array(c, dt.p, n, term, s, true, rs, sc, cap);
      IntervalState iv;
      lcp_intervals(c, s, iv);
      DBuf<itt_repeat> dout(c, s.np);
      DBuf<unsigned int> dn(c, 1);
      dn.zero();
      launch(c, "repeats_collect", s.np * 16.0, k_collect_repeats, dim3(grid_for(s.np, 256)), dim3(256), 0, s.lcp.p,
             iv.cnt.p, iv.par.p, iv.lb.p, s.sa.p, s.np, min_count, max_len, dout.p, dn.p);
      cnt = read1(c, dn.p);
      res = host_alloc<itt_repeat>(cnt);
      d2h(c, res, dout.p, cnt);
      c->sync();
    } else {
      res = host_alloc<itt_repeat>(0);
    }
    *out = res;
    *n_out = cnt;
  });
}

int itt_mine_patterns(itt_ctx* ctx, const int32_t* tokens, uint64_t n, int32_t term, const itt_mining_cfg* loops,
                      uint32_t n_loops, int multi, itt_pattern** out) {
  if (!out) return ITT_E_INVALID_ARGUMENT;
  *out = nullptr;
  return guarded(ctx, [&](Ctx* c) {
    std::vector<itt_mining_cfg> cfgs(loops, loops + n_loops);
    if (multi) {  // mine.hpp:134-146
      if (cfgs.empty()) fail(ITT_E_INVALID_CONFIG, "pattern-mining: no loop specs given");
      std::set<int64_t> seen;
      for (const auto& l : cfgs)
        if (!seen.insert(l.iterations).second)
          fail(ITT_E_INVALID_CONFIG, "pattern-mining: loop iteration counts must be pairwise distinct (duplicate " +
                                         std::to_string(l.iterations) + ")");
    } else {
      if (cfgs.empty()) fail(ITT_E_INVALID_ARGUMENT, "mine_pattern: no config");
      cfgs.resize(1);
    }
    DBuf<int32_t> dt;
    tokens_to_device(c, tokens, n, dt);
    SuffixState s;
    radix::Scratch rs;
    ScanScratch sc;
    build_suffix_array(c, dt.p, n, term, s, true, rs, sc, mining_cap(n, cfgs));
    IntervalState iv;
    lcp_intervals(c, s, iv, mining_cap(n, cfgs) - 1);  // list mode: the candidate intervals only
    const auto res = mine_loops(c, s, iv, cfgs, multi != 0);
    for (const auto& r : res)
      if (r.status) fail(r.status, r.error);
    if (multi)  // mine.hpp:155-164
      for (size_t a = 0; a < res.size(); ++a)
        for (size_t b = a + 1; b < res.size(); ++b)
          if (res[a].tokens == res[b].tokens)
            fail(ITT_E_AMBIGUOUS_LOOPS, "pattern-mining: loops " + std::to_string(a + 1) + " and " + std::to_string(b + 1) +
                                            " mined the same pattern; the loop specs are ambiguous");
    itt_pattern* o = host_alloc<itt_pattern>(res.size());
    for (size_t i = 0; i < res.size(); ++i) {
      o[i].length = static_cast<int64_t>(res[i].tokens.size());
      o[i].tokens = host_alloc<int32_t>(res[i].tokens.size());
      std::memcpy(o[i].tokens, res[i].tokens.data(), res[i].tokens.size() * 4);
      o[i].count = res[i].count;
      o[i].first_token = res[i].first_token;
      o[i].epsilon_used = res[i].epsilon_used;
    }
    *out = o;
  });
}

int itt_free_patterns(itt_ctx*, itt_pattern* p, uint32_t n_loops) {
  if (!p) return ITT_OK;
  for (uint32_t i = 0; i < n_loops; ++i) std::free(p[i].tokens);
  std::free(p);
  return ITT_OK;
}

int itt_mine_patterns_sa(itt_ctx* ctx, const int32_t* tokens, uint64_t n, int32_t term, const uint32_t* sa,
                         const uint32_t* lcp, const itt_mining_cfg* loops, uint32_t n_loops, int multi, itt_pattern** out) {
  if (!out) return ITT_E_INVALID_ARGUMENT;
  *out = nullptr;
  return guarded(ctx, [&](Ctx* c) {
    if (!sa || !lcp || (n && !tokens) || !loops || !n_loops) fail(ITT_E_INVALID_ARGUMENT, "mine_pattern: bad arguments");
    std::vector<itt_mining_cfg> cfgs(loops, loops + n_loops);
    if (!multi) cfgs.resize(1);
    SuffixState s;
    s.n = n;
    s.np = n + 1;
    s.lo = 0;
    s.text.alloc(c, n + 1);
    if (n) ITT_CUDA(cudaMemcpyAsync(s.text.p, tokens, n * 4, cudaMemcpyDeviceToDevice, c->stream));
    h2d(c, s.text.p + n, &term, 1);
    s.sa.alloc(c, n + 1);
    s.lcp.alloc(c, n + 1);
    ITT_CUDA(cudaMemcpyAsync(s.sa.p, sa, (n + 1) * 4, cudaMemcpyDeviceToDevice, c->stream));
    ITT_CUDA(cudaMemcpyAsync(s.lcp.p, lcp, (n + 1) * 4, cudaMemcpyDeviceToDevice, c->stream));
    IntervalState iv;
    lcp_intervals(c, s, iv, mining_cap(n, cfgs) - 1);  // list mode: the candidate intervals only
    const auto res = mine_loops(c, s, iv, cfgs, multi != 0);
    for (const auto& r : res)
      if (r.status) fail(r.status, r.error);
    if (multi)
      for (size_t a = 0; a < res.size(); ++a)
        for (size_t b = a + 1; b < res.size(); ++b)
          if (res[a].tokens == res[b].tokens)
            fail(ITT_E_AMBIGUOUS_LOOPS, "pattern-mining: loops " + std::to_string(a + 1) + " and " + std::to_string(b + 1) +
                                            " mined the same pattern; the loop specs are ambiguous");
    itt_pattern* o = host_alloc<itt_pattern>(res.size());
    for (size_t i = 0; i < res.size(); ++i) {
      o[i].length = static_cast<int64_t>(res[i].tokens.size());
      o[i].tokens = host_alloc<int32_t>(res[i].tokens.size());
      std::memcpy(o[i].tokens, res[i].tokens.data(), res[i].tokens.size() * 4);
      o[i].count = res[i].count;
      o[i].first_token = res[i].first_token;
      o[i].epsilon_used = res[i].epsilon_used;
    }
    *out = o;
  });
}

// ------------------------------------------------------------------ distributed SA steps (dist.cu)
int itt_dsa_keys(itt_ctx* ctx, const int32_t* text, uint64_t np, uint64_t lo, uint64_t cnt, int sym_bits, int k,
                 const uint32_t* rank, const uint32_t* rank2, uint64_t n2, int b, uint64_t* a, uint32_t* v) {
  return guarded(ctx, [&](Ctx* c) {
    if (np >= 0x7FFFFFFFull || lo + cnt > np) fail(ITT_E_INVALID_ARGUMENT, "dsa: positions out of range");
    if (rank ? (b < 1 || b > 32) : (sym_bits < 1 || k < 1 || sym_bits * k > 64)) fail(ITT_E_INVALID_ARGUMENT, "dsa: bad key width");
    dsa::keys(c, text, np, lo, cnt, sym_bits, k, rank, rank2, n2, b, a, v);
  });
}
int itt_dsa_partition(itt_ctx* ctx, const uint64_t* a, const uint32_t* b, uint64_t cnt, int mode, const uint64_t* spl_a,
                      const uint32_t* spl_b, uint32_t nspl, const uint64_t* bounds, uint32_t P, uint64_t* out_a,
                      uint32_t* out_b, uint64_t* counts) {
  return guarded(ctx, [&](Ctx* c) {
    if (!counts || P < 1 || P > 256 || (mode == 0 && (nspl + 1 != P || (nspl && (!spl_a || !spl_b)) || (cnt && !b))) ||
        (mode == 1 && !bounds) || (mode != 0 && mode != 1))
      fail(ITT_E_INVALID_ARGUMENT, "dsa: bad partition arguments");
    dsa::partition(c, a, b, cnt, mode, spl_a, spl_b, nspl, bounds, P, out_a, out_b, counts);
  });
}
int itt_dsa_sort(itt_ctx* ctx, uint64_t* a, uint32_t* b, uint64_t cnt, int bits) {
  return guarded(ctx, [&](Ctx* c) {
    if (bits < 0 || bits > 64) fail(ITT_E_INVALID_ARGUMENT, "dsa: bad sort width");
    dsa::sort(c, a, b, cnt, bits);
  });
}
int itt_dsa_ids(itt_ctx* ctx, const uint64_t* a, const uint32_t* b, uint64_t cnt, int has_prev, uint64_t prev,
                uint32_t offset, uint64_t* out, uint64_t* n_groups) {
  return guarded(ctx, [&](Ctx* c) {
    if (!n_groups) fail(ITT_E_INVALID_ARGUMENT, "dsa: null n_groups");
    *n_groups = dsa::ids(c, a, b, cnt, has_prev != 0, prev, offset, out);
  });
}
int itt_dsa_scatter(itt_ctx* ctx, const uint64_t* p, uint64_t cnt, uint64_t lo, uint32_t* dst) {
  return guarded(ctx, [&](Ctx* c) { dsa::scatter_hi(c, p, cnt, lo, dst); });
}
int itt_dsa_lcp_requests(itt_ctx* ctx, const uint64_t* packed, uint64_t cnt, uint64_t kbase, int has_prev, uint64_t prev,
                         uint64_t* a, uint32_t* b) {
  return guarded(ctx, [&](Ctx* c) { dsa::lcp_requests(c, packed, cnt, kbase, has_prev != 0, prev, a, b); });
}
int itt_dsa_kasai(itt_ctx* ctx, const int32_t* text, uint64_t np, uint64_t lo, uint64_t cnt, const uint64_t* req_a,
                  const uint32_t* req_b, uint32_t cap, uint64_t* out) {
  return guarded(ctx, [&](Ctx* c) {
    if (cap < 1) fail(ITT_E_INVALID_ARGUMENT, "dsa: cap must be >= 1");
    dsa::kasai(c, text, np, lo, cnt, req_a, req_b, cap, out);
  });
}
int itt_dsa_sample(itt_ctx* ctx, const uint64_t* a, const uint32_t* b, uint64_t cnt, uint32_t s, uint64_t* out_a,
                   uint32_t* out_b) {
  return guarded(ctx, [&](Ctx* c) { dsa::sample(c, a, b, cnt, s, out_a, out_b); });
}

// ------------------------------------------------------------------ a12 op profile
namespace {
__global__ void k_check_ops(const int32_t* __restrict__ tok, uint64_t n, uint32_t n_ops, unsigned* bad) {
  const uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j < n && static_cast<uint32_t>(tok[j]) >= n_ops) atomicOr(bad, 1u);
}
}  // namespace

int itt_op_profile(itt_ctx* ctx, const int32_t* tokens, const int64_t* tok_start, const int64_t* tok_end,
                   const uint8_t* tok_kind, uint64_t n, uint32_t n_ops, const itt_span* spans, uint64_t n_spans,
                   int method, itt_op_total* op_totals, itt_iter_op_total* iter_totals, itt_op_cell** cells,
                   uint64_t* n_cells) {
  if (cells && !n_cells) return ITT_E_INVALID_ARGUMENT;
  if (cells) *cells = nullptr;
  if (n_cells) *n_cells = 0;
  if (op_totals && n_ops) std::memset(op_totals, 0, static_cast<size_t>(n_ops) * sizeof(itt_op_total));
  if (n_spans && (!tokens || !tok_start || !tok_end || !tok_kind || !spans)) return ITT_E_INVALID_ARGUMENT;
  return guarded(ctx, [&](Ctx* c) {
    if (n_spans == 0) return;
    if (n >= 0xFFFFFFFFull) fail(ITT_E_INVALID_ARGUMENT, "metrics: sequence too long for 32-bit token indices");
    int64_t prev_end = -1;
    for (uint64_t i = 0; i < n_spans; ++i) {  // spans are approx_match output: disjoint and increasing
      if (spans[i].start_token <= prev_end || spans[i].end_token < spans[i].start_token ||
          static_cast<uint64_t>(spans[i].end_token) >= n)
        fail(ITT_E_INVALID_ARGUMENT, "metrics: spans must be disjoint, increasing and inside the token sequence");
      prev_end = spans[i].end_token;
    }
    auto up = [&](auto* src, auto& d) {  // host or device source (unified addressing)
      d.alloc(c, n);
      ITT_CUDA(cudaMemcpyAsync(d.p, src, n * sizeof(*src), cudaMemcpyDefault, c->stream));
    };
    DBuf<int32_t> dt;
    DBuf<int64_t> ds, de;
    DBuf<uint8_t> dk;
    up(tokens, dt);
    up(tok_start, ds);
    up(tok_end, de);
    up(tok_kind, dk);
    {
      DBuf<unsigned> bad(c, 1);
      bad.zero();
      // op ids must be < n_ops (the table is indexed by them)
      launch(c, "opprof_check", n * 4.0, k_check_ops, dim3(grid_for(n, 256)), dim3(256), 0, dt.p, n, n_ops, bad.p);
      if (read1(c, bad.p)) fail(ITT_E_INVALID_ARGUMENT, "metrics: op id outside [0, n_ops)");
    }
    SpanState sp;
    sp.n = n_spans;
    std::vector<uint32_t> s(n_spans), e(n_spans), x(n_spans);
    for (uint64_t i = 0; i < n_spans; ++i) {
      s[i] = static_cast<uint32_t>(spans[i].start_token);
      e[i] = static_cast<uint32_t>(spans[i].end_token);
      x[i] = static_cast<uint32_t>(spans[i].extra);
    }
    sp.start.alloc(c, n_spans);
    sp.end.alloc(c, n_spans);
    sp.extra.alloc(c, n_spans);
    h2d(c, sp.start.p, s.data(), n_spans);
    h2d(c, sp.end.p, e.data(), n_spans);
    h2d(c, sp.extra.p, x.data(), n_spans);
    ScanScratch sc;
    radix::Scratch rs;
    const OpProfile op =
        op_profile(c, dt.p, ds.p, de.p, dk.p, n, n_ops, sp, method, cells != nullptr, op_totals, iter_totals, sc, rs);
    if (cells) {
      *cells = op.cells;
      *n_cells = op.n;
    }
  });
}

// ------------------------------------------------------------------ matching
int itt_approx_match(itt_ctx* ctx, const int32_t* tokens, uint64_t n, const int32_t* pattern, uint64_t m, int64_t k0,
                     itt_span** out, uint64_t* n_out) {
  if (!out || !n_out) return ITT_E_INVALID_ARGUMENT;
  *out = nullptr;
  *n_out = 0;
  return guarded(ctx, [&](Ctx* c) {
    SpanState sp;
    if (m > 0 && n >= m) {
      DBuf<int32_t> dt, dp;
      tokens_to_device(c, tokens, n, dt);
      tokens_to_device(c, pattern, m, dp);
      ScanScratch sc;
      approx_match_dev(c, dt.p, n, dp.p, pattern[0], m, k0, sp, sc);
    }
    std::vector<uint32_t> s(sp.n), e(sp.n), x(sp.n);
    d2h(c, s.data(), sp.start.p, sp.n);
    d2h(c, e.data(), sp.end.p, sp.n);
    d2h(c, x.data(), sp.extra.p, sp.n);
    c->sync();
    itt_span* o = host_alloc<itt_span>(sp.n);
    for (uint64_t i = 0; i < sp.n; ++i) o[i] = itt_span{s[i], e[i], x[i]};
    *out = o;
    *n_out = sp.n;
  });
}

// ------------------------------------------------------------------ aggregates
namespace {
__global__ void k_gather_tok_times(const uint64_t* __restrict__ ri, uint64_t n, const uint32_t* __restrict__ perm,
                                   const int64_t* __restrict__ start, const int64_t* __restrict__ dur,
                                   int64_t* __restrict__ ts, int64_t* __restrict__ te) {
  const uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const uint64_t k = ri[j];
  const uint64_t i = perm ? perm[k] : k;
  ts[j] = start[i];
  te[j] = start[i] + dur[i];
}
}  // namespace

int itt_iteration_metrics(itt_ctx* ctx, const itt_records* recs, const uint64_t* record_index, uint64_t n_tokens,
                          const itt_span* spans, uint64_t n_spans, itt_iter_row** rows, itt_clamps* clamps) {
  if (!rows || !clamps) return ITT_E_INVALID_ARGUMENT;
  *rows = nullptr;
  return guarded(ctx, [&](Ctx* c) {
    itt_iter_row* o = host_alloc<itt_iter_row>(n_spans);
    struct Free {
      itt_iter_row*& p;
      ~Free() { std::free(p); }
    } guard{o};
    itt_clamps cl{0, 0};
    if (n_spans > 0) {
      for (uint64_t i = 0; i < n_spans; ++i)
        if (spans[i].start_token < 0 || spans[i].end_token < spans[i].start_token ||
            static_cast<uint64_t>(spans[i].end_token) >= n_tokens)
          fail(ITT_E_INVALID_ARGUMENT, "metrics: span outside the token sequence");
      TraceState t;
      prepare(c, t, recs, false);
      compact_main(t, 0xFFFFFFFFu, false);  // HtoD list (all streams); the token columns come from record_index
      DBuf<uint64_t> ri(c, n_tokens);
      h2d(c, ri.p, record_index, n_tokens);
      DBuf<int64_t> ts(c, n_tokens + 1), te(c, n_tokens + 1);
      launch(c, "agg_gather", n_tokens * 40.0, k_gather_tok_times, dim3(grid_for(n_tokens, 256)), dim3(256), 0, ri.p, n_tokens,
             t.sorted ? nullptr : t.perm.p, t.rec.start, t.rec.dur, ts.p, te.p);
      SpanState sp;
      sp.n = n_spans;
      std::vector<uint32_t> s(n_spans), e(n_spans), x(n_spans);
      for (uint64_t i = 0; i < n_spans; ++i) {
        s[i] = static_cast<uint32_t>(spans[i].start_token);
        e[i] = static_cast<uint32_t>(spans[i].end_token);
        x[i] = static_cast<uint32_t>(spans[i].extra);
      }
      sp.start.alloc(c, n_spans);
      sp.end.alloc(c, n_spans);
      sp.extra.alloc(c, n_spans);
      h2d(c, sp.start.p, s.data(), n_spans);
      h2d(c, sp.end.p, e.data(), n_spans);
      h2d(c, sp.extra.p, x.data(), n_spans);
      iteration_aggregates(c, ts.p, te.p, n_tokens, t.htod_start.p, t.htod_end.p, t.htod_size.p, t.n_htod,
                           t.htod_range.p, sp, o, cl,
                           t.scan);
    }
    *rows = o;
    o = nullptr;  // ownership passes to the caller
    *clamps = cl;
  });
}

// ------------------------------------------------------------------ analyze
int itt_analyze(itt_ctx* ctx, const itt_records* recs, const itt_analyze_opts* opts, itt_analysis** out) {
  if (!out || !opts) return ITT_E_INVALID_ARGUMENT;
  *out = nullptr;
  return guarded(ctx, [&](Ctx* c) {
    if (opts->n_loops == 0 || !opts->loops)
      fail(ITT_E_INVALID_CONFIG, "analyze: at least one iteration count is required");
    if (!recs || recs->n == 0) fail(ITT_E_EMPTY_TRACE, "stream-classify: trace has no records");
    TraceState t;
    prepare(c, t, recs, true, /*allow_late_dur=*/true);
    // main stream: override or selection (pipeline.hpp:56-73)
    uint32_t main_stream = 0, n_main_streams = 0;
    int32_t override_non_main = 0;
    for (const auto& s : t.streams) n_main_streams += s.cls == ITT_CLASS_MAIN;
    if (opts->main_stream >= 0) {
      main_stream = static_cast<uint32_t>(opts->main_stream);
      const auto it = std::find_if(t.streams.begin(), t.streams.end(),
                                   [&](const itt_stream_summary& s) { return s.stream == main_stream; });
      if (it == t.streams.end())
        fail(ITT_E_EMPTY_MAIN_STREAM,
             "stream-classify: override stream " + std::to_string(main_stream) + " does not appear in the trace");
      override_non_main = it->cls != ITT_CLASS_MAIN;
    } else {
      main_stream = select_main(t.streams, &n_main_streams);
    }
    int64_t overlaps = 0;
    {
      StageTimer st(c, "tokens");
      compact_main(t, main_stream, false);
      if (t.n_tok == 0)
        fail(ITT_E_EMPTY_MAIN_STREAM, "stream-classify: stream " + std::to_string(main_stream) + " has no records");
      renumber_tokens(t);
      if (!t.rec.dur_host) {
        overlaps = count_overlaps(t);
        release_rows(t);  // row-level arrays are dead from here: HBM for the suffix array
      } else {  // the duration column is still crossing PCIe: ends after the suffix array and mining
        release_rows_but_late(t);
      }
    }
    // mining over one shared SA / LCP / interval set (pipeline.hpp:81-91)
    std::vector<itt_mining_cfg> cfgs;
    for (uint32_t k = 0; k < opts->n_loops; ++k) cfgs.push_back(itt_mining_cfg{opts->loops[k], opts->epsilon0, 0});
    const bool multi = cfgs.size() > 1;
    if (multi) {
      std::set<int64_t> seen;
      for (const auto& l : cfgs)
        if (!seen.insert(l.iterations).second)
          fail(ITT_E_INVALID_CONFIG, "pattern-mining: loop iteration counts must be pairwise distinct (duplicate " +
                                         std::to_string(l.iterations) + ")");
    }
    SuffixState s;
    {
      StageTimer st(c, "sa+lcp");
      if (opts->sa_provider) {  // e.g. the distributed suffix array (dist_sa.py)
        const uint64_t n = t.n_tok;
        const int32_t term = static_cast<int32_t>(t.n_names);
        s.n = n;
        s.np = n + 1;
        s.lo = 0;
        s.text.alloc(c, n + 1);
        ITT_CUDA(cudaMemcpyAsync(s.text.p, t.tokens.p, n * 4, cudaMemcpyDeviceToDevice, c->stream));
        h2d(c, s.text.p + n, &term, 1);
        s.sa.alloc(c, n + 1);
        s.lcp.alloc(c, n + 1);
        c->sync();
        tl_provider_error.clear();
        if (opts->sa_provider(opts->sa_user, s.text.p, n, term, mining_cap(n, cfgs), s.sa.p, s.lcp.p) != 0)
          fail(ITT_E_CUDA, "pattern-mining: the suffix-array provider failed" +
                               (tl_provider_error.empty() ? std::string() : ": " + tl_provider_error));
      } else {
        build_suffix_array(c, t.tokens.p, t.n_tok, static_cast<int32_t>(t.n_names), s, true, t.rs, t.scan,
                           mining_cap(t.n_tok, cfgs), /*known_alphabet=*/true);
      }
    }
    IntervalState iv;
    std::vector<MinedPattern> pats;
    {
      StageTimer st(c, "mine");
      lcp_intervals(c, s, iv, mining_cap(t.n_tok, cfgs) - 1);  // list mode: the candidate intervals only
      pats = mine_loops(c, s, iv, cfgs, multi);
    }
    if (t.rec.dur_host) {  // late durations: stream ends, token / HtoD ends, then the row arrays go
      StageTimer st(c, "late-ends");
      finish_late_durations(t);
      overlaps = count_overlaps(t);
      release_rows(t);
    }
    for (const auto& p : pats)
      if (p.status) fail(p.status, p.error);
    if (multi)
      for (size_t a = 0; a < pats.size(); ++a)
        for (size_t b = a + 1; b < pats.size(); ++b)
          if (pats[a].tokens == pats[b].tokens)
            fail(ITT_E_AMBIGUOUS_LOOPS, "pattern-mining: loops " + std::to_string(a + 1) + " and " + std::to_string(b + 1) +
                                            " mined the same pattern; the loop specs are ambiguous");
    // per loop: match + aggregates (pipeline.hpp:96-132)
    struct Holder {
      itt_analysis* a = nullptr;
      itt_ctx* ctx = nullptr;
      ~Holder() { itt_free_analysis(ctx, a); }
    } hold;
    hold.ctx = ctx;
    itt_analysis* a = hold.a = host_alloc<itt_analysis>(1);
    a->owner = ctx;
    fill_census(t, &a->census);
    a->main_stream = main_stream;
    a->n_main_streams = n_main_streams;
    a->main_stream_override_non_main = override_non_main;
    a->n_tokens = t.n_tok;
    a->n_names = t.n_names;
    a->name_row = host_alloc<uint64_t>(t.n_names);
    std::memcpy(a->name_row, t.name_row.data(), t.n_names * sizeof(uint64_t));
    a->overlapping_kernels = overlaps;
    a->n_loops = static_cast<uint32_t>(pats.size());
    a->loops = host_alloc<itt_loop_result>(pats.size());
    for (size_t k = 0; k < pats.size(); ++k) {
      const auto& p = pats[k];
      itt_loop_result& L = a->loops[k];
      L.iterations_declared = cfgs[k].iterations;
      L.pattern_length = static_cast<int64_t>(p.tokens.size());
      L.pattern_tokens = host_alloc<int32_t>(p.tokens.size());
      std::memcpy(L.pattern_tokens, p.tokens.data(), p.tokens.size() * 4);
      L.pattern_count = p.count;
      L.epsilon_used = p.epsilon_used;
      L.first_token = p.first_token;
      L.k0_used = opts->k0 >= 0 ? opts->k0 : (L.pattern_length + 3) / 4;  // default_k0, match.hpp:19-21
      DBuf<int32_t> dp;
      tokens_to_device(c, p.tokens.data(), p.tokens.size(), dp);
      SpanState sp;
      {
        StageTimer st(c, "match");
        approx_match_dev(c, t.tokens.p, t.n_tok, dp.p, p.tokens.empty() ? 0 : p.tokens[0], p.tokens.size(), L.k0_used, sp,
                         t.scan);
      }
      StageTimer st(c, "aggregates");
      L.n_iterations = sp.n;
      L.rows = static_cast<itt_iter_row*>(c->out_alloc(sp.n * sizeof(itt_iter_row)));  // pinned: DMA target
      iteration_aggregates(c, t.tok_start.p, t.tok_end.p, t.n_tok, t.htod_start.p, t.htod_end.p, t.htod_size.p, t.n_htod,
                           t.htod_range.p, sp,
                           L.rows, L.clamps, t.scan);
      if (opts->flags & (ITT_ANALYZE_OP_PROFILE | ITT_ANALYZE_OP_CELLS)) {  // a12 (no reference counterpart)
        StageTimer so(c, "op_profile");
        L.op_totals = static_cast<itt_op_total*>(c->out_alloc(std::max<size_t>(1, t.n_names) * sizeof(itt_op_total)));
        L.iter_op_totals =
            static_cast<itt_iter_op_total*>(c->out_alloc(std::max<uint64_t>(1, sp.n) * sizeof(itt_iter_op_total)));
        const OpProfile op = op_profile(c, t.tokens.p, t.tok_start.p, t.tok_end.p, t.tok_kind.p, t.n_tok, t.n_names, sp,
                                        ITT_OP_PROFILE_AUTO, (opts->flags & ITT_ANALYZE_OP_CELLS) != 0, L.op_totals,
                                        L.iter_op_totals, t.scan, t.rs);
        L.n_op_cells = op.n;
        L.op_cells = op.cells;
      }
    }
    *out = a;
    hold.a = nullptr;
  });
}

int itt_free_analysis(itt_ctx* ctx, itt_analysis* a) {
  if (!a) return ITT_OK;
  if (a->owner) ctx = a->owner;  // the pinned row blocks go back to the context that made them
  std::free(a->census.streams);
  std::free(a->name_row);
  for (uint32_t k = 0; k < a->n_loops; ++k) {
    std::free(a->loops[k].pattern_tokens);
    itt_free(ctx, a->loops[k].rows);
    itt_free(ctx, a->loops[k].op_cells);
    itt_free(ctx, a->loops[k].op_totals);
    itt_free(ctx, a->loops[k].iter_op_totals);
  }
  std::free(a->loops);
  std::free(a);
  return ITT_OK;
}

// ------------------------------------------------------------------ CSV ingest
struct ParsedHolder {
  itt_parsed_trace pub;  // first member: the C handle points here
  ParsedCsv csv;
  std::vector<const char*> labels, reasons, warnings;
};

int itt_parse_csv(itt_ctx* ctx, const char* text, uint64_t len, const char* origin_label, itt_parsed_trace** out) {
  if (!out || (len && !text)) return ITT_E_INVALID_ARGUMENT;
  *out = nullptr;
  ParsedHolder* h = new (std::nothrow) ParsedHolder;
  if (!h) return ITT_E_CUDA;
  const int rc = guarded(ctx, [&](Ctx* c) {
    parse_csv(c, text, len, origin_label ? origin_label : "trace.csv", h->csv);
    ParsedCsv& p = h->csv;
    itt_parsed_trace& o = h->pub;
    o.records = itt_records{p.n,      p.start, p.dur,    p.size,          p.flags, p.stream, p.device,
                            p.name_off, p.name_bytes, ITT_MEM_DEVICE, ITT_ORDER_UNKNOWN};
    o.line = p.line.data();
    for (const auto& x : p.device_labels) h->labels.push_back(x.c_str());
    for (const auto& x : p.skip_reason) h->reasons.push_back(x.c_str());
    for (const auto& x : p.warnings) h->warnings.push_back(x.c_str());
    o.n_device_labels = static_cast<uint32_t>(h->labels.size());
    o.device_labels = h->labels.data();
    o.rows_total = p.rows_total;
    o.rows_parsed = p.rows_parsed;
    o.rows_skipped = p.rows_skipped;
    o.n_skips = p.skip_line.size();
    o.skip_line = p.skip_line.data();
    o.skip_reason = h->reasons.data();
    for (int q = 0; q < kIngestCols; ++q) o.column[q] = p.col[q];
    o.n_warnings = static_cast<uint32_t>(h->warnings.size());
    o.warnings = h->warnings.data();
  });
  if (rc != ITT_OK) {
    h->csv.release();
    delete h;
    return rc;
  }
  *out = &h->pub;
  return ITT_OK;
}

int itt_free_parsed(itt_ctx* ctx, itt_parsed_trace* p) {
  if (!p) return ITT_OK;
  ParsedHolder* h = reinterpret_cast<ParsedHolder*>(p);
  if (ctx) cudaSetDevice(ctx->c.device);
  h->csv.release();
  delete h;
  return ITT_OK;
}

// ------------------------------------------------------------------ batch executor (C4)
// Batched suffix arrays for the executor (ITT_ANALYZE_BATCHED_SA): every analyze in flight reaches
// its suffix-array stage through itt_analyze_opts.sa_provider; when all of them are waiting there,
// the last to arrive builds all their suffix arrays in one doubling sequence (build_batched_sa,
// on its own context) and releases the others.  A trace that ends before that stage (an error)
// leaves the wave, which may complete it.
struct BatchSA {
  struct Req {
    const int32_t* tok;
    uint64_t n;
    int32_t term;
    uint32_t cap;
    uint32_t* sa;
    uint32_t* lcp;
    int status;
    std::string error;  // the wave build's failure, reported by the waiting trace's own analyze
  };
  std::mutex mu;
  std::condition_variable cv;
  int active = 0;
  bool running = false;
  std::vector<Req*> pending;
  uint64_t batches = 0, traces = 0;
};
static thread_local Ctx* tl_batch_ctx = nullptr;

// run the pending wave if every trace in flight is waiting for it (caller holds the lock)
static void batch_sa_maybe_run(BatchSA* b, std::unique_lock<std::mutex>& lk) {
  while (!b->running && !b->pending.empty() && static_cast<int>(b->pending.size()) == b->active) {
    b->running = true;
    std::vector<BatchSA::Req*> reqs;
    reqs.swap(b->pending);
    lk.unlock();
    int st = 0;
    try {
      Ctx* c = tl_batch_ctx;
      if (!c) throw std::runtime_error("batched suffix array: no context on this thread");
      // one doubling sequence per group of at most kBatchTokens suffixes (bounds 32-bit suffix
      // indices and the wave's HBM: ~60 B per suffix while the sequence runs)
      constexpr uint64_t kBatchTokens = 1ull << 28;
      size_t at = 0;
      while (at < reqs.size()) {
        std::vector<BatchSAItem> items;
        int32_t vmax = 0;
        uint32_t cap = 1;
        uint64_t total = 0;
        while (at < reqs.size() && (items.empty() || total + reqs[at]->n + 1 <= kBatchTokens)) {
          const auto* r = reqs[at++];
          items.push_back(BatchSAItem{r->tok, r->n, r->sa, r->lcp});
          vmax = std::max(vmax, r->term);
          cap = std::max(cap, r->cap);
          total += r->n + 1;
        }
        radix::Scratch rs;
        ScanScratch sc;
        build_batched_sa(c, items, vmax, cap, rs, sc);
      }
    } catch (const std::exception& e) {
      st = 1;
      // the wave's work may still be queued on the builder's stream: drain it before the waiters
      // resume (their outputs are in it), and give every waiter the cause
      if (tl_batch_ctx) cudaStreamSynchronize(tl_batch_ctx->stream);
      for (auto* r : reqs) r->error = e.what();
    }
    lk.lock();
    for (auto* r : reqs) r->status = st;
    ++b->batches;
    b->traces += reqs.size();
    b->running = false;
    b->cv.notify_all();
  }
}

static int batch_sa_provider(void* user, const int32_t* tok, uint64_t n, int32_t term, uint32_t cap, uint32_t* sa, uint32_t* lcp) {
  BatchSA* b = static_cast<BatchSA*>(user);
  BatchSA::Req r{tok, n, term, cap, sa, lcp, -1, {}};
  std::unique_lock<std::mutex> lk(b->mu);
  b->pending.push_back(&r);
  batch_sa_maybe_run(b, lk);
  b->cv.wait(lk, [&] { return r.status >= 0; });
  if (r.status) tl_provider_error = r.error;
  return r.status;
}

struct itt_batch {
  int device = 0;
  std::vector<itt_ctx*> ctx;
  std::vector<std::string> errors;
  BatchSA sa;
};

int itt_batch_create(int device, uint32_t workers, itt_batch** out) {
  if (!out || workers == 0) return ITT_E_INVALID_ARGUMENT;
  *out = nullptr;
  itt_batch* b = new (std::nothrow) itt_batch;
  if (!b) return ITT_E_CUDA;
  b->device = device;
  for (uint32_t w = 0; w < workers; ++w) {
    itt_ctx* c = nullptr;
    const int rc = itt_ctx_create(device, &c);
    if (rc != ITT_OK) {
      for (auto* x : b->ctx) itt_ctx_destroy(x);
      delete b;
      return rc;
    }
    if (const char* e = std::getenv("ITT_BATCH_BLOCKING")) c->c.blocking_sync = std::atoi(e) != 0;
    b->ctx.push_back(c);
  }
  *out = b;
  return ITT_OK;
}

int itt_batch_destroy(itt_batch* b) {
  if (!b) return ITT_OK;
  for (auto* c : b->ctx) itt_ctx_destroy(c);
  delete b;
  return ITT_OK;
}

int itt_batch_analyze(itt_batch* b, const itt_records* traces, uint64_t n, const itt_analyze_opts* opts,
                      int opts_per_trace, itt_analysis** out, int* status) {
  if (!b || (n && (!traces || !opts || !out || !status))) return ITT_E_INVALID_ARGUMENT;
  b->errors.assign(n, std::string());
  std::atomic<uint64_t> next{0};
  static const int seg_env = [] {  // ITT_BATCH_SEGMENTED=0/1 overrides the flag (A/B runs)
    const char* e = std::getenv("ITT_BATCH_SEGMENTED");
    return e && *e ? (*e != '0' ? 1 : 0) : -1;
  }();
  auto work = [&](itt_ctx* c) {
    cudaSetDevice(b->device);
    tl_batch_ctx = &c->c;
    for (uint64_t i = next.fetch_add(1); i < n; i = next.fetch_add(1)) {
      out[i] = nullptr;
      itt_analyze_opts o = opts_per_trace ? opts[i] : *opts;
      const bool batched = (seg_env >= 0 ? seg_env == 1 : (o.flags & ITT_ANALYZE_BATCHED_SA) != 0) && !o.sa_provider;
      if (batched) {
        o.sa_provider = batch_sa_provider;
        o.sa_user = &b->sa;
        std::lock_guard<std::mutex> lk(b->sa.mu);
        ++b->sa.active;
      }
      status[i] = itt_analyze(c, &traces[i], &o, &out[i]);
      if (status[i] != ITT_OK) b->errors[i] = itt_last_error(c);
      if (batched) {  // leaving the wave may complete it (a trace that failed before its SA stage)
        std::unique_lock<std::mutex> lk(b->sa.mu);
        --b->sa.active;
        batch_sa_maybe_run(&b->sa, lk);
      }
    }
    tl_batch_ctx = nullptr;
  };
  std::vector<std::thread> th;
  for (size_t w = 1; w < b->ctx.size(); ++w) th.emplace_back(work, b->ctx[w]);
  work(b->ctx[0]);
  for (auto& t : th) t.join();
  return ITT_OK;
}

int itt_batch_launch_count(itt_batch* b, uint64_t* out) {
  if (!b || !out) return ITT_E_INVALID_ARGUMENT;
  uint64_t t = 0;
  for (auto* c : b->ctx) t += c->c.launches;
  *out = t;
  return ITT_OK;
}

const char* itt_batch_error(itt_batch* b, uint64_t i) {
  if (!b || i >= b->errors.size()) return "";
  return b->errors[i].c_str();
}

int itt_batch_free(itt_batch* b, itt_analysis** out, uint64_t n) {
  (void)b;
  if (!out) return ITT_OK;
  for (uint64_t i = 0; i < n; ++i) {
    itt_free_analysis(nullptr, out[i]);
    out[i] = nullptr;
  }
  return ITT_OK;
}

}  // extern "C"
