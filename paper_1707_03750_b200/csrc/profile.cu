// profile.cu — a12: the second-level per-op profile, sm_100a.
//
// The north star's "per-iteration segmented reductions: kernel, memcpy and idle durations reduced
// per op and per iteration".  The reference has no such function; the cell
// definition is in include/itertrace_cuda.h (itt_op_cell).  It reuses the reference's windows
// (approx_match spans, match.hpp:41-85) and op-gap rule (metrics.hpp:145-157), so the idle column
// of iteration k sums to the reference's clamped gap sum of that iteration.
//
// Two device paths, the same cells bit for bit:
//  * shared-memory table (n_ops <= kSmemOps): one CTA per span accumulates count / kernel /
//    memcpy / idle per op with shared atomics (integer sums: order-independent, deterministic)
//    and compacts the present ops in op order at the span's offset (a distinct-op pre-pass +
//    scan gives the offsets);
//  * sort path (any n_ops): in-span tokens keyed (iteration << op_bits | op) by one LSD radix
//    sort, then a run-length segmented reduction.
#include <algorithm>
#include <cstring>

#include "pipeline.cuh"

namespace itt {

namespace {

constexpr int kOpBlock = 256;
// 28 B of shared memory per op id (3 x u64 sums + u32 count): 7936 ops = 217 KiB, under the
// 227 KiB cap
constexpr uint32_t kSmemOps = 7936;
constexpr size_t kOpSmemBytes = 28;

__device__ __forceinline__ int64_t clamped_gap(const int64_t* ts, const int64_t* te, uint64_t j) {
  const int64_t g = ts[j] - te[j - 1];
  return g > 0 ? g : 0;
}

// Per span: the distinct-op bit set gives distinct_ops (and +1 iteration for every op present),
// thread-local sums the iteration totals.  Each CTA walks a contiguous range of spans; the
// per-op iteration counts stay in shared memory and are flushed once per CTA.
__global__ void __launch_bounds__(kOpBlock) k_op_iter(const int32_t* __restrict__ tokens, const int64_t* __restrict__ ts,
                                                      const int64_t* __restrict__ te, const uint8_t* __restrict__ kind,
                                                      const uint32_t* __restrict__ sp_start,
                                                      const uint32_t* __restrict__ sp_end, uint64_t I, uint32_t n_ops,
                                                      uint32_t* __restrict__ distinct, itt_iter_op_total* __restrict__ it_tot,
                                                      itt_op_total* __restrict__ op_tot) {
  extern __shared__ uint32_t s_dyn[];
  const uint32_t words = (n_ops + 31) / 32;
  uint32_t* s_bits = s_dyn;
  uint32_t* s_iters = s_dyn + words;  // [n_ops] when op_tot
  __shared__ unsigned long long s_red[3][kOpBlock / 32];
  __shared__ uint32_t s_warp[kOpBlock / 32];
  if (op_tot)
    for (uint32_t v = threadIdx.x; v < n_ops; v += kOpBlock) s_iters[v] = 0;
  const uint64_t k0 = I * blockIdx.x / gridDim.x, k1 = I * (blockIdx.x + 1) / gridDim.x;
  for (uint64_t k = k0; k < k1; ++k) {
    for (uint32_t w = threadIdx.x; w < words; w += kOpBlock) s_bits[w] = 0;
    __syncthreads();
    const uint32_t s = sp_start[k], e = sp_end[k];
    unsigned long long kern = 0, mem = 0, idle = 0;
    for (uint32_t j = s + threadIdx.x; j <= e; j += kOpBlock) {
      const uint32_t v = static_cast<uint32_t>(__ldg(&tokens[j]));
      atomicOr(&s_bits[v >> 5], 1u << (v & 31));
      const unsigned long long d = static_cast<unsigned long long>(te[j] - ts[j]);
      if (kind[j] == ITT_KIND_KERNEL) kern += d;
      else mem += d;
      if (j > s) idle += static_cast<unsigned long long>(clamped_gap(ts, te, j));
    }
    for (int o = 16; o > 0; o >>= 1) {
      kern += __shfl_xor_sync(0xffffffffu, kern, o);
      mem += __shfl_xor_sync(0xffffffffu, mem, o);
      idle += __shfl_xor_sync(0xffffffffu, idle, o);
    }
    if (lane_id() == 0) s_red[0][threadIdx.x >> 5] = kern, s_red[1][threadIdx.x >> 5] = mem, s_red[2][threadIdx.x >> 5] = idle;
    __syncthreads();
    uint32_t cnt = 0;
    for (uint32_t w = threadIdx.x; w < words; w += kOpBlock) {
      uint32_t bits = s_bits[w];
      cnt += __popc(bits);
      if (op_tot)  // one thread per word: plain increments
        while (bits) {
          s_iters[w * 32 + __ffs(bits) - 1] += 1;
          bits &= bits - 1;
        }
    }
    uint32_t total;
    block_exclusive_scan<uint32_t, SumOp<uint32_t>, kOpBlock>(cnt, SumOp<uint32_t>(), &total, s_warp);
    if (threadIdx.x == 0) {
      if (distinct) distinct[k] = total;
      if (it_tot) {
        unsigned long long x = 0, y = 0, z = 0;
        for (int w = 0; w < kOpBlock / 32; ++w) x += s_red[0][w], y += s_red[1][w], z += s_red[2][w];
        it_tot[k] = itt_iter_op_total{static_cast<int64_t>(total), static_cast<int64_t>(x), static_cast<int64_t>(y),
                                      static_cast<int64_t>(z)};
      }
    }
    __syncthreads();  // s_bits / s_red reuse
  }
  if (op_tot)
    for (uint32_t v = threadIdx.x; v < n_ops; v += kOpBlock)
      if (s_iters[v]) atomicAdd(reinterpret_cast<unsigned long long*>(&op_tot[v].iterations), static_cast<unsigned long long>(s_iters[v]));
}

// Per-op totals at token level: each CTA takes a contiguous range of spans, accumulates a
// shared table (count / kernel / memcpy / idle per op) and flushes its non-zero entries with
// global atomics — CTAs x n_ops atomics instead of one per token or cell.  (Iterations per op come
// from k_op_iter's per-span bit sets.)
__global__ void __launch_bounds__(kOpBlock) k_op_totals(const int32_t* __restrict__ tokens, const int64_t* __restrict__ ts,
                                                        const int64_t* __restrict__ te, const uint8_t* __restrict__ kind,
                                                        const uint32_t* __restrict__ sp_start,
                                                        const uint32_t* __restrict__ sp_end, uint64_t I, uint32_t n_ops,
                                                        itt_op_total* __restrict__ tot) {
  extern __shared__ unsigned long long s_acc[];
  const uint32_t V = n_ops;
  unsigned long long* s_kern = s_acc;
  unsigned long long* s_mem = s_acc + V;
  unsigned long long* s_idle = s_acc + 2 * static_cast<size_t>(V);
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_acc + 3 * static_cast<size_t>(V));
  for (uint32_t v = threadIdx.x; v < V; v += kOpBlock) s_kern[v] = 0, s_mem[v] = 0, s_idle[v] = 0, s_cnt[v] = 0;
  __syncthreads();
  const uint64_t k0 = I * blockIdx.x / gridDim.x, k1 = I * (blockIdx.x + 1) / gridDim.x;
  for (uint64_t k = k0; k < k1; ++k) {  // no per-span state: no barrier between spans
    const uint32_t s = sp_start[k], e = sp_end[k];
    for (uint32_t j = s + threadIdx.x; j <= e; j += kOpBlock) {
      const uint32_t v = static_cast<uint32_t>(__ldg(&tokens[j]));
      atomicAdd(&s_cnt[v], 1u);
      atomicAdd(kind[j] == ITT_KIND_KERNEL ? &s_kern[v] : &s_mem[v], static_cast<unsigned long long>(te[j] - ts[j]));
      if (j > s) {
        const int64_t g = clamped_gap(ts, te, j);
        if (g) atomicAdd(&s_idle[v], static_cast<unsigned long long>(g));
      }
    }
  }
  __syncthreads();
  for (uint32_t v = threadIdx.x; v < V; v += kOpBlock) {
    if (!s_cnt[v]) continue;
    unsigned long long* o = reinterpret_cast<unsigned long long*>(&tot[v]);
    atomicAdd(&o[1], static_cast<unsigned long long>(s_cnt[v]));
    if (s_kern[v]) atomicAdd(&o[2], s_kern[v]);
    if (s_mem[v]) atomicAdd(&o[3], s_mem[v]);
    if (s_idle[v]) atomicAdd(&o[4], s_idle[v]);
  }
}

struct OffsetsF {  // exclusive prefix of the distinct counts
  const uint32_t* distinct;
  uint64_t* offs;
  __device__ __forceinline__ uint64_t load(uint64_t i) const { return distinct[i]; }
  __device__ __forceinline__ void store(uint64_t i, uint64_t excl, uint64_t) const { offs[i] = excl; }
};

struct CellArgs {
  const int32_t* tokens;
  const int64_t* ts;
  const int64_t* te;
  const uint8_t* kind;
  const uint32_t* sp_start;
  const uint32_t* sp_end;
  const uint64_t* offs;
  uint32_t n_ops;
  itt_op_cell* cells;
};

__global__ void __launch_bounds__(kOpBlock) k_op_cells_smem(CellArgs a) {
  extern __shared__ unsigned long long s_acc[];  // kernel[n_ops], memcpy[n_ops], idle[n_ops], count[n_ops] (u32)
  __shared__ uint32_t s_warp[kOpBlock / 32];
  const uint32_t V = a.n_ops;
  unsigned long long* s_kern = s_acc;
  unsigned long long* s_mem = s_acc + V;
  unsigned long long* s_idle = s_acc + 2 * static_cast<size_t>(V);
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_acc + 3 * static_cast<size_t>(V));
  for (uint32_t v = threadIdx.x; v < V; v += kOpBlock) s_kern[v] = 0, s_mem[v] = 0, s_idle[v] = 0, s_cnt[v] = 0;
  __syncthreads();
  const uint32_t k = blockIdx.x;
  const uint32_t s = a.sp_start[k], e = a.sp_end[k];
  for (uint32_t j = s + threadIdx.x; j <= e; j += kOpBlock) {
    const uint32_t v = static_cast<uint32_t>(__ldg(&a.tokens[j]));
    const int64_t d = a.te[j] - a.ts[j];
    atomicAdd(&s_cnt[v], 1u);
    atomicAdd(a.kind[j] == ITT_KIND_KERNEL ? &s_kern[v] : &s_mem[v], static_cast<unsigned long long>(d));
    if (j > s) {
      const int64_t g = clamped_gap(a.ts, a.te, j);
      if (g) atomicAdd(&s_idle[v], static_cast<unsigned long long>(g));
    }
  }
  __syncthreads();
  // compaction in op order: thread t owns the contiguous op range [t*per, (t+1)*per)
  const uint32_t per = (V + kOpBlock - 1) / kOpBlock;
  const uint32_t v0 = min(V, threadIdx.x * per), v1 = min(V, v0 + per);
  uint32_t mine = 0;
  for (uint32_t v = v0; v < v1; ++v) mine += s_cnt[v] != 0;
  uint32_t total;
  uint32_t pos = block_exclusive_scan<uint32_t, SumOp<uint32_t>, kOpBlock>(mine, SumOp<uint32_t>(), &total, s_warp);
  itt_op_cell* out = a.cells + a.offs[k];
  for (uint32_t v = v0; v < v1; ++v) {
    const uint32_t c = s_cnt[v];
    if (!c) continue;
    itt_op_cell r;
    r.iteration = k;
    r.op = static_cast<int32_t>(v);
    r.count = c;
    r.pad_ = 0;
    r.kernel_ns = static_cast<int64_t>(s_kern[v]);
    r.memcpy_ns = static_cast<int64_t>(s_mem[v]);
    r.idle_ns = static_cast<int64_t>(s_idle[v]);
    out[pos++] = r;
  }
}

// ---- sort path
__global__ void k_span_ids(const uint32_t* __restrict__ sp_start, const uint32_t* __restrict__ sp_end, uint64_t I,
                           uint32_t* __restrict__ sid) {
  const uint64_t k = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (k >= I) return;
  for (uint32_t j = sp_start[k] + lane_id(); j <= sp_end[k]; j += 32) sid[j] = static_cast<uint32_t>(k);
}

struct InSpanF {  // compact in-span tokens into (iteration << op_bits | op, token index)
  const uint32_t* sid;
  const int32_t* tokens;
  int op_bits;
  uint64_t* keys;
  uint32_t* vals;
  __device__ __forceinline__ uint64_t load(uint64_t j) const { return sid[j] != kNone ? 1u : 0u; }
  __device__ __forceinline__ void store(uint64_t j, uint64_t excl, uint64_t v) const {
    if (!v) return;
    keys[excl] = (static_cast<uint64_t>(sid[j]) << op_bits) | static_cast<uint32_t>(tokens[j]);
    vals[excl] = static_cast<uint32_t>(j);
  }
};

struct RunF {  // run id of every sorted element (runs = equal keys)
  const uint64_t* keys;
  uint32_t* run;
  __device__ __forceinline__ uint64_t load(uint64_t i) const { return i == 0 || keys[i] != keys[i - 1] ? 1u : 0u; }
  __device__ __forceinline__ void store(uint64_t i, uint64_t excl, uint64_t v) const {
    run[i] = static_cast<uint32_t>(excl + v - 1);
  }
};

__global__ void k_run_accumulate(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                                 const uint32_t* __restrict__ run, uint64_t m, int op_bits, const int64_t* __restrict__ ts,
                                 const int64_t* __restrict__ te, const uint8_t* __restrict__ kind,
                                 const uint32_t* __restrict__ sp_start, itt_op_cell* __restrict__ cells) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const uint64_t key = keys[i];
  const uint32_t j = vals[i], r = run[i];
  const uint32_t k = static_cast<uint32_t>(key >> op_bits);
  itt_op_cell* c = &cells[r];
  if (i == 0 || run[i - 1] != r) {
    c->iteration = k;
    c->op = static_cast<int32_t>(key & ((1ull << op_bits) - 1));
    c->pad_ = 0;
  }
  atomicAdd(&c->count, 1u);
  const int64_t d = te[j] - ts[j];
  atomicAdd(reinterpret_cast<unsigned long long*>(kind[j] == ITT_KIND_KERNEL ? &c->kernel_ns : &c->memcpy_ns),
            static_cast<unsigned long long>(d));
  if (j > sp_start[k]) {
    const int64_t g = clamped_gap(ts, te, j);
    if (g) atomicAdd(reinterpret_cast<unsigned long long*>(&c->idle_ns), static_cast<unsigned long long>(g));
  }
}

// totals from a cell grid on the device (sort path: many op ids, so little atomic contention)
__global__ void k_cells_totals(const itt_op_cell* __restrict__ cells, uint64_t m, itt_op_total* __restrict__ op_tot,
                               itt_iter_op_total* __restrict__ it_tot) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const itt_op_cell c = cells[i];
  if (op_tot) {
    unsigned long long* o = reinterpret_cast<unsigned long long*>(&op_tot[c.op]);
    atomicAdd(&o[0], 1ull);
    atomicAdd(&o[1], static_cast<unsigned long long>(c.count));
    atomicAdd(&o[2], static_cast<unsigned long long>(c.kernel_ns));
    atomicAdd(&o[3], static_cast<unsigned long long>(c.memcpy_ns));
    atomicAdd(&o[4], static_cast<unsigned long long>(c.idle_ns));
  }
  if (it_tot) {
    unsigned long long* o = reinterpret_cast<unsigned long long*>(&it_tot[c.iteration]);
    atomicAdd(&o[0], 1ull);
    atomicAdd(&o[1], static_cast<unsigned long long>(c.kernel_ns));
    atomicAdd(&o[2], static_cast<unsigned long long>(c.memcpy_ns));
    atomicAdd(&o[3], static_cast<unsigned long long>(c.idle_ns));
  }
}

}  // namespace

OpProfile op_profile(Ctx* c, const int32_t* tokens, const int64_t* tok_start, const int64_t* tok_end,
                     const uint8_t* tok_kind, uint64_t n_tok, uint32_t n_ops, const SpanState& spans, int method,
                     bool want_cells, itt_op_total* op_totals, itt_iter_op_total* iter_totals, ScanScratch& scan,
                     radix::Scratch& rs) {
  OpProfile out;
  const uint64_t I = spans.n;
  if (op_totals && n_ops) std::memset(op_totals, 0, static_cast<size_t>(n_ops) * sizeof(itt_op_total));
  if (I == 0) return out;
  if (I > 0xFFFFFFFFull) fail(ITT_E_INVALID_ARGUMENT, "metrics: too many iterations for the op profile");
  if (method == ITT_OP_PROFILE_AUTO) method = n_ops <= kSmemOps ? ITT_OP_PROFILE_SMEM : ITT_OP_PROFILE_SORT;
  DBuf<itt_op_total> dot;
  DBuf<itt_iter_op_total> dit;
  if (op_totals) {
    dot.alloc(c, n_ops);
    dot.zero();
  }
  if (iter_totals) dit.alloc(c, I);
  DBuf<itt_op_cell> dc;
  if (method == ITT_OP_PROFILE_SMEM) {
    if (n_ops > kSmemOps) fail(ITT_E_INVALID_ARGUMENT, "metrics: too many op ids for the shared-memory op profile");
    const size_t bits_smem = ((n_ops + 31) / 32) * 4;
    const size_t table_smem = static_cast<size_t>(n_ops) * kOpSmemBytes;
    DBuf<uint32_t> distinct;
    if (want_cells) distinct.alloc(c, I);
    const unsigned span_grid = static_cast<unsigned>(std::min<uint64_t>(I, static_cast<uint64_t>(c->sm_count) * 8));
    if (want_cells || iter_totals || op_totals) {
      const size_t iter_smem = bits_smem + (op_totals ? static_cast<size_t>(n_ops) * 4 : 0);
      smem_optin(c, k_op_iter, iter_smem);
      launch(c, "opprof_iter", static_cast<double>(n_tok) * 21.0 + I * 40.0, k_op_iter, dim3(span_grid), dim3(kOpBlock),
             iter_smem, tokens, tok_start, tok_end, tok_kind, spans.start.p, spans.end.p, I, n_ops,
             want_cells ? distinct.p : nullptr, iter_totals ? dit.p : nullptr, op_totals ? dot.p : nullptr);
    }
    if (op_totals) {
      smem_optin(c, k_op_totals, table_smem);
      const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(I, static_cast<uint64_t>(c->sm_count) * 2));
      launch(c, "opprof_totals", static_cast<double>(n_tok) * 21.0, k_op_totals, dim3(grid), dim3(kOpBlock), table_smem,
             tokens, tok_start, tok_end, tok_kind, spans.start.p, spans.end.p, I, n_ops, dot.p);
    }
    if (want_cells) {
      DBuf<uint64_t> offs(c, I);
      device_scan<uint64_t, SumOp<uint64_t>>(c, "opprof_offsets", I * 12.0, OffsetsF{distinct.p, offs.p}, I, scan);
      out.n = scan.total(c);
      if (out.n) {
        dc.alloc(c, out.n);
        smem_optin(c, k_op_cells_smem, table_smem);
        CellArgs a{tokens, tok_start, tok_end, tok_kind, spans.start.p, spans.end.p, offs.p, n_ops, dc.p};
        launch(c, "opprof_cells", static_cast<double>(n_tok) * 21.0 + out.n * sizeof(itt_op_cell), k_op_cells_smem,
               dim3(static_cast<unsigned>(I)), dim3(kOpBlock), table_smem, a);
      }
    }
  } else {
    if (method != ITT_OP_PROFILE_SORT) fail(ITT_E_INVALID_ARGUMENT, "metrics: unknown op-profile method");
    DBuf<uint32_t> sid(c, n_tok);
    sid.fill_bytes(0xFF);
    launch(c, "opprof_span_ids", static_cast<double>(n_tok) * 4.0, k_span_ids, dim3(grid_for(I * 32, 256)), dim3(256), 0,
           spans.start.p, spans.end.p, I, sid.p);
    const int op_bits = bits_for(n_ops ? n_ops - 1 : 0);
    const int it_bits = bits_for(I - 1);
    if (op_bits + it_bits > 64) fail(ITT_E_INVALID_ARGUMENT, "metrics: op-profile key exceeds 64 bits");
    DBuf<uint64_t> k0(c, n_tok), k1(c, n_tok);
    DBuf<uint32_t> v0(c, n_tok), v1(c, n_tok);
    device_scan<uint64_t, SumOp<uint64_t>>(c, "opprof_in_span", n_tok * 20.0, InSpanF{sid.p, tokens, op_bits, k0.p, v0.p},
                                           n_tok, scan);
    const uint64_t m = scan.total(c);
    if (m) {
      const bool alt = radix_sort_pairs<uint64_t>(c, k0.p, v0.p, k1.p, v1.p, m, 0, op_bits + it_bits, rs);
      const uint64_t* keys = alt ? k1.p : k0.p;
      const uint32_t* vals = alt ? v1.p : v0.p;
      DBuf<uint32_t> run(c, m);
      device_scan<uint64_t, SumOp<uint64_t>>(c, "opprof_runs", m * 20.0, RunF{keys, run.p}, m, scan);
      out.n = scan.total(c);
      dc.alloc(c, out.n);
      dc.zero();
      launch(c, "opprof_accumulate", m * 45.0, k_run_accumulate, dim3(grid_for(m, 256)), dim3(256), 0, keys, vals, run.p,
             m, op_bits, tok_start, tok_end, tok_kind, spans.start.p, dc.p);
    }
    if (iter_totals) dit.zero();
    if (out.n && (op_totals || iter_totals))
      launch(c, "opprof_cell_totals", out.n * 40.0, k_cells_totals, dim3(grid_for(out.n, 256)), dim3(256), 0, dc.p, out.n,
             op_totals ? dot.p : nullptr, iter_totals ? dit.p : nullptr);
    if (!want_cells) out.n = 0;
  }
  if (op_totals) d2h(c, op_totals, dot.p, n_ops);
  if (iter_totals) d2h(c, iter_totals, dit.p, I);
  if (want_cells && out.n) {
    out.cells = static_cast<itt_op_cell*>(c->out_alloc(out.n * sizeof(itt_op_cell)));
    d2h(c, out.cells, dc.p, out.n);
  }
  c->sync();
  return out;
}

}  // namespace itt
