// common.cuh — shared infrastructure of libitertrace_cuda.so: context, errors, device
// buffers, profiled launches, small device helpers.  sm_100a only.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "itertrace_cuda.h"

namespace itt {

// ---------------------------------------------------------------- errors
// Pipeline errors carry the reference's ErrorKind (as 1 + kind) and a stage-prefixed
// message (errors.hpp:23-34); device failures carry ITT_E_CUDA.
struct Error : std::runtime_error {
  int status;
  Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void fail(int status, const std::string& msg) { throw Error(status, msg); }

#define ITT_CUDA(call)                                                                                   \
  do {                                                                                                   \
    cudaError_t e_ = (call);                                                                             \
    if (e_ != cudaSuccess) {                                                                             \
      cudaGetLastError(); /* a non-sticky error must not resurface at the next launch check */           \
      ::itt::fail(ITT_E_CUDA, std::string("cuda: ") + cudaGetErrorString(e_) + " at " + __FILE__ + ":" + \
                                  std::to_string(__LINE__));                                             \
    }                                                                                                    \
  } while (0)

// ---------------------------------------------------------------- context
struct KStat {
  uint64_t launches = 0;
  double total_ms = 0, bytes = 0;
};

struct Ctx {
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // host->device streaming that overlaps kernels on `stream`
  const char* last_launch = "";
  std::string last_error;
  uint64_t launches = 0;
  bool profiling = false;
  std::map<std::string, KStat> stats;
  struct Pending {
    std::string name;
    double bytes;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> event_pool;
  cudaMemPool_t pool = nullptr;  // per-context stream-ordered pool (no cross-context lock contention)
  void* pinned = nullptr;  // small staging buffer for scalar readbacks
  size_t pinned_bytes = 0;

  cudaEvent_t take_event() {
    if (!event_pool.empty()) {
      cudaEvent_t e = event_pool.back();
      event_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    ITT_CUDA(cudaEventCreate(&e));
    return e;
  }
  // resolve event pairs after a stream synchronize
  // ITT_TIMELINE=1 (with profiling on): idle time of the stream between consecutive profiled
  // launches, booked as "gap:<previous>-><next>" (host round trips and launch latency)
  cudaEvent_t tl_last = nullptr;
  std::string tl_last_name;
  void resolve_profile() {
    static const bool timeline = std::getenv("ITT_TIMELINE") != nullptr;
    for (auto& p : pending) {
      float ms = 0;
      ITT_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
      KStat& s = stats[p.name];
      s.launches += 1;
      s.total_ms += ms;
      s.bytes += p.bytes;
      if (timeline) {
        if (tl_last) {
          float g = 0;
          ITT_CUDA(cudaEventElapsedTime(&g, tl_last, p.a));
          KStat& gs = stats["gap:" + tl_last_name + "->" + p.name];
          gs.launches += 1;
          gs.total_ms += g;
          event_pool.push_back(tl_last);
        }
        tl_last = p.b;
        tl_last_name = p.name;
      } else {
        event_pool.push_back(p.b);
      }
      event_pool.push_back(p.a);
    }
    pending.clear();
  }
  // blocking_sync: host waits sleep on an event instead of spinning — for many concurrent
  // contexts (the batch executor), where spinning waiters starve each other's host threads
  bool blocking_sync = false;
  cudaEvent_t sync_event = nullptr;
  void sync() {
    if (blocking_sync) {
      if (!sync_event) ITT_CUDA(cudaEventCreateWithFlags(&sync_event, cudaEventBlockingSync | cudaEventDisableTiming));
      ITT_CUDA(cudaEventRecord(sync_event, stream));
      ITT_CUDA(cudaEventSynchronize(sync_event));
    } else {
      ITT_CUDA(cudaStreamSynchronize(stream));
    }
    if (!pending.empty()) resolve_profile();
  }
  // Pinned host blocks for large variable-size outputs (per-iteration rows): the device writes them
  // directly, and itt_free returns them here for reuse instead of paying cudaMallocHost again.
  std::map<void*, size_t> out_live;
  std::multimap<size_t, void*> out_free;
  void* out_alloc(size_t bytes) {
    bytes = bytes < 256 ? 256 : bytes;
    auto it = out_free.lower_bound(bytes);
    if (it != out_free.end() && it->first <= 2 * bytes) {
      void* p = it->second;
      out_live[p] = it->first;
      out_free.erase(it);
      return p;
    }
    void* p = nullptr;
    ITT_CUDA(cudaMallocHost(&p, bytes));
    out_live[p] = bytes;
    return p;
  }
  bool out_release(void* p) {
    auto it = out_live.find(p);
    if (it == out_live.end()) return false;
    out_free.emplace(it->second, p);
    out_live.erase(it);
    return true;
  }
  // streamed-name windows: two persistent device buffers (cudaMalloc, outside the pool) reused
  // across calls — gigabyte-sized per-call pool blocks fragment the pool and force remapping
  void* win[2] = {nullptr, nullptr};
  size_t win_bytes = 0;
  uint8_t* window(int i, size_t bytes) {
    if (bytes > win_bytes) {
      ITT_CUDA(cudaStreamSynchronize(stream));
      if (copy_stream) ITT_CUDA(cudaStreamSynchronize(copy_stream));
      for (auto& w : win) {
        if (w) ITT_CUDA(cudaFree(w));
        w = nullptr;
      }
      for (auto& w : win) ITT_CUDA(cudaMalloc(&w, bytes));
      win_bytes = bytes;
    }
    return static_cast<uint8_t*>(win[i]);
  }
  // pinned bounce buffers for streaming names out of pageable host memory
  void* bounce[2] = {nullptr, nullptr};
  size_t bounce_bytes = 0;
  uint8_t* bounce_buf(int i, size_t bytes) {
    if (bytes > bounce_bytes) {
      if (copy_stream) ITT_CUDA(cudaStreamSynchronize(copy_stream));
      for (auto& b : bounce) {
        if (b) ITT_CUDA(cudaFreeHost(b));
        b = nullptr;
      }
      for (auto& b : bounce) ITT_CUDA(cudaMallocHost(&b, bytes));
      bounce_bytes = bytes;
    }
    return static_cast<uint8_t*>(bounce[i]);
  }
  // Small-allocation arena: one device block, bump-allocated during a call and reset when the
  // next call starts (guarded() synchronizes at the end of every call, and every DBuf of a call is
  // dead by then).  A 100K-event trace makes ~60 small allocations per analyze; taking them here
  // saves the allocator API calls that bound many-small-trace batches (C4).
  static constexpr size_t kArenaBytes = 64ull << 20, kArenaMaxAlloc = 2ull << 20;
  uint8_t* arena = nullptr;
  size_t arena_top = 0;
  // Large buffers (>= kBigBytes) bypass the stream-ordered pool: a per-context best-fit cache of
  // cudaMalloc'd blocks.  Calls repeat the same sizes, so steady state allocates nothing; the
  // pool, by contrast, fragments under mixed sizes and then maps fresh memory mid-call (measured:
  // 6-25 ms stalls for 100-400 MB requests on C3).  Single stream per context: a block handed
  // back is only reused by later work on the same stream, so stream order protects it.
  static constexpr size_t kBigBytes = 16u << 20;
  std::multimap<size_t, void*> big_free;  // capacity -> block
  std::map<void*, size_t> big_cap;        // every cached block (live or free) -> capacity
  size_t big_live = 0, big_high = 0;
  void big_trim() {  // give every free cached block back to the driver (allocation pressure)
    if (big_free.empty()) return;
    cudaStreamSynchronize(stream);
    for (auto& kv : big_free) {
      cudaFree(kv.second);
      big_cap.erase(kv.second);
    }
    big_free.clear();
  }
  void* big_take(size_t bytes) {
    auto it = big_free.lower_bound(bytes);
    void* p = nullptr;
    if (it != big_free.end() && it->first <= bytes + bytes / 4) {
      p = it->second;
      big_free.erase(it);
    } else {
      if (cudaMalloc(&p, bytes) != cudaSuccess) {
        cudaGetLastError();
        big_trim();
        if (cudaMalloc(&p, bytes) != cudaSuccess) {
          cudaGetLastError();
          fail(ITT_E_CUDA, "cuda: out of device memory (" + std::to_string(bytes >> 20) + " MiB block)");
        }
      }
      big_cap[p] = bytes;
    }
    big_live += big_cap[p];
    big_high = std::max(big_high, big_live);
    return p;
  }
  void big_give(void* p) {
    const size_t cap = big_cap.at(p);
    big_live -= cap;
    big_free.emplace(cap, p);
  }
  void* arena_take(size_t bytes) {
    bytes = (bytes + 255) & ~static_cast<size_t>(255);
    if (bytes > kArenaMaxAlloc) return nullptr;
    if (!arena) ITT_CUDA(cudaMalloc(&arena, kArenaBytes));
    if (arena_top + bytes > kArenaBytes) return nullptr;
    void* p = arena + arena_top;
    arena_top += bytes;
    return p;
  }
  cudaStream_t copier() {
    if (!copy_stream) ITT_CUDA(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
    return copy_stream;
  }
  // a second small pinned block for reads whose result is only needed after a later sync
  // (deferred_ev marks the copy): they must not share the staging buffer readback() reuses
  void* deferred = nullptr;
  cudaEvent_t deferred_ev = nullptr;
  // pinned ring for small host->device uploads (h2d), bump-allocated per call
  uint8_t* upload = nullptr;
  size_t upload_top = 0;
  static constexpr size_t kUploadBytes = 1u << 20;
  void* upload_slot(size_t bytes) {
    if (bytes > (64u << 10)) return nullptr;
    if (!upload) ITT_CUDA(cudaMallocHost(reinterpret_cast<void**>(&upload), kUploadBytes));
    const size_t at = (upload_top + 15) & ~static_cast<size_t>(15);
    if (at + bytes > kUploadBytes) return nullptr;
    upload_top = at + bytes;
    return upload + at;
  }
  void* deferred_block() {
    if (!deferred) {
      ITT_CUDA(cudaMallocHost(&deferred, 4096));
      ITT_CUDA(cudaEventCreateWithFlags(&deferred_ev, cudaEventDisableTiming));
    }
    return deferred;
  }
  void* staging(size_t bytes) {
    if (bytes > pinned_bytes) {
      if (pinned) cudaFreeHost(pinned);
      pinned_bytes = bytes < 4096 ? 4096 : bytes;
      ITT_CUDA(cudaMallocHost(&pinned, pinned_bytes));
    }
    return pinned;
  }
};

// Opt a kernel in to `bytes` of dynamic shared memory once per (kernel, device, size): the
// attribute is per device, and setting it on every call is an avoidable driver call.
template <typename K>
inline void smem_optin(Ctx* c, K* kernel, size_t bytes) {
  if (bytes <= 48 * 1024) return;
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{reinterpret_cast<const void*>(kernel), c->device}];
  if (have >= bytes) return;
  ITT_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
  have = bytes;
}

// Profiled launch: records CUDA events on the context stream around the launch when
// profiling is on; `bytes` is the launch's algorithmic HBM traffic.
struct LaunchScope {
  Ctx* c;
  const char* name;
  double bytes;
  cudaEvent_t a = nullptr;
  LaunchScope(Ctx* c_, const char* n, double b) : c(c_), name(n), bytes(b) {
    if (c->profiling) {
      a = c->take_event();
      ITT_CUDA(cudaEventRecord(a, c->stream));
    }
  }
  ~LaunchScope() noexcept(false) {
    c->last_launch = name;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fail(ITT_E_CUDA, std::string("cuda launch ") + name + ": " + cudaGetErrorString(e));
    c->launches += 1;
    if (c->profiling) {
      cudaEvent_t b = c->take_event();
      ITT_CUDA(cudaEventRecord(b, c->stream));
      c->pending.push_back({name, bytes, a, b});
    }
  }
};

// launch through a kernel pointer: <<<>>> on the context stream inside a LaunchScope
template <typename... KArgs, typename... Args>
inline void launch(Ctx* c, const char* name, double bytes, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                   Args&&... args) {
  LaunchScope ls(c, name, bytes);
  k<<<grid, block, smem, c->stream>>>(static_cast<KArgs>(args)...);
}

// Several small memsets in ONE launch (each cudaMemsetAsync is a GPU operation of its own; small
// traces are bound by the number of operations, not bytes).  Jobs need 4-byte aligned, 4-byte
// multiple ranges (pool / arena buffers are); anything else goes through cudaMemsetAsync.
struct FillJob {
  void* p;
  uint64_t words;   // 4-byte words
  uint32_t value;   // byte value replicated into the word
};
constexpr int kMaxFillJobs = 12;
struct FillBatch {
  FillJob j[kMaxFillJobs];
  int n;
};
static __global__ void k_fill_many(FillBatch b) {
  const FillJob& f = b.j[blockIdx.y];
  uint32_t* w = static_cast<uint32_t*>(f.p);
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < f.words;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    w[i] = f.value;
}
struct Fills {
  Ctx* c;
  FillBatch b{};
  uint64_t max_words = 0;
  explicit Fills(Ctx* ctx) : c(ctx) {}
  void add(void* p, size_t bytes, int value) {
    if (!bytes) return;
    if ((reinterpret_cast<uintptr_t>(p) & 3) || (bytes & 3) || b.n == kMaxFillJobs) {
      ITT_CUDA(cudaMemsetAsync(p, value, bytes, c->stream));
      return;
    }
    const uint32_t v = static_cast<uint8_t>(value) * 0x01010101u;
    b.j[b.n++] = FillJob{p, bytes / 4, v};
    max_words = std::max<uint64_t>(max_words, bytes / 4);
  }
  void flush();
};
inline void Fills::flush() {
  if (!b.n) return;
  const unsigned gx = static_cast<unsigned>(std::min<uint64_t>(64, (max_words + 255) / 256));
  launch(c, "fill_many", static_cast<double>(max_words) * 4.0, k_fill_many, dim3(std::max(1u, gx), b.n), dim3(256), 0, b);
  b.n = 0;
  max_words = 0;
}

// ---------------------------------------------------------------- device buffers
// Stream-ordered allocations from the device's default pool (release threshold raised
// at context creation so memory is recycled across calls instead of returned to the OS).
template <typename T>
struct DBuf {
  Ctx* c = nullptr;
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(Ctx* ctx, size_t count) { alloc(ctx, count); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : c(o.c), p(o.p), n(o.n), from_arena(o.from_arena), from_big(o.from_big) {
    o.p = nullptr, o.n = 0, o.from_arena = false, o.from_big = false;
  }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      c = o.c, p = o.p, n = o.n, from_arena = o.from_arena, from_big = o.from_big;
      o.p = nullptr, o.n = 0, o.from_arena = false, o.from_big = false;
    }
    return *this;
  }
  bool from_arena = false;
  bool from_big = false;
  void alloc(Ctx* ctx, size_t count) {
    release();
    c = ctx;
    n = count;
    if (count && (p = static_cast<T*>(ctx->arena_take(count * sizeof(T))))) {
      from_arena = true;
      return;
    }
    if (count * sizeof(T) >= Ctx::kBigBytes) {
      p = static_cast<T*>(ctx->big_take(count * sizeof(T)));
      from_big = true;
      return;
    }
    if (count) {
      timespec a, b;
      clock_gettime(CLOCK_MONOTONIC, &a);
      if (cudaMallocFromPoolAsync(reinterpret_cast<void**>(&p), count * sizeof(T), ctx->pool, ctx->stream) != cudaSuccess) {
        cudaGetLastError();
        ctx->big_trim();  // cached large blocks back to the driver, then retry
        ITT_CUDA(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&p), count * sizeof(T), ctx->pool, ctx->stream));
      }
      clock_gettime(CLOCK_MONOTONIC, &b);
      const double ms = (b.tv_sec - a.tv_sec) * 1e3 + (b.tv_nsec - a.tv_nsec) * 1e-6;
      if (ms > 5.0 && std::getenv("ITT_TRACE"))
        std::fprintf(stderr, "[itt]   slow alloc %.1f ms (%.1f MB) after %s\n", ms, count * sizeof(T) / 1e6, ctx->last_launch);
    }
  }
  void release() {
    if (p && from_arena) {
      p = nullptr;
      n = 0;
      from_arena = false;
      return;
    }
    if (p && from_big) {
      c->big_give(p);
      p = nullptr;
      n = 0;
      from_big = false;
      return;
    }
    if (p) {
      timespec a, b;
      clock_gettime(CLOCK_MONOTONIC, &a);
      cudaFreeAsync(p, c->stream);
      clock_gettime(CLOCK_MONOTONIC, &b);
      const double ms = (b.tv_sec - a.tv_sec) * 1e3 + (b.tv_nsec - a.tv_nsec) * 1e-6;
      if (ms > 5.0 && std::getenv("ITT_TRACE"))
        std::fprintf(stderr, "[itt]   slow free %.1f ms (%.1f MB) after %s\n", ms, n * sizeof(T) / 1e6, c->last_launch);
    }
    p = nullptr;
    n = 0;
  }
  ~DBuf() { release(); }
  T* get() const { return p; }
  size_t bytes() const { return n * sizeof(T); }
  void zero() {
    if (n) ITT_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), c->stream));
  }
  void fill_bytes(int v) {
    if (n) ITT_CUDA(cudaMemsetAsync(p, v, n * sizeof(T), c->stream));
  }
};

template <typename T>
inline void h2d(Ctx* c, T* dst, const T* src, size_t count) {
  if (!count) return;
  // small uploads go through the per-call pinned ring: a copy from pageable memory may wait for
  // the stream (a hidden round trip); the ring is reset when the next call starts (the previous
  // one synchronized), so a slot is never rewritten while its copy is pending
  const size_t bytes = count * sizeof(T);
  if (void* slot = c->upload_slot(bytes)) {
    std::memcpy(slot, src, bytes);
    src = static_cast<const T*>(slot);
  }
  ITT_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
}
template <typename T>
inline void d2h(Ctx* c, T* dst, const T* src, size_t count) {
  if (count) ITT_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDeviceToHost, c->stream));
}
// ITT_TRACE=1: per-stage wall time (synchronizing) and host round-trip counts on stderr
struct StageTimer {
  Ctx* c;
  const char* name;
  double t0;
  uint64_t l0;
  static bool on() {
    static const bool v = [] {
      const char* e = std::getenv("ITT_TRACE");
      return e && *e == '1';
    }();
    return v;
  }
  static double now() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
  }
  static uint64_t& syncs() {
    static uint64_t s = 0;
    return s;
  }
  StageTimer(Ctx* c_, const char* n) : c(c_), name(n), t0(0), l0(0) {
    if (on()) {
      cudaStreamSynchronize(c->stream);
      t0 = now();
      l0 = syncs();
    }
  }
  ~StageTimer() {
    if (on()) {
      cudaStreamSynchronize(c->stream);
      std::fprintf(stderr, "[itt] %-14s %8.3f ms  host syncs %llu\n", name, now() - t0,
                   static_cast<unsigned long long>(syncs() - l0));
    }
  }
};

// read `count` values back through the pinned staging buffer (synchronizes)
template <typename T>
inline void readback(Ctx* c, T* dst, const T* src, size_t count) {
  ++StageTimer::syncs();
  T* st = static_cast<T*>(c->staging(count * sizeof(T)));
  const double t0 = StageTimer::on() ? StageTimer::now() : 0.0;
  d2h(c, st, src, count);
  c->sync();
  if (StageTimer::on() && StageTimer::now() - t0 > 20.0)
    std::fprintf(stderr, "[itt]   slow readback %.1f ms after %s\n", StageTimer::now() - t0, c->last_launch);
  std::memcpy(static_cast<void*>(dst), st, count * sizeof(T));
}
// host memcpy split across threads (pageable source -> pinned bounce buffer)
inline void parallel_memcpy(uint8_t* dst, const uint8_t* src, uint64_t bytes) {
  constexpr uint64_t kMinPerThread = 32ull << 20;
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  const unsigned nt = static_cast<unsigned>(std::min<uint64_t>(hw, std::max<uint64_t>(1, bytes / kMinPerThread)));
  if (nt <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> th;
  const uint64_t per = (bytes + nt - 1) / nt;
  for (unsigned i = 0; i < nt; ++i) {
    const uint64_t a = i * per, b = std::min(bytes, a + per);
    if (a < b) th.emplace_back([=] { std::memcpy(dst + a, src + a, b - a); });
  }
  for (auto& x : th) x.join();
}

// Host -> device from memory that may be pageable: large unpinned copies go through the
// context's two pinned bounce buffers (multi-threaded host memcpy overlapping the DMA of the
// previous chunk) instead of the driver's single-threaded staging (~11 GB/s measured).
inline void h2d_bulk(Ctx* c, void* dst, const void* src, uint64_t bytes, cudaStream_t stream = nullptr) {
  if (!bytes) return;
  if (!stream) stream = c->stream;
  cudaPointerAttributes pa{};
  if (cudaPointerGetAttributes(&pa, src) != cudaSuccess) cudaGetLastError();
  if (pa.type == cudaMemoryTypeHost || bytes < (64ull << 20)) {
    ITT_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream));
    return;
  }
  constexpr uint64_t kChunk = 256ull << 20;
  cudaEvent_t done[2];
  for (auto& e : done) ITT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  const uint8_t* s = static_cast<const uint8_t*>(src);
  uint8_t* d = static_cast<uint8_t*>(dst);
  int k = 0;
  for (uint64_t off = 0; off < bytes; off += kChunk, ++k) {
    const int b = k & 1;
    const uint64_t n = std::min(kChunk, bytes - off);
    uint8_t* bb = c->bounce_buf(b, kChunk);
    if (k >= 2) ITT_CUDA(cudaEventSynchronize(done[b]));  // the DMA that last read this buffer
    parallel_memcpy(bb, s + off, n);
    ITT_CUDA(cudaMemcpyAsync(d + off, bb, n, cudaMemcpyHostToDevice, stream));
    ITT_CUDA(cudaEventRecord(done[b], stream));
  }
  ITT_CUDA(cudaStreamSynchronize(stream));  // the bounce buffers are reused by later calls
  for (auto& e : done) cudaEventDestroy(e);
}

// two device ranges in one host round trip
template <typename T, typename U>
inline void readback2(Ctx* c, T* a, const T* da, size_t na, U* b, const U* db, size_t nb) {
  ++StageTimer::syncs();
  const size_t ba = (na * sizeof(T) + 15) & ~static_cast<size_t>(15);
  uint8_t* st = static_cast<uint8_t*>(c->staging(ba + nb * sizeof(U)));
  d2h(c, reinterpret_cast<T*>(st), da, na);
  d2h(c, reinterpret_cast<U*>(st + ba), db, nb);
  c->sync();
  std::memcpy(static_cast<void*>(a), st, na * sizeof(T));
  std::memcpy(static_cast<void*>(b), st + ba, nb * sizeof(U));
}
template <typename T>
inline T read1(Ctx* c, const T* src) {
  T v;
  readback(c, &v, src, 1);
  return v;
}

inline unsigned grid_for(uint64_t n, unsigned block, unsigned cap = 1u << 30) {
  uint64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<unsigned>(g);
}

inline int bits_for(uint64_t maxval) {  // number of bits to represent values <= maxval (>= 1)
  int b = 1;
  while (b < 64 && (maxval >> b) != 0) ++b;
  return b;
}

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Bulk L2 prefetch (cp.async.bulk.prefetch.L2, sm_90+) of [p, p + bytes): the 16-byte aligned
// interior only.  Streaming kernels whose CTAs each take one tile issue it for the tile the CTA
// launched one residency wave later will take, so that CTA's loads hit L2 and DRAM stays busy
// while the resident CTAs rank / scan / look back.
__device__ __forceinline__ void prefetch_l2(const void* p, uint64_t bytes) {
  const uint64_t a = (reinterpret_cast<uint64_t>(p) + 15) & ~15ull;
  const uint64_t e = (reinterpret_cast<uint64_t>(p) + bytes) & ~15ull;
  if (e > a) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(static_cast<uint32_t>(e - a)) : "memory");
}
// tiles ahead to prefetch: one residency wave (CTAs per SM x SMs); ITT_L2_PREFETCH=0 disables
inline uint32_t prefetch_distance(int sm_count, int ctas_per_sm) {
  static const int on = [] {
    const char* e = std::getenv("ITT_L2_PREFETCH");
    return e && *e ? std::atoi(e) : 1;
  }();
  return on > 0 ? static_cast<uint32_t>(sm_count * ctas_per_sm * on) : 0u;
}
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

}  // namespace itt

namespace itt {
__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ uint64_t umax64(uint64_t a, uint64_t b) { return a > b ? a : b; }
}  // namespace itt
