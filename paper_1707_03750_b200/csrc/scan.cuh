// scan.cuh — single-pass device-wide scan with decoupled look-back.
//
// One launch scans n items: tiles are claimed in order through an atomic counter, each
// tile publishes its aggregate (flag A) and then its inclusive prefix (flag P) in one
// 64-bit status word (2 flag bits + 62-bit value), and warp 0 of the next tile looks back
// over up to 32 predecessors per step.  Items are in a blocked arrangement (thread t owns
// ITEMS consecutive items), so functors see consecutive indices per thread and can fuse
// arbitrary per-item work (compaction writes, group-head scatters) into load/store.
//
//   struct F {
//     __device__ T load(uint64_t i) const;                  // i < n
//     __device__ void store(uint64_t i, T excl, T v) const;  // excl = op-prefix of items < i
//   };
#pragma once
#include "common.cuh"

namespace itt {

template <typename T>
struct SumOp {
  __device__ __forceinline__ T operator()(T a, T b) const { return a + b; }
  static __device__ __forceinline__ T identity() { return T(0); }
};
template <typename T>
struct MaxOp {
  __device__ __forceinline__ T operator()(T a, T b) const { return a > b ? a : b; }
  static __device__ __forceinline__ T identity() { return T(0); }
};

constexpr uint64_t kFlagA = 1ull << 62;
constexpr uint64_t kFlagP = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

template <typename T, typename Op>
__device__ __forceinline__ T warp_allreduce(T v, Op op) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Called by all 32 lanes of one warp; returns the exclusive prefix of `tile` (all lanes).
template <typename T, typename Op>
__device__ T tile_lookback(uint64_t* status, uint32_t tile, T aggregate, Op op) {
  const unsigned lane = lane_id();
  if (tile == 0) {
    if (lane == 0) st_relaxed_u64(&status[0], kFlagP | (static_cast<uint64_t>(aggregate) & kValMask));
    return Op::identity();
  }
  if (lane == 0) st_relaxed_u64(&status[tile], kFlagA | (static_cast<uint64_t>(aggregate) & kValMask));
  T excl = Op::identity();
  int64_t base = static_cast<int64_t>(tile) - 1;
  for (;;) {
    const int64_t idx = base - static_cast<int64_t>(lane);
    uint64_t s = kFlagP;  // idx < 0: identity inclusive prefix
    if (idx >= 0) {
      do {
        s = ld_relaxed_u64(&status[idx]);
      } while ((s >> 62) == 0);
    }
    __syncwarp();
    const unsigned pm = __ballot_sync(0xffffffffu, (s >> 62) == 2);
    const int stop = pm ? __ffs(pm) - 1 : 31;
    T v = (static_cast<int>(lane) <= stop) ? static_cast<T>(s & kValMask) : Op::identity();
    v = warp_allreduce(v, op);
    excl = op(excl, v);
    if (pm) break;
    base -= 32;
  }
  if (lane == 0) st_relaxed_u64(&status[tile], kFlagP | (static_cast<uint64_t>(op(excl, aggregate)) & kValMask));
  return excl;
}

// Block-wide exclusive scan of one value per thread; returns exclusive prefix, writes total.
template <typename T, typename Op, int BLOCK>
__device__ __forceinline__ T block_exclusive_scan(T v, Op op, T* total, T* smem_warp /*[BLOCK/32]*/) {
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  T inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, inc, o);
    if (static_cast<int>(lane) >= o) inc = op(inc, u);
  }
  if (lane == 31) smem_warp[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    constexpr int NW = BLOCK / 32;
    T w = static_cast<int>(lane) < NW ? smem_warp[lane] : Op::identity();
    T wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T u = __shfl_up_sync(0xffffffffu, wi, o);
      if (static_cast<int>(lane) >= o) wi = op(wi, u);
    }
    if (static_cast<int>(lane) < NW) smem_warp[lane] = wi;  // inclusive warp prefix
  }
  __syncthreads();
  const T warp_excl = warp == 0 ? Op::identity() : smem_warp[warp - 1];
  *total = smem_warp[BLOCK / 32 - 1];
  // exclusive within warp: inclusive minus own (via shfl of previous lane's inclusive)
  T prev = __shfl_up_sync(0xffffffffu, inc, 1);
  T excl_in_warp = lane == 0 ? Op::identity() : prev;
  return op(warp_excl, excl_in_warp);
}

template <typename T, typename Op, typename F, int BLOCK, int ITEMS>
__global__ void __launch_bounds__(BLOCK) k_scan(F f, uint64_t n, uint64_t* status, uint32_t* tile_counter) {
  __shared__ T s_warp[BLOCK / 32];
  __shared__ uint32_t s_tile;
  __shared__ T s_prefix;
  Op op;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t base = static_cast<uint64_t>(tile) * (BLOCK * ITEMS) + static_cast<uint64_t>(threadIdx.x) * ITEMS;
  T vals[ITEMS];
  T run = Op::identity();
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint64_t i = base + k;
    vals[k] = i < n ? f.load(i) : Op::identity();
    run = op(run, vals[k]);
  }
  T total;
  T texcl = block_exclusive_scan<T, Op, BLOCK>(run, op, &total, s_warp);
  if (threadIdx.x < 32) {
    T p = tile_lookback<T, Op>(status, tile, total, op);
    if (threadIdx.x == 0) s_prefix = p;
  }
  __syncthreads();
  T acc = op(s_prefix, texcl);
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint64_t i = base + k;
    if (i < n) f.store(i, acc, vals[k]);
    acc = op(acc, vals[k]);
  }
}

// Scratch for one scan launch: [counter u64][status u64 x tiles], zeroed per launch.
struct ScanScratch {
  DBuf<uint64_t> buf;
  uint64_t tiles = 0;
  void prepare(Ctx* c, uint64_t t) {
    if (buf.n < t + 1) buf.alloc(c, t + 1);
    tiles = t;
    ITT_CUDA(cudaMemsetAsync(buf.p, 0, (t + 1) * sizeof(uint64_t), c->stream));
  }
  // inclusive total of the last scan (the last tile's P word), synchronizes
  uint64_t total(Ctx* c) {
    if (tiles == 0) return 0;
    const uint64_t w = read1(c, buf.p + tiles);
    return w & kValMask;
  }
};

// Reduce-then-scan for large scans: (1) per-tile totals, (2) one block scans them, (3) every tile
// rescans its items from a known prefix and stores.  Loads run twice (functors' loads are pure),
// but no CTA waits at a barrier behind a look-back chain — on long scans that wait, not the
// bytes, set the single-pass kernel's time (C3 compaction: 1.97 -> 1.48 ms).
template <typename T, typename Op, typename F, int BLOCK, int ITEMS>
__global__ void __launch_bounds__(BLOCK) k_scan_reduce(F f, uint64_t n, T* __restrict__ tile_vals) {
  __shared__ T s_w[BLOCK / 32];
  Op op;
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * (BLOCK * ITEMS) + static_cast<uint64_t>(threadIdx.x) * ITEMS;
  T run = Op::identity();
#pragma unroll
  for (int k = 0; k < ITEMS; ++k)
    if (base + k < n) run = op(run, f.load(base + k));
  run = warp_allreduce(run, op);
  if (lane_id() == 0) s_w[threadIdx.x >> 5] = run;
  __syncthreads();
  if (threadIdx.x == 0) {
    T t = s_w[0];
    for (int w = 1; w < BLOCK / 32; ++w) t = op(t, s_w[w]);
    tile_vals[blockIdx.x] = t;
  }
}
// exclusive scan of the tile totals in place: one block walking chunks of 8K (coalesced)
template <typename T, typename Op>
__global__ void __launch_bounds__(1024) k_scan_tile_totals(T* __restrict__ tv, uint64_t tiles) {
  __shared__ T s_warp[32];
  constexpr int kPer = 8;
  Op op;
  T carry = Op::identity();
  for (uint64_t c0 = 0; c0 < tiles; c0 += 1024 * kPer) {
    const uint64_t b0 = c0 + static_cast<uint64_t>(threadIdx.x) * kPer;
    T v[kPer], run = Op::identity();
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      v[q] = b0 + q < tiles ? tv[b0 + q] : Op::identity();
      run = op(run, v[q]);
    }
    T total;
    T acc = op(carry, block_exclusive_scan<T, Op, 1024>(run, op, &total, s_warp));
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      if (b0 + q < tiles) tv[b0 + q] = acc;
      acc = op(acc, v[q]);
    }
    carry = op(carry, total);
    __syncthreads();
  }
}
// the last tile also writes the inclusive total where ScanScratch::total reads it
template <typename T, typename Op, typename F, int BLOCK, int ITEMS>
__global__ void __launch_bounds__(BLOCK) k_scan_apply(F f, uint64_t n, const T* __restrict__ tile_excl, uint64_t* total_word) {
  __shared__ T s_warp[BLOCK / 32];
  Op op;
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * (BLOCK * ITEMS) + static_cast<uint64_t>(threadIdx.x) * ITEMS;
  const T prefix = tile_excl[blockIdx.x];
  T vals[ITEMS];
  T run = Op::identity();
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    vals[k] = base + k < n ? f.load(base + k) : Op::identity();
    run = op(run, vals[k]);
  }
  T total;
  T acc = op(prefix, block_exclusive_scan<T, Op, BLOCK>(run, op, &total, s_warp));
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    if (base + k < n) f.store(base + k, acc, vals[k]);
    acc = op(acc, vals[k]);
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0)
    *total_word = kFlagP | (static_cast<uint64_t>(op(prefix, total)) & kValMask);
}

constexpr uint64_t kScanRsTiles = 4096;  // from this many tiles (8M items) on: reduce-then-scan

template <typename T, typename Op, int BLOCK = 256, int ITEMS = 8, typename F>
void device_scan(Ctx* c, const char* name, double bytes, F f, uint64_t n, ScanScratch& scratch) {
  if (n == 0) {
    scratch.tiles = 0;
    return;
  }
  constexpr uint64_t TILE = BLOCK * ITEMS;
  const uint64_t tiles = (n + TILE - 1) / TILE;
  scratch.prepare(c, tiles);
  if (tiles >= kScanRsTiles) {  // tile totals in the status words' space ([1, tiles]), the total at [tiles]
    T* tv = reinterpret_cast<T*>(scratch.buf.p + 1);
    launch(c, name, bytes * 0.5, k_scan_reduce<T, Op, F, BLOCK, ITEMS>, dim3(static_cast<unsigned>(tiles)), dim3(BLOCK), 0, f, n,
           tv);
    launch(c, "scan_tiles", tiles * 2.0 * sizeof(T), k_scan_tile_totals<T, Op>, dim3(1), dim3(1024), 0, tv, tiles);
    launch(c, name, bytes, k_scan_apply<T, Op, F, BLOCK, ITEMS>, dim3(static_cast<unsigned>(tiles)), dim3(BLOCK), 0, f, n, tv,
           scratch.buf.p + tiles);
    return;
  }
  uint32_t* counter = reinterpret_cast<uint32_t*>(scratch.buf.p);
  uint64_t* status = scratch.buf.p + 1;
  launch(c, name, bytes, k_scan<T, Op, F, BLOCK, ITEMS>, dim3(static_cast<unsigned>(tiles)), dim3(BLOCK), 0, f, n,
         status, counter);
}

}  // namespace itt
