// radix.cuh — hand-written onesweep LSD radix sort of (key, u32 value) pairs, sm_100a.
//
// Per sort: one upfront histogram pass computes the 256-bin histograms of every 8-bit
// digit at once (or the caller supplies them), passes whose digit is constant are
// skipped, and each remaining pass is ONE kernel (onesweep): a tile of BLOCK*ITEMS keys
// is loaded warp-striped with coalesced 4/8-byte loads, ranked per warp with
// __match_any_sync (stable: warp-major, round-major, lane order), the per-digit tile
// counts are published and prefixed by a decoupled look-back (one thread per digit),
// and the tile is re-ordered through shared memory so the global scatter writes
// contiguous runs per digit.
//
// Algorithmic traffic per pass: n * 2 * (sizeof(K) + 4) bytes (read + write key/value).
#pragma once
#include "common.cuh"

namespace itt {
namespace radix {

constexpr int kRadixBits = 8;
constexpr int kBins = 256;
constexpr int kBlock = 512;
constexpr int kItems = 8;
constexpr int kTile = kBlock * kItems;
constexpr int kWarps = kBlock / 32;
constexpr uint32_t kStA = 1u << 30;  // aggregate
constexpr uint32_t kStP = 2u << 30;  // inclusive prefix
constexpr uint32_t kStMask = (1u << 30) - 1;

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K k, int shift) {
  return static_cast<uint32_t>(k >> shift) & 0xFFu;
}

// hist[p*256 + d] += count of keys with digit d at pass p
template <typename K>
__global__ void __launch_bounds__(256) k_hist(const K* __restrict__ keys, uint64_t n, int begin_bit, int passes,
                                              uint32_t* __restrict__ hist) {
  extern __shared__ uint32_t sh[];  // passes * 256
  for (int i = threadIdx.x; i < passes * kBins; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  // all lanes run the same trip count so the warp-level match below is converged
  for (uint64_t b = static_cast<uint64_t>(blockIdx.x) * blockDim.x; b < n; b += stride) {
    const uint64_t i = b + threadIdx.x;
    const bool valid = i < n;
    const K k = valid ? keys[i] : K(0);
    for (int p = 0; p < passes; ++p) {
      const uint32_t d = digit_of(k, begin_bit + p * kRadixBits);
      // warp-aggregate equal digits before the shared atomic (long runs of equal keys)
      const unsigned peers = __match_any_sync(0xffffffffu, valid ? d : 0x100u + lane_id());
      if (valid && lane_id() == static_cast<unsigned>(__ffs(peers) - 1)) atomicAdd(&sh[p * kBins + d], __popc(peers));
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kBins; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// exclusive scan of each pass histogram (one block of 256 threads per pass)
static __global__ void k_hist_offsets(const uint32_t* __restrict__ hist, uint32_t* __restrict__ offs) {
  __shared__ uint32_t s[kBins];
  const int p = blockIdx.x, d = threadIdx.x;
  s[d] = hist[p * kBins + d];
  __syncthreads();
  // Hillis-Steele inclusive scan over 256 values
  for (int o = 1; o < kBins; o <<= 1) {
    uint32_t v = d >= o ? s[d - o] : 0;
    __syncthreads();
    s[d] += v;
    __syncthreads();
  }
  offs[p * kBins + d] = s[d] - hist[p * kBins + d];
}

template <typename K>
struct SmemLayout {
  K keys[kTile];
  uint32_t vals[kTile];
  uint16_t warp_hist[kWarps][kBins];  // per-warp digit counts, then exclusive offsets across warps
  uint32_t tile_count[kBins];
  uint32_t local_off[kBins];
  uint32_t global_base[kBins];
  uint32_t tile;
};

template <typename K>
__global__ void __launch_bounds__(kBlock) k_onesweep(const K* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
                                                      K* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
                                                      uint64_t n, int shift, const uint32_t* __restrict__ digit_offs,
                                                      uint32_t* __restrict__ status, uint32_t* __restrict__ counter) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SmemLayout<K>& S = *reinterpret_cast<SmemLayout<K>*>(smem_raw);
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;

  if (threadIdx.x == 0) S.tile = atomicAdd(counter, 1u);
  for (int i = threadIdx.x; i < kWarps * kBins; i += kBlock) (&S.warp_hist[0][0])[i] = 0;
  __syncthreads();
  const uint32_t tile = S.tile;
  const uint64_t tile_base = static_cast<uint64_t>(tile) * kTile;
  const uint64_t warp_base = tile_base + static_cast<uint64_t>(warp) * (32 * kItems);

  K key[kItems];
  uint32_t val[kItems];
  uint32_t rank[kItems];
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const uint64_t i = warp_base + r * 32 + lane;
    if (i < n) {
      key[r] = keys_in[i];
      val[r] = vals_in[i];
    }
  }
  // ---- stable per-warp ranking
  uint16_t* wh = S.warp_hist[warp];
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const uint64_t i = warp_base + r * 32 + lane;
    const bool valid = i < n;
    const uint32_t d = valid ? digit_of(key[r], shift) : (0x100u + lane);
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    uint32_t base = 0;
    if (valid) base = wh[d];
    __syncwarp();
    if (valid && lane == static_cast<unsigned>(__ffs(peers) - 1)) wh[d] = static_cast<uint16_t>(base + __popc(peers));
    __syncwarp();
    rank[r] = base + __popc(peers & lanemask_lt());
  }
  __syncthreads();
  // ---- per-digit: warp offsets and tile counts
  if (threadIdx.x < kBins) {
    const int d = threadIdx.x;
    uint32_t sum = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = S.warp_hist[w][d];
      S.warp_hist[w][d] = static_cast<uint16_t>(sum);
      sum += c;
    }
    S.tile_count[d] = sum;
    // ---- decoupled look-back per digit
    uint32_t* st = status + static_cast<uint64_t>(tile) * kBins + d;
    uint32_t excl = 0;
    if (tile == 0) {
      st_relaxed_u32(st, kStP | sum);
    } else {
      st_relaxed_u32(st, kStA | sum);
      const uint32_t* pred = st - kBins;
      for (;;) {
        uint32_t s;
        do {
          s = ld_relaxed_u32(pred);
        } while ((s >> 30) == 0);
        excl += s & kStMask;
        if ((s >> 30) == 2) break;
        pred -= kBins;
      }
      st_relaxed_u32(st, kStP | (excl + sum));
    }
    S.global_base[d] = digit_offs[d] + excl;
  }
  __syncthreads();
  // ---- tile-local exclusive scan over digits (8 warps x 32 digits)
  if (threadIdx.x < kBins) {
    const uint32_t c = S.tile_count[threadIdx.x];
    uint32_t inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
      if (static_cast<int>(lane) >= o) inc += u;
    }
    S.local_off[threadIdx.x] = inc - c;  // exclusive within the 32-digit group
    if (lane == 31) S.tile_count[threadIdx.x] = inc;  // group total (only read below as group sums)
  }
  __syncthreads();
  if (threadIdx.x < kBins) {
    const int g = threadIdx.x >> 5;
    uint32_t add = 0;
    for (int h = 0; h < g; ++h) add += S.tile_count[h * 32 + 31];
    __syncwarp();
    S.local_off[threadIdx.x] += add;
  }
  __syncthreads();
  // ---- scatter into shared memory in sorted order
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const uint64_t i = warp_base + r * 32 + lane;
    if (i < n) {
      const uint32_t d = digit_of(key[r], shift);
      const uint32_t pos = S.local_off[d] + S.warp_hist[warp][d] + rank[r];
      S.keys[pos] = key[r];
      S.vals[pos] = val[r];
    }
  }
  __syncthreads();
  // ---- write out: consecutive positions of one digit land contiguously
  const uint32_t valid = static_cast<uint32_t>(n - tile_base < static_cast<uint64_t>(kTile) ? n - tile_base : kTile);
  for (uint32_t p = threadIdx.x; p < valid; p += kBlock) {
    const K k = S.keys[p];
    const uint32_t d = digit_of(k, shift);
    const uint32_t o = S.global_base[d] + (p - S.local_off[d]);
    keys_out[o] = k;
    vals_out[o] = S.vals[p];
  }
}

// Scratch reused across sorts on one context.
struct Scratch {
  DBuf<uint32_t> hist;    // passes*256 counts
  DBuf<uint32_t> offs;    // passes*256 exclusive offsets
  DBuf<uint32_t> status;  // passes * tiles * 256 look-back words + passes counters
  std::vector<uint32_t> host_hist;
};

}  // namespace radix

// Sort n (key, value) pairs on bits [begin_bit, end_bit).  Double-buffered: the result is
// in (keys, vals) when the return value is false, in (keys_alt, vals_alt) when true.
// If `hist_in` is non-null it holds the precomputed per-pass histograms (passes*256).
template <typename K>
bool radix_sort_pairs(Ctx* c, K* keys, uint32_t* vals, K* keys_alt, uint32_t* vals_alt, uint64_t n, int begin_bit,
                      int end_bit, radix::Scratch& s, const uint32_t* hist_in = nullptr, const char* tag = "radix") {
  using namespace radix;
  if (n <= 1 || end_bit <= begin_bit) return false;
  const int passes = (end_bit - begin_bit + kRadixBits - 1) / kRadixBits;
  const uint64_t tiles = (n + kTile - 1) / kTile;
  if (s.hist.n < static_cast<size_t>(passes) * kBins) {
    s.hist.alloc(c, static_cast<size_t>(passes) * kBins);
    s.offs.alloc(c, static_cast<size_t>(passes) * kBins);
  }
  const uint32_t* hist = hist_in;
  if (!hist) {
    ITT_CUDA(cudaMemsetAsync(s.hist.p, 0, static_cast<size_t>(passes) * kBins * 4, c->stream));
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(c->sm_count) * 8));
    launch(c, "radix_hist", static_cast<double>(n) * sizeof(K), k_hist<K>, dim3(grid), dim3(256),
           static_cast<size_t>(passes) * kBins * 4, keys, n, begin_bit, passes, s.hist.p);
    hist = s.hist.p;
  }
  launch(c, "radix_offsets", 0.0, k_hist_offsets, dim3(passes), dim3(kBins), 0, hist, s.offs.p);
  // skip passes whose digit is constant (one bin holds all n keys)
  s.host_hist.resize(static_cast<size_t>(passes) * kBins);
  readback(c, s.host_hist.data(), hist, s.host_hist.size());
  std::vector<int> live;
  for (int p = 0; p < passes; ++p) {
    bool trivial = false;
    for (int d = 0; d < kBins; ++d)
      if (s.host_hist[static_cast<size_t>(p) * kBins + d] == n) trivial = true;
    if (!trivial) live.push_back(p);
  }
  if (live.empty()) return false;
  const size_t per_pass = tiles * kBins + 1;
  if (s.status.n < per_pass * live.size()) s.status.alloc(c, per_pass * live.size());
  ITT_CUDA(cudaMemsetAsync(s.status.p, 0, per_pass * live.size() * 4, c->stream));
  const size_t smem = sizeof(SmemLayout<K>);
  static bool attr_set = false;
  if (!attr_set) {
    ITT_CUDA(cudaFuncSetAttribute(k_onesweep<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    attr_set = true;
  }
  bool alt = false;
  for (size_t q = 0; q < live.size(); ++q) {
    const int p = live[q];
    uint32_t* st = s.status.p + q * per_pass;
    const K* ki = alt ? keys_alt : keys;
    const uint32_t* vi = alt ? vals_alt : vals;
    K* ko = alt ? keys : keys_alt;
    uint32_t* vo = alt ? vals : vals_alt;
    launch(c, "radix_onesweep", static_cast<double>(n) * 2.0 * (sizeof(K) + 4), k_onesweep<K>,
           dim3(static_cast<unsigned>(tiles)), dim3(kBlock), smem, ki, vi, ko, vo, n, begin_bit + p * kRadixBits,
           s.offs.p + p * kBins, st + 1, st);
    alt = !alt;
  }
  (void)tag;
  return alt;
}

}  // namespace itt
