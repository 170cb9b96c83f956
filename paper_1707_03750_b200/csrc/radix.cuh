// radix.cuh — hand-written onesweep LSD radix sort of (key, u32 value) pairs, sm_100a.
//
// Per sort: the 256-bin histograms of every 8-bit digit come from one upfront pass (or from
// the producer kernel, e.g. the SA rank update), and each digit pass is ONE kernel:
//   1. a tile of BLOCK*ITEMS pairs is loaded warp-striped (coalesced) — or produced on the fly
//      by a Loader (the SA emission gathers rank[SA[j]-h] inside the first pass);
//   2. each warp ranks its 32*ITEMS keys with __match_any_sync (stable: warp-major, then
//      round, then lane), leaving per-warp digit counts in shared memory;
//   3. one thread per digit publishes the tile's count (flag A) at once, the tile is re-ordered
//      by digit in shared memory, and only then does each digit thread run its decoupled
//      look-back, so predecessors have had the whole scatter phase to publish;
//   4. the tile is written out from shared memory: consecutive positions of one digit go to
//      consecutive global addresses.
// Algorithmic traffic per pass: n * 2 * (sizeof(K) + 4) bytes.
#pragma once
#include "common.cuh"

namespace itt {
namespace radix {

constexpr int kRadixBits = 8;
constexpr int kBins = 256;
constexpr uint32_t kStA = 1u << 30;  // aggregate
constexpr uint32_t kStP = 2u << 30;  // inclusive prefix
constexpr uint32_t kStMask = (1u << 30) - 1;
constexpr int kLook = 4;  // look-back window per step (A/B on C2: 1 -> 1.27 ms, 4 and 8 -> 1.16 ms of passes per step)

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K k, int shift) {
  return static_cast<uint32_t>(k >> shift) & 0xFFu;
}

// plain arrays
template <typename K>
struct ArrayLoader {
  const K* keys;
  const uint32_t* vals;
  __device__ __forceinline__ void operator()(uint64_t i, K& k, uint32_t& v) const {
    k = __ldcs(&keys[i]);  // streaming: evict-first, keeps L2 for the random-access arrays
    v = __ldcs(&vals[i]);
  }
  // bulk (TMA) staging: the tile's keys and values are copied to shared memory as they are
  static constexpr bool kBulkKeys = true;
  __host__ __device__ const K* bulk_keys() const { return keys; }
  __host__ __device__ const uint32_t* bulk_vals() const { return vals; }
  __device__ __forceinline__ void fix(uint64_t, K&, uint32_t&) const {}
};

// Lanes of the warp holding the same 8-bit digit (valid lanes only among themselves): ballots
// instead of MATCH.ANY, whose long MIO latency dominated the ranking loop on sm_100a.  Only the
// digit bits that vary across the warp need a ballot (two warp reductions find them): the keys of
// periodic traces (dense group ids in SA order) are mostly equal within a warp, so most rounds
// take no ballot at all; all 8 bits varying takes the unrolled path.
__device__ __forceinline__ unsigned digit_peers(uint32_t d, bool valid) {
  const unsigned vm = __ballot_sync(0xffffffffu, valid);
  unsigned peers = valid ? vm : ~vm;
  const unsigned vary = (__reduce_or_sync(0xffffffffu, d) ^ __reduce_and_sync(0xffffffffu, d)) & 0xFFu;
  if (vary == 0xFFu) {
#pragma unroll
    for (int b = 0; b < kRadixBits; ++b) {
      const bool bit = (d >> b) & 1u;
      const unsigned m = __ballot_sync(0xffffffffu, bit);
      peers &= bit ? m : ~m;
    }
  } else {
    for (unsigned v = vary; v; v &= v - 1) {
      const bool bit = (d >> (__ffs(v) - 1)) & 1u;
      const unsigned m = __ballot_sync(0xffffffffu, bit);
      peers &= bit ? m : ~m;
    }
  }
  return peers;
}

// hist[p*256 + d] += count of keys with digit d at pass p.  Each thread walks a contiguous run of
// keys and issues one shared atomic per run of equal digits (skewed / structured keys are cheap).
template <typename K>
__global__ void __launch_bounds__(256) k_hist(const K* __restrict__ keys, uint64_t n, int begin_bit, int passes,
                                              uint32_t* __restrict__ hist) {
  extern __shared__ uint32_t sh[];  // passes * 256
  for (int i = threadIdx.x; i < passes * kBins; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  constexpr int kPer = 16;
  const uint64_t chunks = (n + kPer - 1) / kPer;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t ch = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; ch < chunks; ch += stride) {
    const uint64_t i0 = ch * kPer;
    const int cnt = static_cast<int>(n - i0 < kPer ? n - i0 : kPer);
    K kk[kPer];
#pragma unroll
    for (int q = 0; q < kPer; ++q) kk[q] = q < cnt ? keys[i0 + q] : K(0);
    for (int p = 0; p < passes; ++p) {
      const int sh_bits = begin_bit + p * kRadixBits;
      uint32_t cur = digit_of(kk[0], sh_bits), len = 0;
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        if (q >= cnt) break;
        const uint32_t d = digit_of(kk[q], sh_bits);
        if (d != cur) {
          atomicAdd(&sh[p * kBins + cur], len);
          cur = d;
          len = 0;
        }
        ++len;
      }
      if (len) atomicAdd(&sh[p * kBins + cur], len);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kBins; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

template <typename K, int BLOCK, int ITEMS>
struct SmemLayout {
  static constexpr int kTile = BLOCK * ITEMS;
  static constexpr int kWarps = BLOCK / 32;
  K keys[kTile];
  uint32_t vals[kTile];
  uint16_t warp_hist[kWarps][kBins];  // per-warp digit counts, then exclusive offsets across warps
  uint32_t tile_count[kBins];
  uint32_t local_off[kBins];
  uint32_t global_base[kBins];
  uint32_t digit_off[kBins];
  uint32_t group_sum[8];
  uint32_t hgroup_sum[8];
  uint32_t tile;
};

template <typename K, int BLOCK, int ITEMS, typename Loader, int MINB>
__global__ void __launch_bounds__(BLOCK, MINB) k_onesweep(Loader ld, K* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
                                                    uint64_t n, int shift, const uint32_t* __restrict__ digit_hist,
                                                    uint32_t* __restrict__ status, uint32_t* __restrict__ counter) {
  static_assert(BLOCK >= kBins, "one thread per digit");
  using S_t = SmemLayout<K, BLOCK, ITEMS>;
  constexpr int kTile = S_t::kTile;
  constexpr int kWarps = S_t::kWarps;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S_t& S = *reinterpret_cast<S_t*>(smem_raw);
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t hv = threadIdx.x < kBins ? __ldg(&digit_hist[threadIdx.x]) : 0u;  // this pass's digit counts

  if (threadIdx.x == 0) S.tile = atomicAdd(counter, 1u);
  for (int i = threadIdx.x; i < kWarps * kBins; i += BLOCK) (&S.warp_hist[0][0])[i] = 0;
  __syncthreads();
  const uint32_t tile = S.tile;
  const uint64_t tile_base = static_cast<uint64_t>(tile) * kTile;
  const uint64_t warp_base = tile_base + static_cast<uint64_t>(warp) * (32 * ITEMS);

  K key[ITEMS];
  uint32_t val[ITEMS];
  uint32_t rank[ITEMS];
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    const uint64_t i = warp_base + r * 32 + lane;
    if (i < n) ld(i, key[r], val[r]);
  }
  // ---- stable per-warp ranking
  uint16_t* wh = S.warp_hist[warp];
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    const uint64_t i = warp_base + r * 32 + lane;
    const bool valid = i < n;
    const uint32_t d = valid ? digit_of(key[r], shift) : 0u;
    const unsigned peers = digit_peers(d, valid);
    uint32_t base = 0;
    if (valid) base = wh[d];
    __syncwarp();
    if (valid && lane == static_cast<unsigned>(__ffs(peers) - 1)) wh[d] = static_cast<uint16_t>(base + __popc(peers));
    __syncwarp();
    rank[r] = base + __popc(peers & lanemask_lt());
  }
  __syncthreads();
  // ---- per digit: warp offsets, tile count, early publication of the aggregate
  uint32_t my_count = 0;
  if (threadIdx.x < kBins) {
    const int d = threadIdx.x;
    uint32_t sum = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = S.warp_hist[w][d];
      S.warp_hist[w][d] = static_cast<uint16_t>(sum);
      sum += c;
    }
    my_count = sum;
    st_relaxed_u32(status + static_cast<uint64_t>(tile) * kBins + d, (tile == 0 ? kStP : kStA) | sum);
    // exclusive scan over the 256 digits: 8 groups of 32 lanes
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
      if (static_cast<int>(lane) >= o) inc += u;
    }
    S.local_off[d] = inc - sum;
    if (lane == 31) S.group_sum[d >> 5] = inc;
    // this pass's global digit offsets: exclusive scan of the histogram (no separate launch)
    uint32_t hinc = hv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, hinc, o);
      if (static_cast<int>(lane) >= o) hinc += u;
    }
    S.digit_off[d] = hinc - hv;
    if (lane == 31) S.hgroup_sum[d >> 5] = hinc;
  }
  __syncthreads();
  if (threadIdx.x < kBins) {
    uint32_t add = 0, hadd = 0;
    const int g = threadIdx.x >> 5;
    for (int h = 0; h < g; ++h) add += S.group_sum[h], hadd += S.hgroup_sum[h];
    S.local_off[threadIdx.x] += add;
    S.digit_off[threadIdx.x] += hadd;
  }
  __syncthreads();
  // ---- scatter into shared memory in digit order
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    const uint64_t i = warp_base + r * 32 + lane;
    if (i < n) {
      const uint32_t d = digit_of(key[r], shift);
      const uint32_t pos = S.local_off[d] + S.warp_hist[warp][d] + rank[r];
      S.keys[pos] = key[r];
      S.vals[pos] = val[r];
    }
  }
  // ---- decoupled look-back per digit (predecessors had the whole scatter to publish)
  if (threadIdx.x < kBins) {
    const int d = threadIdx.x;
    uint32_t excl = 0;
    if (tile > 0) {
      // walk back kLook predecessors per step (their status words load in parallel): the
      // first tiles of a wave otherwise pay one L2 round trip per predecessor
      int64_t t = static_cast<int64_t>(tile) - 1;
      for (bool done = false; !done; t -= kLook) {
        uint32_t sv[kLook];
#pragma unroll
        for (int u = 0; u < kLook; ++u) sv[u] = t - u >= 0 ? ld_relaxed_u32(status + static_cast<uint64_t>(t - u) * kBins + d) : 0u;
#pragma unroll
        for (int u = 0; u < kLook; ++u) {
          if (done) break;
          uint32_t v = sv[u];
          while ((v >> 30) == 0) v = ld_relaxed_u32(status + static_cast<uint64_t>(t - u) * kBins + d);
          excl += v & kStMask;
          done = (v >> 30) == 2;
        }
      }
      st_relaxed_u32(status + static_cast<uint64_t>(tile) * kBins + d, kStP | (excl + my_count));
    }
    S.global_base[d] = S.digit_off[d] + excl;
  }
  __syncthreads();
  // ---- write out
  const uint32_t valid = static_cast<uint32_t>(n - tile_base < static_cast<uint64_t>(kTile) ? n - tile_base : kTile);
  for (uint32_t p = threadIdx.x; p < valid; p += BLOCK) {
    const K k = S.keys[p];
    const uint32_t d = digit_of(k, shift);
    const uint32_t o = S.global_base[d] + (p - S.local_off[d]);
    __stcs(&keys_out[o], k);
    __stcs(&vals_out[o], S.vals[p]);
  }
}


// ---------------------------------------------------------------- persistent, TMA-staged pass
// Same pass as k_onesweep, restructured so HBM latency leaves the per-tile critical path:
//  * persistent CTAs (grid = resident capacity) claim tiles in order from the counter;
//  * while tile t is ranked / scattered / looked back / written, the NEXT tile's keys and values
//    are already streaming into the other half of a double-buffered shared-memory stage by
//    cp.async.bulk (the TMA bulk-copy engine; one thread issues it, completion on an mbarrier),
//    so no register file is spent holding loads in flight;
//  * ranks are computed from the staged tile (LDS, conflict-free) and the scatter re-reads it, so
//    only the 8 ranks live in registers across the block barriers.
// Progress: every claimed tile publishes its aggregate right after ranking, before it waits on
// anything; a CTA's prefetched tile is always larger than the tile it is processing, so the
// smallest unpublished tile is always a CTA's current tile and never waits (no deadlock).
// Partial last tile (bulk sizes must be 16-B multiples): plain cooperative loads.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <typename K, int BLOCK, int ITEMS>
struct TmaLayout {
  static constexpr int kTile = BLOCK * ITEMS;
  static constexpr int kWarps = BLOCK / 32;
  K in_keys[2][kTile];
  uint32_t in_vals[2][kTile];
  K out_keys[kTile];
  uint32_t out_vals[kTile];
  uint16_t warp_hist[kWarps][kBins];
  uint32_t local_off[kBins];
  uint32_t global_base[kBins];
  uint32_t digit_off[kBins];
  uint32_t group_sum[8];
  uint32_t hgroup_sum[8];
  uint64_t bar[2];
  uint32_t tile[2];
};

template <typename K, int BLOCK, int ITEMS, typename Loader>
__global__ void __launch_bounds__(BLOCK) k_onesweep_tma(Loader ld, K* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
                                                        uint64_t n, int shift, const uint32_t* __restrict__ digit_hist,
                                                        uint32_t* __restrict__ status, uint32_t* __restrict__ counter) {
  static_assert(BLOCK >= kBins, "one thread per digit");
  static_assert(ITEMS <= 16, "16-bit ranks");
  using S_t = TmaLayout<K, BLOCK, ITEMS>;
  constexpr int kTile = S_t::kTile;
  constexpr int kWarps = S_t::kWarps;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  S_t& S = *reinterpret_cast<S_t*>(smem_raw);
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t hv = threadIdx.x < kBins ? __ldg(&digit_hist[threadIdx.x]) : 0u;  // this pass's digit counts
  const uint64_t tiles = (n + kTile - 1) / kTile;
  const uint64_t full_tiles = n / kTile;

  auto issue = [&](uint32_t t, int b) {  // thread 0: stage full tile t into buffer b
    fence_proxy_async_smem();
    const uint64_t base = static_cast<uint64_t>(t) * kTile;
    const uint32_t vb = kTile * 4;
    if constexpr (Loader::kBulkKeys) {
      mbar_expect_tx(&S.bar[b], vb + kTile * sizeof(K));
      bulk_g2s(S.in_keys[b], ld.bulk_keys() + base, kTile * sizeof(K), &S.bar[b]);
    } else {
      mbar_expect_tx(&S.bar[b], vb);
    }
    bulk_g2s(S.in_vals[b], ld.bulk_vals() + base, vb, &S.bar[b]);
  };
  if (threadIdx.x == 0) {
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t t0 = atomicAdd(counter, 1u);
    S.tile[0] = t0;
    if (t0 < full_tiles) issue(t0, 0);
  }
  __syncthreads();
  uint32_t parity = 0;  // bit b: phase of bar[b]
  int cur = 0;
  for (;;) {
    const uint32_t tile = S.tile[cur];
    if (tile >= tiles) break;
    if (threadIdx.x == 0) {  // claim and prefetch the next tile into the other buffer
      const uint32_t tn = atomicAdd(counter, 1u);
      S.tile[cur ^ 1] = tn;
      if (tn < full_tiles) issue(tn, cur ^ 1);
    }
    {
      uint4* wh4 = reinterpret_cast<uint4*>(&S.warp_hist[0][0]);
      for (int i = threadIdx.x; i < kWarps * kBins * 2 / 16; i += BLOCK) wh4[i] = make_uint4(0, 0, 0, 0);
    }
    const uint64_t tile_base = static_cast<uint64_t>(tile) * kTile;
    const uint32_t valid = static_cast<uint32_t>(umin64(n - tile_base, kTile));
    K* ik = S.in_keys[cur];
    uint32_t* iv = S.in_vals[cur];
    if (tile < full_tiles) {
      mbar_wait(&S.bar[cur], (parity >> cur) & 1u);
      parity ^= 1u << cur;
    } else {
      for (uint32_t p = threadIdx.x; p < valid; p += BLOCK) ld(tile_base + p, ik[p], iv[p]);
    }
    __syncthreads();
    // ---- stable per-warp ranking over the staged tile (warp-striped)
    const uint32_t wbase = warp * (32 * ITEMS);
    uint16_t* wh = S.warp_hist[warp];
    uint32_t rank[ITEMS];
#pragma unroll
    for (int r = 0; r < ITEMS; ++r) {
      const uint32_t idx = wbase + r * 32 + lane;
      const bool ok = idx < valid;
      K k = K(0);
      if (ok) {
        k = ik[idx];
        if constexpr (!Loader::kBulkKeys) {
          if (tile < full_tiles) {
            uint32_t v = iv[idx];
            ld.fix(tile_base + idx, k, v);
            ik[idx] = k;
            iv[idx] = v;
          }
        }
      }
      const uint32_t d = ok ? digit_of(k, shift) : 0u;
      const unsigned peers = digit_peers(d, ok);
      uint32_t base = 0;
      if (ok) base = wh[d];
      __syncwarp();
      if (ok && lane == static_cast<unsigned>(__ffs(peers) - 1)) wh[d] = static_cast<uint16_t>(base + __popc(peers));
      __syncwarp();
      rank[r] = base + __popc(peers & lanemask_lt());
    }
    __syncthreads();
    uint32_t my_count = 0;
    if (threadIdx.x < kBins) {
      const int d = threadIdx.x;
      uint32_t sum = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        const uint32_t c = S.warp_hist[w][d];
        S.warp_hist[w][d] = static_cast<uint16_t>(sum);
        sum += c;
      }
      my_count = sum;
      st_relaxed_u32(status + static_cast<uint64_t>(tile) * kBins + d, (tile == 0 ? kStP : kStA) | sum);
      uint32_t inc = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
        if (static_cast<int>(lane) >= o) inc += u;
      }
      S.local_off[d] = inc - sum;
      if (lane == 31) S.group_sum[d >> 5] = inc;
      // this pass's global digit offsets: exclusive scan of the histogram (no separate launch)
      uint32_t hinc = hv;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, hinc, o);
        if (static_cast<int>(lane) >= o) hinc += u;
      }
      S.digit_off[d] = hinc - hv;
      if (lane == 31) S.hgroup_sum[d >> 5] = hinc;
    }
    __syncthreads();
    if (threadIdx.x < kBins) {
      uint32_t add = 0, hadd = 0;
      const int g = threadIdx.x >> 5;
      for (int h = 0; h < g; ++h) add += S.group_sum[h], hadd += S.hgroup_sum[h];
      S.local_off[threadIdx.x] += add;
      S.digit_off[threadIdx.x] += hadd;
    }
    __syncthreads();
    // ---- scatter the staged tile into digit order
#pragma unroll
    for (int r = 0; r < ITEMS; ++r) {
      const uint32_t idx = wbase + r * 32 + lane;
      if (idx < valid) {
        const K k = ik[idx];
        const uint32_t d = digit_of(k, shift);
        const uint32_t pos = S.local_off[d] + S.warp_hist[warp][d] + rank[r];
        S.out_keys[pos] = k;
        S.out_vals[pos] = iv[idx];
      }
    }
    if (threadIdx.x < kBins) {
      const int d = threadIdx.x;
      uint32_t excl = 0;
      if (tile > 0) {
        int64_t t = static_cast<int64_t>(tile) - 1;
        for (bool done = false; !done; t -= kLook) {
          uint32_t sv[kLook];
#pragma unroll
          for (int u = 0; u < kLook; ++u) sv[u] = t - u >= 0 ? ld_relaxed_u32(status + static_cast<uint64_t>(t - u) * kBins + d) : 0u;
#pragma unroll
          for (int u = 0; u < kLook; ++u) {
            if (done) break;
            uint32_t v = sv[u];
            while ((v >> 30) == 0) v = ld_relaxed_u32(status + static_cast<uint64_t>(t - u) * kBins + d);
            excl += v & kStMask;
            done = (v >> 30) == 2;
          }
        }
        st_relaxed_u32(status + static_cast<uint64_t>(tile) * kBins + d, kStP | (excl + my_count));
      }
      S.global_base[d] = S.digit_off[d] + excl;
    }
    __syncthreads();
    for (uint32_t p = threadIdx.x; p < valid; p += BLOCK) {
      const K k = S.out_keys[p];
      const uint32_t d = digit_of(k, shift);
      const uint32_t o = S.global_base[d] + (p - S.local_off[d]);
      __stcs(&keys_out[o], k);
      __stcs(&vals_out[o], S.out_vals[p]);
    }
    __syncthreads();
    cur ^= 1;
  }
}

template <typename K, int BLOCK, int ITEMS, typename Loader>
void launch_pass_tma(Ctx* c, const Loader& ld, K* ko, uint32_t* vo, uint64_t n, int shift, const uint32_t* dhist, uint32_t* st) {
  constexpr int TILE = BLOCK * ITEMS;
  const size_t smem = sizeof(TmaLayout<K, BLOCK, ITEMS>);
  auto kern = k_onesweep_tma<K, BLOCK, ITEMS, Loader>;
  smem_optin(c, kern, smem);
  static int per_sm[64] = {0};  // resident CTAs per SM, per device
  int& occ = per_sm[c->device & 63];
  if (occ == 0) {
    ITT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, BLOCK, smem));
    if (occ < 1) occ = 1;
  }
  const uint64_t tiles = (n + TILE - 1) / TILE;
  const uint64_t grid = std::min<uint64_t>(tiles, static_cast<uint64_t>(c->sm_count) * occ);
  launch(c, "radix_onesweep", static_cast<double>(n) * 2.0 * (sizeof(K) + 4), kern, dim3(static_cast<unsigned>(grid)), dim3(BLOCK),
         smem, ld, ko, vo, n, shift, dhist, st + 1, st);
}

// Scratch reused across sorts on one context.
struct Scratch {
  DBuf<uint32_t> hist;    // passes*256 counts
  DBuf<uint32_t> status;  // passes * (tiles * 256 look-back words + counter)
  std::vector<uint32_t> host_hist;
};

// tile shapes (BLOCK, ITEMS); selected at runtime (ITT_RADIX_CFG) for tuning sweeps
constexpr int kCfgBlock[] = {512, 256, 384, 256, 512, 512, 512, 256, 256, 256, 512, 256, 256};
constexpr int kCfgItems[] = {8, 16, 12, 8, 16, 8, 8, 8, 16, 12, 8, 8, 16};
int config_index();

template <typename K, int BLOCK, int ITEMS, typename Loader, int MINB = 1024 / BLOCK>
void launch_pass(Ctx* c, const Loader& ld, K* ko, uint32_t* vo, uint64_t n, int shift, const uint32_t* dhist,
                 uint32_t* st, bool first_use) {
  constexpr int TILE = BLOCK * ITEMS;
  const size_t smem = sizeof(SmemLayout<K, BLOCK, ITEMS>);
  (void)first_use;
  smem_optin(c, k_onesweep<K, BLOCK, ITEMS, Loader, MINB>, smem);
  const uint64_t tiles = (n + TILE - 1) / TILE;
  launch(c, "radix_onesweep", static_cast<double>(n) * 2.0 * (sizeof(K) + 4), k_onesweep<K, BLOCK, ITEMS, Loader, MINB>,
         dim3(static_cast<unsigned>(tiles)), dim3(BLOCK), smem, ld, ko, vo, n, shift, dhist, st + 1, st);
}

template <typename K, typename Loader>
void dispatch_pass(Ctx* c, int cfg, const Loader& ld, K* ko, uint32_t* vo, uint64_t n, int shift, const uint32_t* dhist,
                   uint32_t* st) {
  static bool seen[16] = {false};
  const bool first = !seen[cfg];
  seen[cfg] = true;
  if (cfg >= 10) {  // bulk copies need 16-byte aligned sources
    const uintptr_t a = reinterpret_cast<uintptr_t>(ld.bulk_vals()) | reinterpret_cast<uintptr_t>(ld.bulk_keys());
    if (a & 15u) fail(ITT_E_INVALID_ARGUMENT, "internal: radix staging needs 16-byte aligned arrays");
  }
  switch (cfg) {
    case 1: launch_pass<K, 256, 16>(c, ld, ko, vo, n, shift, dhist, st, first); break;
    case 2: launch_pass<K, 384, 12>(c, ld, ko, vo, n, shift, dhist, st, first); break;
    case 3: launch_pass<K, 256, 8>(c, ld, ko, vo, n, shift, dhist, st, first); break;
    case 4: launch_pass<K, 512, 16>(c, ld, ko, vo, n, shift, dhist, st, first); break;
    case 5: launch_pass<K, 512, 8, Loader, 3>(c, ld, ko, vo, n, shift, dhist, st, first); break;
    case 6: launch_pass<K, 512, 8, Loader, 4>(c, ld, ko, vo, n, shift, dhist, st, first); break;
    case 7: launch_pass<K, 256, 8, Loader, 6>(c, ld, ko, vo, n, shift, dhist, st, first); break;
    case 8: launch_pass<K, 256, 16, Loader, 4>(c, ld, ko, vo, n, shift, dhist, st, first); break;
    case 9: launch_pass<K, 256, 12, Loader, 5>(c, ld, ko, vo, n, shift, dhist, st, first); break;
    case 10: launch_pass_tma<K, 512, 8>(c, ld, ko, vo, n, shift, dhist, st); break;
    case 11: launch_pass_tma<K, 256, 8>(c, ld, ko, vo, n, shift, dhist, st); break;
    case 12: launch_pass_tma<K, 256, 16>(c, ld, ko, vo, n, shift, dhist, st); break;
    default: launch_pass<K, 512, 8>(c, ld, ko, vo, n, shift, dhist, st, first); break;
  }
}

inline uint64_t tile_of(int cfg) { return static_cast<uint64_t>(kCfgBlock[cfg]) * kCfgItems[cfg]; }

}  // namespace radix

// Sort n (key, value) pairs on bits [begin_bit, end_bit).  Double-buffered: the result is
// in (keys, vals) when the return value is false, in (keys_alt, vals_alt) when true.
//  * hist_in: precomputed per-pass histograms (passes*256) — skips the histogram kernel;
//  * first_loader: produces the first pass's input instead of reading (keys, vals);
//  * skip_trivial: read the histograms back and drop passes whose digit is constant.
// Zero the look-back words of a later sort of n keys with up to `passes` passes now (e.g. while the
// host waits on a readback anyway), so that sort can pass status_zeroed = true.
inline void radix_prezero_status(Ctx* c, radix::Scratch& s, uint64_t n, int passes) {
  const int cfg = radix::config_index();
  const uint64_t tiles = (n + radix::tile_of(cfg) - 1) / radix::tile_of(cfg);
  const size_t need = (tiles * radix::kBins + 1) * static_cast<size_t>(passes);
  if (s.status.n < need) s.status.alloc(c, need);
  ITT_CUDA(cudaMemsetAsync(s.status.p, 0, need * 4, c->stream));
}

template <typename K, typename FirstLoader = radix::ArrayLoader<K>>
bool radix_sort_pairs(Ctx* c, K* keys, uint32_t* vals, K* keys_alt, uint32_t* vals_alt, uint64_t n, int begin_bit,
                      int end_bit, radix::Scratch& s, const uint32_t* hist_in = nullptr,
                      const FirstLoader* first_loader = nullptr, bool skip_trivial = true,
                      bool status_zeroed = false) {
  using namespace radix;
  if (end_bit <= begin_bit) end_bit = begin_bit + 1;
  const int passes = (end_bit - begin_bit + kRadixBits - 1) / kRadixBits;
  const int cfg = config_index();
  const uint64_t tiles = (n + tile_of(cfg) - 1) / tile_of(cfg);
  if (n == 0) return false;
  if (s.hist.n < static_cast<size_t>(passes) * kBins) {
    s.hist.alloc(c, static_cast<size_t>(passes) * kBins);
  }
  const uint32_t* hist = hist_in;
  if (!hist) {
    if (first_loader) fail(ITT_E_INVALID_ARGUMENT, "internal: a first-pass loader needs precomputed histograms");
    ITT_CUDA(cudaMemsetAsync(s.hist.p, 0, static_cast<size_t>(passes) * kBins * 4, c->stream));
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(c->sm_count) * 8));
    launch(c, "radix_hist", static_cast<double>(n) * sizeof(K), k_hist<K>, dim3(grid), dim3(256),
           static_cast<size_t>(passes) * kBins * 4, keys, n, begin_bit, passes, s.hist.p);
    hist = s.hist.p;
  }
  std::vector<int> live;
  if (skip_trivial) {
    s.host_hist.resize(static_cast<size_t>(passes) * kBins);
    readback(c, s.host_hist.data(), hist, s.host_hist.size());
    for (int p = 0; p < passes; ++p) {
      bool trivial = false;
      for (int d = 0; d < kBins; ++d)
        if (s.host_hist[static_cast<size_t>(p) * kBins + d] == n) trivial = true;
      if (!trivial) live.push_back(p);
    }
  } else {
    for (int p = 0; p < passes; ++p) live.push_back(p);
  }
  if (first_loader && (live.empty() || live[0] != 0)) live.insert(live.begin(), 0);  // the loader must run
  if (live.empty()) return false;
  const size_t per_pass = tiles * kBins + 1;
  if (status_zeroed) {  // the caller zeroed the look-back words ahead of time (prezero_status)
    if (s.status.n < per_pass * live.size()) fail(ITT_E_INVALID_ARGUMENT, "internal: radix status not prepared");
  } else {
    if (s.status.n < per_pass * live.size()) s.status.alloc(c, per_pass * live.size());
    ITT_CUDA(cudaMemsetAsync(s.status.p, 0, per_pass * live.size() * 4, c->stream));
  }
  bool alt = false;
  for (size_t q = 0; q < live.size(); ++q) {
    const int p = live[q];
    uint32_t* st = s.status.p + q * per_pass;
    K* ko = alt ? keys : keys_alt;
    uint32_t* vo = alt ? vals : vals_alt;
    if (q == 0 && first_loader) {
      dispatch_pass<K>(c, cfg, *first_loader, ko, vo, n, begin_bit + p * kRadixBits, hist + p * kBins, st);
    } else {
      const ArrayLoader<K> ld{alt ? keys_alt : keys, alt ? vals_alt : vals};
      dispatch_pass<K>(c, cfg, ld, ko, vo, n, begin_bit + p * kRadixBits, hist + p * kBins, st);
    }
    alt = !alt;
  }
  return alt;
}

}  // namespace itt
