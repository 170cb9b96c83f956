// radix.cuh — hand-written onesweep LSD radix sort of (key, u32 value) pairs, sm_100a.
//
// Per sort: the histograms of every digit come from one upfront pass (or from the producer
// kernel, e.g. the SA rank update), and each digit pass is ONE kernel:
//   1. a tile of BLOCK*ITEMS pairs is loaded warp-striped (coalesced) — or produced on the fly
//      by a Loader (the SA emission gathers rank[SA[j]-h] inside the first pass);
//   2. each warp ranks its 32*ITEMS keys by ballots over the digit bits that vary in the warp
//      (stable: warp-major, then round, then lane), leaving per-warp digit counts in shared memory;
//   3. the tile's per-digit counts are published at once (flag A), the tile is re-ordered by
//      digit in shared memory, and only then do the digit owners run their decoupled look-back,
//      so predecessors have had the whole scatter phase to publish;
//   4. the tile is written out from shared memory: consecutive positions of one digit go to
//      consecutive global addresses.
// Digits are RB bits wide: 8 (256 bins) by default; 10 (1024 bins, two digits per thread) when it
// saves a pass — a b-bit key takes ceil(b/RB) passes, so e.g. the 9-bit group ids of a periodic
// trace take one 10-bit pass instead of two 8-bit ones.
// Algorithmic traffic per pass: n * 2 * (sizeof(K) + 4) bytes.
#pragma once
#include "common.cuh"

namespace itt {
namespace radix {

constexpr int kRadixBits = 8;  // the default digit width (k_hist, generic sorts)
constexpr int kBins = 256;
constexpr int kWideBits = 10;  // the wide digit of the SA rounds
// Look-back status words: 2 flag bits (aggregate / inclusive prefix) above the per-digit count.
// 32-bit words hold counts below 2^30; sorts of 2^30 or more keys (one digit can then hold 2^30+
// keys) use 64-bit words (radix_sort_pairs picks them by n).
template <typename SW>
struct Status {
  static constexpr int kShift = static_cast<int>(sizeof(SW)) * 8 - 2;
  static constexpr SW kA = SW(1) << kShift;  // aggregate
  static constexpr SW kP = SW(2) << kShift;  // inclusive prefix
  static constexpr SW kMask = kA - 1;
  __device__ __forceinline__ static SW load(const SW* p) {
    if constexpr (sizeof(SW) == 8) return ld_relaxed_u64(p);
    else return ld_relaxed_u32(p);
  }
  __device__ __forceinline__ static void store(SW* p, SW v) {
    if constexpr (sizeof(SW) == 8) st_relaxed_u64(p, v);
    else st_relaxed_u32(p, v);
  }
};
constexpr uint64_t kWideStatusN = 1ull << 30;  // sorts of at least this many keys use 64-bit words
constexpr int kLook = 4;  // look-back window per step (A/B on C2: 1 -> 1.27 ms, 4 and 8 -> 1.16 ms of passes per step)

template <int RB, typename K>
__device__ __forceinline__ uint32_t digit_of(K k, int shift) {
  return static_cast<uint32_t>(k >> shift) & ((1u << RB) - 1u);
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
  __device__ __forceinline__ void prefetch(uint64_t i, uint64_t cnt) const {
    prefetch_l2(keys + i, cnt * sizeof(K));
    prefetch_l2(vals + i, cnt * 4);
  }
};

// keys from an array, values = their positions (the first pass of a sort whose values are 0..n-1:
// no value array to write beforehand or read here)
template <typename K>
struct IotaLoader {
  const K* keys;
  __device__ __forceinline__ void operator()(uint64_t i, K& k, uint32_t& v) const {
    k = __ldcs(&keys[i]);
    v = static_cast<uint32_t>(i);
  }
  __device__ __forceinline__ void prefetch(uint64_t i, uint64_t cnt) const { prefetch_l2(keys + i, cnt * sizeof(K)); }
};

// Lanes of the warp holding the same RB-bit digit (valid lanes only among themselves): ballots
// instead of MATCH.ANY, whose long MIO latency dominated the ranking loop on sm_100a.  Only the
// digit bits that vary across the warp need a ballot (two warp reductions find them): the keys of
// periodic traces (dense group ids in SA order) are mostly equal within a warp, so most rounds
// take no ballot at all; all bits varying takes the unrolled path.
template <int RB>
__device__ __forceinline__ unsigned digit_peers(uint32_t d, bool valid) {
  constexpr unsigned kAll = (1u << RB) - 1u;
  const unsigned vm = __ballot_sync(0xffffffffu, valid);
  unsigned peers = valid ? vm : ~vm;
  const unsigned vary = (__reduce_or_sync(0xffffffffu, d) ^ __reduce_and_sync(0xffffffffu, d)) & kAll;
  if (vary == kAll) {
#pragma unroll
    for (int b = 0; b < RB; ++b) {
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

// hist[p*2^RB + d] += count of keys with RB-bit digit d at pass p.  Each thread walks a contiguous
// run of keys and issues one shared atomic per run of equal digits (skewed / structured keys are cheap).
template <typename K, int RB = kRadixBits>
__global__ void __launch_bounds__(256) k_hist(const K* __restrict__ keys, uint64_t n, int begin_bit, int passes,
                                              uint32_t* __restrict__ hist) {
  extern __shared__ uint32_t sh[];  // passes * 2^RB
  constexpr int kD = 1 << RB;
  for (int i = threadIdx.x; i < passes * kD; i += blockDim.x) sh[i] = 0;
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
      const int sh_bits = begin_bit + p * RB;
      uint32_t cur = digit_of<RB>(kk[0], sh_bits), len = 0;
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        if (q >= cnt) break;
        const uint32_t d = digit_of<RB>(kk[q], sh_bits);
        if (d != cur) {
          atomicAdd(&sh[p * kD + cur], len);
          cur = d;
          len = 0;
        }
        ++len;
      }
      if (len) atomicAdd(&sh[p * kD + cur], len);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kD; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

#ifndef ITT_RADIX_MATCH_OR
#define ITT_RADIX_MATCH_OR 1
#endif
constexpr bool kMatchOr = ITT_RADIX_MATCH_OR != 0;

template <typename K, int BLOCK, int ITEMS, int RB>
struct SmemLayout {
  static constexpr int kTile = BLOCK * ITEMS;
  static constexpr int kWarps = BLOCK / 32;
  static constexpr int kDigits = 1 << RB;
  K keys[kTile];
  uint32_t vals[kTile];
  uint16_t warp_hist[kWarps][kDigits];  // per-warp digit counts, then exclusive offsets across warps
  static constexpr bool kOr = kMatchOr && RB <= 9;  // (10-bit digits: 4 KiB per warp, ballots only)
  uint32_t match[kOr ? kWarps : 1][kOr ? kDigits : 1];  // per-warp lane masks per digit (kept zero)
  uint32_t local_off[kDigits];
  uint32_t global_base[kDigits];
  uint32_t warp_sum[2][kWarps];  // block scan of (tile count, histogram) per digit owner
  uint32_t tile;
};

template <typename K, int BLOCK, int ITEMS, typename Loader, int MINB, int RB, typename SW>
__global__ void __launch_bounds__(BLOCK, MINB) k_onesweep(Loader ld, K* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
                                                          uint64_t n, int shift, const uint32_t* __restrict__ digit_hist,
                                                          SW* __restrict__ status, uint32_t* __restrict__ counter,
                                                          uint32_t pf_dist) {
  using St = Status<SW>;
  using S_t = SmemLayout<K, BLOCK, ITEMS, RB>;
  constexpr int kTile = S_t::kTile;
  constexpr int kWarps = S_t::kWarps;
  constexpr int kDigits = S_t::kDigits;
  // digit owners: thread t owns digits [t*DPT, (t+1)*DPT) (all threads when kDigits >= BLOCK)
  constexpr int DPT = kDigits >= BLOCK ? kDigits / BLOCK : 1;
  constexpr int kOwners = kDigits / DPT;
  static_assert(kDigits % DPT == 0 && kOwners <= BLOCK, "digit ownership");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S_t& S = *reinterpret_cast<S_t*>(smem_raw);
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const bool owner = threadIdx.x < kOwners;
  const int d0 = static_cast<int>(threadIdx.x) * DPT;
  uint32_t hv[DPT];  // this pass's global digit counts
#pragma unroll
  for (int q = 0; q < DPT; ++q) hv[q] = owner ? __ldg(&digit_hist[d0 + q]) : 0u;

  if (threadIdx.x == 0) S.tile = atomicAdd(counter, 1u);
  {
    uint4* wh4 = reinterpret_cast<uint4*>(&S.warp_hist[0][0]);
    for (int i = threadIdx.x; i < kWarps * kDigits * 2 / 16; i += BLOCK) wh4[i] = make_uint4(0, 0, 0, 0);
    if constexpr (S_t::kOr) {
      uint4* m4 = reinterpret_cast<uint4*>(&S.match[0][0]);
      for (int i = threadIdx.x; i < kWarps * kDigits / 4; i += BLOCK) m4[i] = make_uint4(0, 0, 0, 0);
    }
  }
  __syncthreads();
  const uint32_t tile = S.tile;
  const uint64_t tile_base = static_cast<uint64_t>(tile) * kTile;
  if (pf_dist && threadIdx.x == 0) {  // the tile the CTA one residency wave later takes
    const uint64_t pb = tile_base + static_cast<uint64_t>(pf_dist) * kTile;
    if (pb < n) ld.prefetch(pb, umin64(kTile, n - pb));
  }
  const uint64_t warp_base = tile_base + static_cast<uint64_t>(warp) * (32 * ITEMS);

  K key[ITEMS];
  uint32_t val[ITEMS];
  uint32_t rank[ITEMS];
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    const uint64_t i = warp_base + r * 32 + lane;
    if (i < n) ld(i, key[r], val[r]);
  }
  // ---- stable per-warp ranking.  Peers (the lanes holding the same digit) come from ballots over
  // the digit bits that vary in the warp when there are few of them (the group ids of periodic
  // traces: often none), else from one shared-memory atomic OR of the lane bit into the digit's
  // word (kMatchOr): one atomic and one load instead of up to RB ballots.
  uint16_t* wh = S.warp_hist[warp];
  uint32_t* wb = S.match[warp];
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    const uint64_t i = warp_base + r * 32 + lane;
    const bool valid = i < n;
    const uint32_t d = valid ? digit_of<RB>(key[r], shift) : 0u;
    unsigned peers;
    bool or_path = false;
    if constexpr (S_t::kOr) {
      const unsigned vary = (__reduce_or_sync(0xffffffffu, d) ^ __reduce_and_sync(0xffffffffu, d)) & ((1u << RB) - 1u);
      or_path = __popc(vary) > 2;
      if (or_path) {
        if (valid) atomicOr(&wb[d], 1u << lane);
        __syncwarp();
        peers = valid ? wb[d] : 0u;
      } else {
        peers = digit_peers<RB>(d, valid);
      }
    } else {
      peers = digit_peers<RB>(d, valid);
    }
    uint32_t base = 0;
    if (valid) base = wh[d];
    __syncwarp();
    if (valid && lane == static_cast<unsigned>(__ffs(peers) - 1)) {
      wh[d] = static_cast<uint16_t>(base + __popc(peers));
      if (or_path) wb[d] = 0u;  // every peer has read the word (the barrier above)
    }
    __syncwarp();
    rank[r] = base + __popc(peers & lanemask_lt());
  }
  __syncthreads();
  // ---- per digit: warp offsets, tile count (published at once), and the exclusive scans over
  // digits of the tile counts (local offsets) and of the pass histogram (global digit offsets)
  uint32_t cnt[DPT];
  uint32_t csum = 0, hsum = 0;
#pragma unroll
  for (int q = 0; q < DPT; ++q) cnt[q] = 0;
  if (owner) {
#pragma unroll
    for (int q = 0; q < DPT; ++q) {
      const int d = d0 + q;
      uint32_t sum = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        const uint32_t c = S.warp_hist[w][d];
        S.warp_hist[w][d] = static_cast<uint16_t>(sum);
        sum += c;
      }
      cnt[q] = sum;
      St::store(status + static_cast<uint64_t>(tile) * kDigits + d, (tile == 0 ? St::kP : St::kA) | SW(sum));
      csum += sum;
      hsum += hv[q];
    }
  }
  // block exclusive scan of (csum, hsum) over the owners (in digit order = thread order)
  uint32_t ci = csum, hi = hsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t uc = __shfl_up_sync(0xffffffffu, ci, o);
    const uint32_t uh = __shfl_up_sync(0xffffffffu, hi, o);
    if (static_cast<int>(lane) >= o) ci += uc, hi += uh;
  }
  if (lane == 31) S.warp_sum[0][warp] = ci, S.warp_sum[1][warp] = hi;
  __syncthreads();
  uint32_t cex = ci - csum, hex = hi - hsum;
  for (unsigned w = 0; w < warp; ++w) cex += S.warp_sum[0][w], hex += S.warp_sum[1][w];
  uint32_t gofs[DPT];
  if (owner) {
#pragma unroll
    for (int q = 0; q < DPT; ++q) {
      S.local_off[d0 + q] = cex;
      gofs[q] = hex;
      cex += cnt[q];
      hex += hv[q];
    }
  }
  __syncthreads();
  // ---- scatter into shared memory in digit order
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    const uint64_t i = warp_base + r * 32 + lane;
    if (i < n) {
      const uint32_t d = digit_of<RB>(key[r], shift);
      const uint32_t pos = S.local_off[d] + S.warp_hist[warp][d] + rank[r];
      S.keys[pos] = key[r];
      S.vals[pos] = val[r];
    }
  }
  // ---- decoupled look-back per owned digit (predecessors had the whole scatter to publish); the
  // owner's digits walk back together, so their status loads are in flight at the same time
  if (owner) {
    uint32_t excl[DPT];
#pragma unroll
    for (int q = 0; q < DPT; ++q) excl[q] = 0;
    if (tile > 0) {
      bool done[DPT];
#pragma unroll
      for (int q = 0; q < DPT; ++q) done[q] = false;
      for (int64_t t = static_cast<int64_t>(tile) - 1;; t -= kLook) {
        SW sv[DPT][kLook];
#pragma unroll
        for (int q = 0; q < DPT; ++q)
#pragma unroll
          for (int u = 0; u < kLook; ++u)
            sv[q][u] = (!done[q] && t - u >= 0) ? St::load(status + static_cast<uint64_t>(t - u) * kDigits + d0 + q) : SW(0);
        bool all = true;
#pragma unroll
        for (int q = 0; q < DPT; ++q) {
#pragma unroll
          for (int u = 0; u < kLook; ++u) {
            if (done[q]) break;
            SW v = sv[q][u];
            while ((v >> St::kShift) == 0) v = St::load(status + static_cast<uint64_t>(t - u) * kDigits + d0 + q);
            excl[q] += static_cast<uint32_t>(v & St::kMask);
            done[q] = (v >> St::kShift) == 2;
          }
          all = all && done[q];
        }
        if (all) break;
      }
#pragma unroll
      for (int q = 0; q < DPT; ++q)
        St::store(status + static_cast<uint64_t>(tile) * kDigits + d0 + q, St::kP | SW(excl[q] + cnt[q]));
    }
#pragma unroll
    for (int q = 0; q < DPT; ++q) S.global_base[d0 + q] = gofs[q] + excl[q];
  }
  __syncthreads();
  // ---- write out
  const uint32_t valid = static_cast<uint32_t>(n - tile_base < static_cast<uint64_t>(kTile) ? n - tile_base : kTile);
  for (uint32_t p = threadIdx.x; p < valid; p += BLOCK) {
    const K k = S.keys[p];
    const uint32_t d = digit_of<RB>(k, shift);
    const uint32_t o = S.global_base[d] + (p - S.local_off[d]);
    __stcs(&keys_out[o], k);
    __stcs(&vals_out[o], S.vals[p]);
  }
}

// Scratch reused across sorts on one context.
struct Scratch {
  DBuf<uint32_t> hist;    // passes*256 counts
  DBuf<uint32_t> status;  // passes * (tiles * bins look-back words + counter)
  std::vector<uint32_t> host_hist;
};

// tile shapes (BLOCK, ITEMS) of the 8-bit passes; selected at runtime (ITT_RADIX_CFG) for tuning
// sweeps.  Wide (10-bit) passes always use (512, 8).
constexpr int kCfgBlock[] = {512, 256, 384, 256, 512, 512, 512, 256, 256, 256};
constexpr int kCfgItems[] = {8, 16, 12, 8, 16, 8, 8, 8, 16, 12};
int config_index();

// st: this pass's scratch: word 0 = tile counter, then the look-back words (u32 from word 1, or
// u64 from word 2 when n >= kWideStatusN)
template <typename K, int BLOCK, int ITEMS, typename Loader, int MINB = 1024 / BLOCK, int RB = kRadixBits>
void launch_pass(Ctx* c, const Loader& ld, K* ko, uint32_t* vo, uint64_t n, int shift, const uint32_t* dhist, uint32_t* st) {
  constexpr int TILE = BLOCK * ITEMS;
  const size_t smem = sizeof(SmemLayout<K, BLOCK, ITEMS, RB>);
  const uint64_t tiles = (n + TILE - 1) / TILE;
  const char* name = RB <= 9 ? "radix_onesweep" : "radix_onesweep_w10";
  const double bytes = static_cast<double>(n) * 2.0 * (sizeof(K) + 4);
  if (n >= kWideStatusN) {
    auto kern = k_onesweep<K, BLOCK, ITEMS, Loader, MINB, RB, uint64_t>;
    smem_optin(c, kern, smem);
    launch(c, name, bytes, kern, dim3(static_cast<unsigned>(tiles)), dim3(BLOCK), smem, ld, ko, vo, n, shift, dhist,
           reinterpret_cast<uint64_t*>(st + 2), st, prefetch_distance(c->sm_count, MINB));
  } else {
    auto kern = k_onesweep<K, BLOCK, ITEMS, Loader, MINB, RB, uint32_t>;
    smem_optin(c, kern, smem);
    launch(c, name, bytes, kern, dim3(static_cast<unsigned>(tiles)), dim3(BLOCK), smem, ld, ko, vo, n, shift, dhist, st + 1,
           st, prefetch_distance(c->sm_count, MINB));
  }
}

// u32 scratch words one pass of n keys needs (counter + look-back words, see launch_pass)
inline size_t pass_status_words(uint64_t n, uint64_t tiles, int digits) {
  return n >= kWideStatusN ? 2 * (tiles * digits + 1) : tiles * digits + 1;
}

template <typename K, int RB, typename Loader>
void dispatch_pass(Ctx* c, int cfg, const Loader& ld, K* ko, uint32_t* vo, uint64_t n, int shift, const uint32_t* dhist,
                   uint32_t* st) {
  if (n >= kWideStatusN) {  // 64-bit look-back words: one tile shape only
    launch_pass<K, 512, 8, Loader, 2, RB>(c, ld, ko, vo, n, shift, dhist, st);
    return;
  }
  if constexpr (RB != kRadixBits) {
    launch_pass<K, 512, 8, Loader, 2, RB>(c, ld, ko, vo, n, shift, dhist, st);
  } else {
    switch (cfg) {
      case 1: launch_pass<K, 256, 16>(c, ld, ko, vo, n, shift, dhist, st); break;
      case 2: launch_pass<K, 384, 12>(c, ld, ko, vo, n, shift, dhist, st); break;
      case 3: launch_pass<K, 256, 8>(c, ld, ko, vo, n, shift, dhist, st); break;
      case 4: launch_pass<K, 512, 16>(c, ld, ko, vo, n, shift, dhist, st); break;
      case 5: launch_pass<K, 512, 8, Loader, 3>(c, ld, ko, vo, n, shift, dhist, st); break;
      case 6: launch_pass<K, 512, 8, Loader, 4>(c, ld, ko, vo, n, shift, dhist, st); break;
      case 7: launch_pass<K, 256, 8, Loader, 6>(c, ld, ko, vo, n, shift, dhist, st); break;
      case 8: launch_pass<K, 256, 16, Loader, 4>(c, ld, ko, vo, n, shift, dhist, st); break;
      case 9: launch_pass<K, 256, 12, Loader, 5>(c, ld, ko, vo, n, shift, dhist, st); break;
      default: launch_pass<K, 512, 8>(c, ld, ko, vo, n, shift, dhist, st); break;
    }
  }
}

template <int RB>
inline uint64_t tile_of(int cfg) {
  return RB == kRadixBits ? static_cast<uint64_t>(kCfgBlock[cfg]) * kCfgItems[cfg] : 512u * 8u;
}

}  // namespace radix

// Zero the look-back words of a later sort of n keys now (e.g. while the host waits on a readback
// anyway), so that sort can pass status_zeroed = true.  Sized for up to passes8 8-bit or passes_w
// wide passes.
inline void radix_prezero_status(Ctx* c, radix::Scratch& s, uint64_t n, int passes8, int passes_w) {
  const int cfg = n >= radix::kWideStatusN ? 0 : radix::config_index();  // 64-bit words: one tile shape
  const uint64_t t8 = (n + radix::tile_of<radix::kRadixBits>(cfg) - 1) / radix::tile_of<radix::kRadixBits>(cfg);
  const uint64_t tw = (n + radix::tile_of<radix::kWideBits>(cfg) - 1) / radix::tile_of<radix::kWideBits>(cfg);
  const size_t need = std::max(radix::pass_status_words(n, t8, 1 << radix::kRadixBits) * static_cast<size_t>(passes8),
                               radix::pass_status_words(n, tw, 1 << radix::kWideBits) * static_cast<size_t>(passes_w));
  if (s.status.n < need) s.status.alloc(c, need);
  ITT_CUDA(cudaMemsetAsync(s.status.p, 0, need * 4, c->stream));
}

// Sort n (key, value) pairs on bits [begin_bit, end_bit) with RB-bit digits.  Double-buffered: the
// result is in (keys, vals) when the return value is false, in (keys_alt, vals_alt) when true.
//  * hist_in: precomputed per-pass histograms (passes * 2^RB) — skips the histogram kernel;
//  * first_loader: produces the first pass's input instead of reading (keys, vals);
//  * skip_trivial: read the histograms back and drop passes whose digit is constant.
template <typename K, typename FirstLoader = radix::ArrayLoader<K>, int RB = radix::kRadixBits>
bool radix_sort_pairs(Ctx* c, K* keys, uint32_t* vals, K* keys_alt, uint32_t* vals_alt, uint64_t n, int begin_bit,
                      int end_bit, radix::Scratch& s, const uint32_t* hist_in = nullptr,
                      const FirstLoader* first_loader = nullptr, bool skip_trivial = true,
                      bool status_zeroed = false) {
  using namespace radix;
  constexpr int kD = 1 << RB;
  if (end_bit <= begin_bit) end_bit = begin_bit + 1;
  const int passes = (end_bit - begin_bit + RB - 1) / RB;
  const int cfg = n >= kWideStatusN ? 0 : config_index();  // 64-bit look-back words: one tile shape
  const uint64_t tiles = (n + tile_of<RB>(cfg) - 1) / tile_of<RB>(cfg);
  if (n == 0) return false;
  const uint32_t* hist = hist_in;
  if (!hist) {
    if (first_loader) fail(ITT_E_INVALID_ARGUMENT, "internal: a first-pass loader needs precomputed histograms");
    if (s.hist.n < static_cast<size_t>(passes) * kD) s.hist.alloc(c, static_cast<size_t>(passes) * kD);
    ITT_CUDA(cudaMemsetAsync(s.hist.p, 0, static_cast<size_t>(passes) * kD * 4, c->stream));
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(c->sm_count) * 8));
    auto kh = k_hist<K, RB>;
    smem_optin(c, kh, static_cast<size_t>(passes) * kD * 4);
    launch(c, "radix_hist", static_cast<double>(n) * sizeof(K), kh, dim3(grid), dim3(256), static_cast<size_t>(passes) * kD * 4,
           keys, n, begin_bit, passes, s.hist.p);
    hist = s.hist.p;
  }
  std::vector<int> live;
  if (skip_trivial) {
    s.host_hist.resize(static_cast<size_t>(passes) * kD);
    readback(c, s.host_hist.data(), hist, s.host_hist.size());
    for (int p = 0; p < passes; ++p) {
      bool trivial = false;
      for (int d = 0; d < kD; ++d)
        if (s.host_hist[static_cast<size_t>(p) * kD + d] == n) trivial = true;
      if (!trivial) live.push_back(p);
    }
  } else {
    for (int p = 0; p < passes; ++p) live.push_back(p);
  }
  if (first_loader && (live.empty() || live[0] != 0)) live.insert(live.begin(), 0);  // the loader must run
  if (live.empty()) return false;
  const size_t per_pass = pass_status_words(n, tiles, kD);
  if (status_zeroed) {  // the caller zeroed the look-back words ahead of time (radix_prezero_status)
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
      dispatch_pass<K, RB>(c, cfg, *first_loader, ko, vo, n, begin_bit + p * RB, hist + p * kD, st);
    } else {
      const ArrayLoader<K> ld{alt ? keys_alt : keys, alt ? vals_alt : vals};
      dispatch_pass<K, RB>(c, cfg, ld, ko, vo, n, begin_bit + p * RB, hist + p * kD, st);
    }
    alt = !alt;
  }
  return alt;
}

}  // namespace itt
