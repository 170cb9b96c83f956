// sa.cu — suffix array by prefix doubling + LCP by phi / chunked Kasai, sm_100a.
//
// Replaces the Ukkonen suffix tree (suffix_tree.hpp:21-190, built by mine.hpp:38-40): the
// tree's leaves in child-key order are the suffixes of tokens+[terminator] in sorted order
// (SA); internal nodes are the LCP intervals, depth = LCP value, leaf_count = interval width,
// first_leaf = min SA over the interval.
//
// Doubling with dense group ids (rank_i = index of i's group among groups in SA order):
//   init   key_i = the first k symbols of suffix i packed into 32 bits (k = 32 / bits per
//          symbol); one onesweep sort; ids = inclusive count of group starts - 1.
//   round  the sequence E_j = SA_j - h (SA_j + n' - h for SA_j < h: those suffixes are
//          singletons) lists every suffix i in the order of rank_{i+h}.  A STABLE sort of E by
//          rank_i yields SA ordered by (rank_i, rank_{i+h}).  E is never stored: the first radix
//          pass gathers rank[E_j] itself (EmitLoader).  Keys need only bits(G-1) bits (G = group
//          count), so early rounds take 1-2 passes.
//   update one kernel per round: flags from (rank_i, rank_{i+h}) of adjacent suffixes (the
//          second key is gathered here), ids by a decoupled look-back sum scan, scatter
//          rank_new[SA_j], group count, and the digit histograms of the NEXT round's keys
//          (the ids themselves: a non-decreasing run per thread, so one shared atomic per run).
//   stop   when G == n'.
// Every round's id array is kept: level r identifies equal (k * 2^r)-prefixes, so
// lcp(i, j) = sum of the levels where the ids agree (binary lifting) + < k direct compares.
//
// LCP: phi[SA_j] = SA_{j-1}; PLCP by Kasai in chunks of kChunk text positions per thread (each
// chunk restarts at l = 0); a direct comparison longer than kLiftAfter symbols switches to
// lifting, so periodic traces (Sum LCP ~ n^2/2) stay O(n log n); LCP_j = PLCP[SA_j].
#include <algorithm>
#include <climits>
#include <type_traits>

#include "pipeline.cuh"

namespace itt {

namespace {

constexpr int kChunk = 16;
constexpr int kLiftAfter = 24;
constexpr int kRankBlock = 256;
constexpr int kRankItems = 8;  // smaller tiles, 8 CTAs per SM: more look-back chains and scatters in flight (A/B: 182 vs 197 us at 16)
constexpr int kMaxPasses = 4;   // ids < 2^32 in 8-bit digits
constexpr uint32_t kWideGroups = 1u << (2 * radix::kWideBits);  // wide digits for up to 2 passes (G <= 2^20)

// Rank levels are u32, or u16 while the group count allows (periodic traces keep it small): half
// the bytes for the random scatter of the rank update and the gathers that read it back.  A level
// is passed as a tagged address: bit 0 set = u16 (device allocations are 256-B aligned).
constexpr uint64_t kNarrowGroups = 1u << 16;     // ids of a u16 level
constexpr uint64_t kNarrowTry = 1u << 14;        // try u16 for the next level while G <= this
__device__ __forceinline__ uint32_t rank_at(uintptr_t lv, uint64_t i) {
  return (lv & 1u) ? static_cast<uint32_t>(__ldg(reinterpret_cast<const uint16_t*>(lv - 1) + i))
                   : __ldg(reinterpret_cast<const uint32_t*>(lv) + i);
}
__device__ __forceinline__ void rank_put(uintptr_t lv, uint64_t i, uint32_t v) {
  if (lv & 1u) reinterpret_cast<uint16_t*>(lv - 1)[i] = static_cast<uint16_t>(v);
  else reinterpret_cast<uint32_t*>(lv)[i] = v;
}

__global__ void k_token_stats(const int32_t* __restrict__ tok, uint64_t n, int32_t term, int* out /*min,max,termhits*/) {
  int mn = INT_MAX, mx = INT_MIN, hits = 0;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int v = tok[i];
    mn = min(mn, v);
    mx = max(mx, v);
    hits += v == term;
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    hits += __shfl_xor_sync(0xffffffffu, hits, o);
  }
  if (lane_id() == 0) {
    atomicMin(&out[0], mn);
    atomicMax(&out[1], mx);
    if (hits) atomicAdd(&out[2], hits);
  }
}

// codes (tokens - lo, terminator appended at n) and the first k symbols of every suffix packed
// into 32 bits, in one pass over the tokens
// The same keys, plus the 8-bit digit histograms of every pass of the init sort (shared-memory
// counts flushed once per block): the sort then needs no histogram pass over the keys.
template <int RB>
__global__ void __launch_bounds__(256) k_text_keys_hist(const int32_t* __restrict__ tok, uint64_t n, int32_t term, int32_t lo,
                                                        int bits, int k, int passes, int32_t* __restrict__ text,
                                                        uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                                        uint32_t* __restrict__ hist) {
  // tiles of 1024 positions: the codes (+ k-1 halo) staged in shared memory with 16-byte loads,
  // four consecutive keys per thread written with 16-byte stores
  constexpr int kB = 1 << RB, kT = 1024;
  __shared__ uint32_t sh[(32 / RB + 1) * kB];
  __shared__ __align__(16) uint32_t s_c[kT + 32];
  for (int i = threadIdx.x; i < passes * kB; i += blockDim.x) sh[i] = 0;
  const uint64_t np = n + 1;
  const auto code = [&](uint64_t j) -> uint32_t {
    return j < n ? static_cast<uint32_t>(__ldg(&tok[j]) - lo) : (j == n ? static_cast<uint32_t>(term - lo) : 0u);
  };
  const bool tok_vec = (reinterpret_cast<uintptr_t>(tok) & 15) == 0;
  const bool out_vec = ((reinterpret_cast<uintptr_t>(text) | reinterpret_cast<uintptr_t>(keys) |
                         (vals ? reinterpret_cast<uintptr_t>(vals) : 0)) & 15) == 0;
  const uint64_t tiles = (np + kT - 1) / kT;
  for (uint64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const uint64_t base = tile * kT;
    __syncthreads();  // the previous tile's codes are consumed (and the histogram is zeroed)
    const uint64_t j0 = base + threadIdx.x * 4;
    if (tok_vec && j0 + 4 <= n) {
      const int4 v = __ldcs(reinterpret_cast<const int4*>(tok + j0));
      *reinterpret_cast<uint4*>(&s_c[threadIdx.x * 4]) =
          make_uint4(static_cast<uint32_t>(v.x - lo), static_cast<uint32_t>(v.y - lo), static_cast<uint32_t>(v.z - lo),
                     static_cast<uint32_t>(v.w - lo));
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) s_c[threadIdx.x * 4 + e] = code(j0 + e);
    }
    if (threadIdx.x < 32) s_c[kT + threadIdx.x] = code(base + kT + threadIdx.x);
    __syncthreads();
    uint32_t kv[4], cv[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int o = threadIdx.x * 4 + e;
      uint32_t key = 0;
      for (int q = 0; q < k; ++q) key = (key << bits) | s_c[o + q];
      kv[e] = key;
      cv[e] = s_c[o];
    }
    if (out_vec && j0 + 4 <= np) {
      __stcs(reinterpret_cast<uint4*>(keys + j0), make_uint4(kv[0], kv[1], kv[2], kv[3]));
      *reinterpret_cast<uint4*>(text + j0) = make_uint4(cv[0], cv[1], cv[2], cv[3]);
      if (vals) __stcs(reinterpret_cast<uint4*>(vals + j0), make_uint4(j0, j0 + 1, j0 + 2, j0 + 3));
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (j0 + e < np) {
          keys[j0 + e] = kv[e];
          text[j0 + e] = static_cast<int32_t>(cv[e]);
          if (vals) vals[j0 + e] = static_cast<uint32_t>(j0 + e);  // null: the sort's first pass generates positions
        }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (j0 + e < np)
        for (int p = 0; p < passes; ++p) atomicAdd(&sh[p * kB + ((kv[e] >> (RB * p)) & (kB - 1u))], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kB; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

__global__ void k_text_keys(const int32_t* __restrict__ tok, uint64_t n, int32_t term, int32_t lo, int bits, int k,
                            int32_t* __restrict__ text, uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t np = n + 1;
  if (i >= np) return;
  uint32_t key = 0;
  for (int q = 0; q < k; ++q) {
    // padding past the unique terminator is never decisive
    const uint64_t j = i + q;
    const uint32_t c = j < n ? static_cast<uint32_t>(__ldg(&tok[j]) - lo) : (j == n ? static_cast<uint32_t>(term - lo) : 0u);
    if (q == 0) text[i] = static_cast<int32_t>(c);
    key = (key << bits) | c;
  }
  keys[i] = key;
  vals[i] = static_cast<uint32_t>(i);
}

// first radix pass input of a doubling round: E_j and its key rank_{E_j}
struct EmitLoader {
  const uint32_t* sa;
  uintptr_t rank;  // tagged level (rank_at)
  uint64_t np;
  uint32_t h;
  __device__ __forceinline__ void operator()(uint64_t j, uint32_t& k, uint32_t& v) const {
    const uint32_t x = __ldcs(&sa[j]);
    const uint32_t i = x >= h ? x - h : static_cast<uint32_t>(x + np - h);
    k = rank_at(rank, i);
    v = i;
  }
  __device__ __forceinline__ void prefetch(uint64_t j, uint64_t cnt) const { prefetch_l2(sa + j, cnt * 4); }
};

// New dense ids.  flag_j = (key_j, r2_j) != (key_{j-1}, r2_{j-1}) with key = old id of SA_j (the
// sorted keys) and r2 = old id of SA_j + h (gathered here; none when SA_j + h >= n' or when
// rank_old is null in the init round).  id_j = inclusive count of flags - 1 (decoupled look-back
// sum scan); rank_new[SA_j] = id_j; hist_next[p][digit_p(id_j)] += 1.
// kHeads: rank_new holds the SA position of each group's head instead of a dense id (u32; the
// scan is a max over head positions and G is counted separately into *gcount) — what refinement
// rounds continue from without a conversion pass.
// The first level (k-gram keys, head positions) without the random scatter: while the init rank
// update walks SA order, each group head enters its (key -> head position) into a small hash
// table; k_init_fill then writes rank[x] = table[key(x)] in TEXT order — sequential stores
// instead of one 32-byte sector read-modify-write per suffix.  Only while the distinct k-grams
// fit the table (periodic traces: thousands); otherwise the scatter (the overflow bit, bit 63 of
// the group counter, makes the host re-run the update without the table).
constexpr uint32_t kInitMapBits = 16;  // 64K entries of 8 bytes: L1/L2-resident during the fill
constexpr int kInitMapProbe = 64;
__device__ __forceinline__ uint32_t init_map_slot(uint32_t key, uint32_t mask) {
  return static_cast<uint32_t>((static_cast<uint64_t>(key) * 0x9E3779B97F4A7C15ull) >> 32) & mask;
}
// entry = head << 33 | 1 << 32 | key (0 = empty; heads < 2^31 in heads mode)
__device__ __forceinline__ void init_map_insert(unsigned long long* map, uint32_t mask, uint32_t key, uint32_t val,
                                                unsigned long long* overflow) {
  uint32_t sl = init_map_slot(key, mask);
  const unsigned long long e = (static_cast<unsigned long long>(val) << 33) | (1ull << 32) | key;
  for (int p = 0; p < kInitMapProbe; ++p) {
    if (atomicCAS(&map[sl], 0ull, e) == 0ull) return;  // every key is inserted once (at its group's head)
    sl = (sl + 1) & mask;
  }
  atomicOr(overflow, 1ull << 63);
}
// 4 positions per thread: one 16-byte store of ranks (u32 levels)
__global__ void __launch_bounds__(256) k_init_fill(const int32_t* __restrict__ text, uint64_t np, int bits, int k,
                                                   const unsigned long long* __restrict__ map, uint32_t mask,
                                                   uint32_t* __restrict__ level) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x * 4;
  for (uint64_t x0 = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4; x0 < np; x0 += stride) {
    uint32_t r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t x = x0 + u;
      r[u] = 0;
      if (x >= np) continue;
      uint32_t key = 0;
      for (int q = 0; q < k; ++q) {  // the same packing as k_text_keys (text[np - 1] is the terminator code)
        const uint64_t j = x + q;
        key = (key << bits) | (j < np ? static_cast<uint32_t>(__ldg(&text[j])) : 0u);
      }
      uint32_t sl = init_map_slot(key, mask);
      const unsigned long long want = (1ull << 32) | key;
      unsigned long long e = __ldg(&map[sl]);
      while ((e & 0x1FFFFFFFFull) != want) {
        sl = (sl + 1) & mask;
        e = __ldg(&map[sl]);
      }
      r[u] = static_cast<uint32_t>(e >> 33);
    }
    if (x0 + 4 <= np) {
      __stcs(reinterpret_cast<uint4*>(level + x0), make_uint4(r[0], r[1], r[2], r[3]));
    } else {
      for (int u = 0; u < 4; ++u)
        if (x0 + u < np) level[x0 + u] = r[u];
    }
  }
}

// The init level through the k-gram table needs no scan: a head's rank is its own SA position,
// the level is filled in text order afterwards (k_init_fill), and head-position levels take their
// digit histograms from the level itself.  So: heads from adjacent sorted keys, G, table inserts —
// the sorted keys read once with 16-byte loads, no look-back chain and no SA read.
__global__ void __launch_bounds__(256) k_init_heads(const uint32_t* __restrict__ keys, uint64_t np,
                                                    uint8_t* __restrict__ heads_out, unsigned long long* gcount,
                                                    unsigned long long* init_map, uint32_t map_mask) {
  static_assert(kRankItems == 8, "one head byte per thread");
  const uint64_t base = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * kRankItems;
  uint32_t kv[kRankItems];
  uint32_t fmask = 0;
  if (base < np) {
    if (base + kRankItems <= np) {
      const uint4 a = __ldcs(reinterpret_cast<const uint4*>(keys + base));
      const uint4 b = __ldcs(reinterpret_cast<const uint4*>(keys + base + 4));
      kv[0] = a.x, kv[1] = a.y, kv[2] = a.z, kv[3] = a.w, kv[4] = b.x, kv[5] = b.y, kv[6] = b.z, kv[7] = b.w;
    } else {
#pragma unroll
      for (int q = 0; q < kRankItems; ++q) kv[q] = base + q < np ? keys[base + q] : 0u;
    }
    uint32_t pk = base > 0 ? keys[base - 1] : 0u;
#pragma unroll
    for (int q = 0; q < kRankItems; ++q) {
      const uint64_t j = base + q;
      if (j < np && (j == 0 || kv[q] != pk)) fmask |= 1u << q;
      pk = kv[q];
    }
    heads_out[base / kRankItems] = static_cast<uint8_t>(fmask);
    for (uint32_t m = fmask; m; m &= m - 1) {
      const int q = __ffs(m) - 1;
      init_map_insert(init_map, map_mask, kv[q], static_cast<uint32_t>(base + q), gcount);
    }
  }
  uint32_t g = __popc(fmask);
  g = __reduce_add_sync(0xffffffffu, g);
  if (lane_id() == 0 && g) atomicAdd(gcount, static_cast<unsigned long long>(g));
}

template <bool kHeads>
__global__ void __launch_bounds__(kRankBlock, 8) k_rank_update(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ sa,
                                                            uintptr_t rank_old, uint32_t h, uint64_t np,
                                                            uintptr_t rank_new, uint32_t* __restrict__ hist_next,
                                                            int passes, uint32_t* __restrict__ gstart,
                                                            uint64_t* status, uint32_t* counter, uint32_t pf_dist,
                                                            uint8_t* __restrict__ heads_out,
                                                            unsigned long long* __restrict__ gcount,
                                                            unsigned long long* __restrict__ init_map, uint32_t map_mask) {
  __shared__ uint32_t s_warp[kRankBlock / 32];
  __shared__ uint32_t s_tile, s_prefix;
  __shared__ uint32_t s_hist[kMaxPasses][256];
  for (int i = threadIdx.x; i < kMaxPasses * 256; i += kRankBlock) (&s_hist[0][0])[i] = 0;
  if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t base = static_cast<uint64_t>(tile) * (kRankBlock * kRankItems) + static_cast<uint64_t>(threadIdx.x) * kRankItems;
  if (pf_dist && threadIdx.x == 0) {  // keys + SA of the tile one residency wave later
    const uint64_t pb = (static_cast<uint64_t>(tile) + pf_dist) * (kRankBlock * kRankItems);
    if (pb < np) {
      const uint64_t cnt = umin64(kRankBlock * kRankItems, np - pb);
      prefetch_l2(keys + pb, cnt * 4);
      prefetch_l2(sa + pb, cnt * 4);
    }
  }
  auto second = [&](uint32_t x) -> uint32_t {
    if (!rank_old) return 0u;
    const uint64_t y = static_cast<uint64_t>(x) + h;
    return y < np ? rank_at(rank_old, y) : kNone;
  };
  // phase 1: this thread's SA entries and sorted keys (16-byte loads when the run is whole)
  uint32_t s_idx[kRankItems], kv[kRankItems], r2[kRankItems];
  const bool whole = base + kRankItems <= np;
  if (whole) {
#pragma unroll
    for (int q = 0; q < kRankItems; q += 4) {
      const uint4 a = __ldcs(reinterpret_cast<const uint4*>(sa + base + q));
      const uint4 b = __ldcs(reinterpret_cast<const uint4*>(keys + base + q));
      s_idx[q] = a.x, s_idx[q + 1] = a.y, s_idx[q + 2] = a.z, s_idx[q + 3] = a.w;
      kv[q] = b.x, kv[q + 1] = b.y, kv[q + 2] = b.z, kv[q + 3] = b.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < kRankItems; ++q) {
      s_idx[q] = base + q < np ? sa[base + q] : 0u;
      kv[q] = base + q < np ? keys[base + q] : 0u;
    }
  }
  // phase 2: every second-key gather in flight before any compare
  uint32_t pk = 0, pr = 0;
  if (base < np && base > 0) {
    pk = keys[base - 1];
    pr = second(sa[base - 1]);
  }
#pragma unroll
  for (int q = 0; q < kRankItems; ++q) r2[q] = base + q < np ? second(s_idx[q]) : 0u;
  // phase 3: group-start flags as a bit mask (keeps the register footprint to s_idx + mask)
  uint32_t fmask = 0;
#pragma unroll
  for (int q = 0; q < kRankItems; ++q) {
    const uint64_t j = base + q;
    if (j < np) {
      if (j == 0 || kv[q] != pk || r2[q] != pr) fmask |= 1u << q;
      pk = kv[q];
      pr = r2[q];
    }
  }
  if (heads_out && base < np) heads_out[base / kRankItems] = static_cast<uint8_t>(fmask);  // group heads, SA order
  using ScanOp = typename std::conditional<kHeads, MaxOp<uint32_t>, SumOp<uint32_t>>::type;
  // dense: flags in the run; heads: (last head position in the run) + 1, 0 = none
  const uint32_t run = kHeads ? (fmask ? static_cast<uint32_t>(base) + (31 - __clz(fmask)) + 1 : 0u) : __popc(fmask);
  uint32_t total;
  const uint32_t texcl = block_exclusive_scan<uint32_t, ScanOp, kRankBlock>(run, ScanOp(), &total, s_warp);
  if (threadIdx.x < 32) {
    const uint32_t p = tile_lookback<uint32_t, ScanOp>(status, tile, total, ScanOp());
    if (threadIdx.x == 0) s_prefix = p;
  }
  if constexpr (kHeads) {  // G = number of heads
    uint32_t g = __popc(fmask);
    for (int o = 16; o > 0; o >>= 1) g += __shfl_xor_sync(0xffffffffu, g, o);
    if (lane_id() == 0 && g) atomicAdd(gcount, static_cast<unsigned long long>(g));
  }
  __syncthreads();
  const uint32_t pre = ScanOp()(s_prefix, texcl);
  uint32_t last_head = pre;  // kHeads: running (last head + 1)
  // ids are non-decreasing across the thread's items: one shared atomic per run of equal digits
  uint32_t cur[kMaxPasses], len[kMaxPasses];
#pragma unroll
  for (int p = 0; p < kMaxPasses; ++p) cur[p] = kNone, len[p] = 0;
#pragma unroll
  for (int q = 0; q < kRankItems; ++q) {
    const uint64_t j = base + q;
    if (j < np) {
      uint32_t id;
      if constexpr (kHeads) {
        if ((fmask >> q) & 1u) last_head = static_cast<uint32_t>(j) + 1;
        id = last_head - 1;
      } else {
        id = pre + __popc(fmask & ((2u << q) - 1u)) - 1;
      }
      if (kHeads && init_map) {  // init: key -> head position for the text-order fill (k_init_fill), no scatter
        if ((fmask >> q) & 1u) init_map_insert(init_map, map_mask, kv[q], id, gcount);
      } else {
        rank_put(rank_new, s_idx[q], id);  // ids beyond a u16 level are caught by the host (G > 2^16)
      }
      // group starts (SA position of each group's first suffix) for the wide-digit histograms
      if (!kHeads && gstart && ((fmask >> q) & 1u) && id < kWideGroups) gstart[id] = static_cast<uint32_t>(j);
#pragma unroll
      for (int p = 0; p < kMaxPasses; ++p) {
        if (p >= passes) break;
        const uint32_t d = (id >> (8 * p)) & 0xFFu;
        if (d != cur[p]) {
          if (len[p]) atomicAdd(&s_hist[p][cur[p]], len[p]);
          cur[p] = d;
          len[p] = 0;
        }
        ++len[p];
      }
    }
  }
#pragma unroll
  for (int p = 0; p < kMaxPasses; ++p)
    if (p < passes && len[p]) atomicAdd(&s_hist[p][cur[p]], len[p]);
  __syncthreads();
  for (int i = threadIdx.x; i < passes * 256; i += kRankBlock) {
    const uint32_t v = (&s_hist[0][0])[i];
    if (v) atomicAdd(&hist_next[i], v);
  }
}

// 10-bit digit histograms of the next round's keys from the group sizes: every suffix carries its
// group's id, so digit d of pass p counts the suffixes of the groups whose id has digit d
// (G <= kWideGroups groups, one thread each)
__global__ void k_wide_hist(const uint32_t* __restrict__ gstart, uint64_t g, uint64_t np, int passes,
                            uint32_t* __restrict__ hist) {
  constexpr int kW = 1 << radix::kWideBits;
  __shared__ uint32_t sh[2 * kW];
  for (int i = threadIdx.x; i < passes * kW; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (uint64_t id = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; id < g;
       id += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t size = static_cast<uint32_t>((id + 1 < g ? gstart[id + 1] : np) - gstart[id]);
    for (int p = 0; p < passes; ++p) atomicAdd(&sh[p * kW + ((id >> (radix::kWideBits * p)) & (kW - 1))], size);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kW; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// ---------------------------------------------------------------- refinement rounds
// largest prefix-length ratio between consecutive levels kept for LCP lifting (ITT_LIFT_RATIO: A/B)
inline uint64_t lift_ratio() {
  static const uint64_t r = [] {
    const char* e = std::getenv("ITT_LIFT_RATIO");
    const long v = e && *e ? std::atol(e) : 16;
    return static_cast<uint64_t>(v >= 2 ? v : 2);
  }();
  return r;
}
// A doubling round that finds every group already ordered by its second key needs no sort: the
// SA stays, groups split where the second key changes.  Traces of training loops reach this state
// after a few rounds (every group is one rotation class of the loop body; a round only splits off
// the members whose second half reaches the end of the trace, and they already sit last in their
// group, in order).  Within a group the members are in text-position order (every sort is stable
// from the position order of the first one), so the check is: for each non-head j, r2_j >= r2_{j-1}.
// Levels written by refinement rounds hold the SA position of the group head (u32) instead of a
// dense id: then a round rewrites only the ranks of suffixes whose group head moved.
struct HeadPair {  // (last new head + 1, last old head + 1) in two 31-bit halves; positions < 2^31
  __device__ __forceinline__ uint64_t operator()(uint64_t a, uint64_t b) const {
    const uint64_t m = (1ull << 31) - 1;
    return (umax64(a >> 31, b >> 31) << 31) | umax64(a & m, b & m);
  }
  static __device__ __forceinline__ uint64_t identity() { return 0; }
};

// r2_j = rank_h[SA_j + h] (kNone past the end); new head flags; counts of new groups and inversions
__global__ void __launch_bounds__(kRankBlock) k_refine_detect(const uint32_t* __restrict__ sa, const uint8_t* __restrict__ heads,
                                                             uintptr_t rank, uint32_t h, uint64_t np,
                                                             uint8_t* __restrict__ heads_next,
                                                             unsigned long long* __restrict__ counts /*[0] groups, [1] inversions*/,
                                                             unsigned int* __restrict__ abort_flag) {
  __shared__ uint32_t s_last[kRankBlock / 32];
  __shared__ unsigned long long s_cnt[2];
  __shared__ unsigned int s_abort;
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_abort = ld_relaxed_u32(abort_flag);
  if (threadIdx.x < 2) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  if (s_abort) return;  // an earlier round (or block of this one) found inversions: the host redoes it
  const uint64_t base = (static_cast<uint64_t>(blockIdx.x) * kRankBlock + threadIdx.x) * kRankItems;
  auto second = [&](uint32_t x) -> uint32_t {
    const uint64_t y = static_cast<uint64_t>(x) + h;
    return y < np ? rank_at(rank, y) : kNone;
  };
  uint32_t r2[kRankItems];
  uint8_t hb = 0;
  if (base < np) {
    hb = heads[base / kRankItems];
    if (base + kRankItems <= np) {
#pragma unroll
      for (int q = 0; q < kRankItems; q += 4) {
        const uint4 a = __ldcs(reinterpret_cast<const uint4*>(sa + base + q));
        r2[q] = second(a.x), r2[q + 1] = second(a.y), r2[q + 2] = second(a.z), r2[q + 3] = second(a.w);
      }
    } else {
#pragma unroll
      for (int q = 0; q < kRankItems; ++q) r2[q] = base + q < np ? second(sa[base + q]) : 0u;
    }
  } else {
#pragma unroll
    for (int q = 0; q < kRankItems; ++q) r2[q] = 0u;
  }
  // r2 of item base - 1: the previous lane, the previous warp, or (thread 0) one more gather
  uint32_t prev = __shfl_up_sync(0xffffffffu, r2[kRankItems - 1], 1);
  if (lane == 31) s_last[warp] = r2[kRankItems - 1];
  __syncthreads();
  if (lane == 0) prev = warp > 0 ? s_last[warp - 1] : (base > 0 && base < np ? second(sa[base - 1]) : 0u);
  uint32_t nh = 0, inv = 0;
#pragma unroll
  for (int q = 0; q < kRankItems; ++q) {
    const uint64_t j = base + q;
    if (j < np) {
      const bool head = j == 0 || ((hb >> q) & 1u);
      if (!head && r2[q] < prev) ++inv;
      if (head || r2[q] != prev) nh |= 1u << q;
    }
    prev = r2[q];
  }
  if (base < np) heads_next[base / kRankItems] = static_cast<uint8_t>(nh);
  uint32_t g = __popc(nh);
  for (int o = 16; o > 0; o >>= 1) {
    g += __shfl_xor_sync(0xffffffffu, g, o);
    inv += __shfl_xor_sync(0xffffffffu, inv, o);
  }
  if (lane == 0) {
    if (g) atomicAdd(&s_cnt[0], static_cast<unsigned long long>(g));
    if (inv) atomicAdd(&s_cnt[1], static_cast<unsigned long long>(inv));
  }
  __syncthreads();
  if (threadIdx.x < 2 && s_cnt[threadIdx.x]) atomicAdd(&counts[threadIdx.x], s_cnt[threadIdx.x]);
  if (threadIdx.x == 1 && s_cnt[1]) atomicOr(abort_flag, 1u);  // rounds queued after this one return at once
}

// rank_{2h}[SA_j] = position of j's new group head, written where it differs from the old head
// (all j when the previous level holds dense ids): a max-scan of (last new head, last old head)
// over SA order with decoupled look-back.  kApplyWords words of each bitmap (32 positions each) per
// thread, so a tile covers 64K positions and the look-back chain is short; SA is read only where a
// rank is written, so a settled round touches little more than the bitmaps.
constexpr int kApplyItems = 32;   // positions per bitmap word
// final groups at most np / kHeadsLcpRatio: LCP from the head bitmap + lifting (k_lcp_heads)
// instead of phi + capped Kasai + gather
constexpr uint64_t kHeadsLcpRatio = 64;
#ifndef ITT_APPLY_WORDS
#define ITT_APPLY_WORDS 8  // C3: 106 -> 53 -> 39 us per launch for 1, 4, 8 words (16: 41)
#endif
constexpr int kApplyWords = ITT_APPLY_WORDS;  // words per thread
// this thread's (last new head + 1, last old head + 1) over its kApplyWords bitmap words
__device__ __forceinline__ uint64_t apply_run(const uint32_t* __restrict__ heads_old, const uint32_t* __restrict__ heads_new,
                                              uint64_t np, uint64_t w0, uint32_t (&ho)[kApplyWords], uint32_t (&hn)[kApplyWords]) {
  uint64_t ln = 0, lo = 0;
  if (kApplyWords % 4 == 0 && (w0 + kApplyWords) * kApplyItems <= np) {  // whole words: 16-byte loads
#pragma unroll
    for (int u = 0; u < kApplyWords; u += 4) {
      const uint4 a = __ldcs(reinterpret_cast<const uint4*>(heads_old + w0 + u));
      const uint4 b = __ldcs(reinterpret_cast<const uint4*>(heads_new + w0 + u));
      ho[u] = a.x, ho[u + 1] = a.y, ho[u + 2] = a.z, ho[u + 3] = a.w;
      hn[u] = b.x, hn[u + 1] = b.y, hn[u + 2] = b.z, hn[u + 3] = b.w;
    }
  } else {
#pragma unroll
    for (int u = 0; u < kApplyWords; ++u) {
      const uint64_t base = (w0 + u) * kApplyItems;
      ho[u] = hn[u] = 0;
      if (base < np) {
        const uint32_t live = np - base >= kApplyItems ? 0xFFFFFFFFu : (1u << (np - base)) - 1u;  // bits past np are unset
        ho[u] = __ldcs(&heads_old[w0 + u]) & live;
        hn[u] = __ldcs(&heads_new[w0 + u]) & live;
      }
    }
  }
#pragma unroll
  for (int u = 0; u < kApplyWords; ++u) {
    const uint64_t base = (w0 + u) * kApplyItems;
    if (hn[u]) ln = base + (31 - __clz(hn[u])) + 1;
    if (ho[u]) lo = base + (31 - __clz(ho[u])) + 1;
  }
  return (ln << 31) | lo;
}
// reduce-then-scan form of the apply (ITT_APPLY_RS=1; A/B only, the look-back form is faster at C3):
// per-tile HeadPair totals, one block scans them (k_scan_tile_totals), then k_refine_apply<true>
__global__ void __launch_bounds__(kRankBlock) k_refine_totals(const uint32_t* __restrict__ heads_old,
                                                             const uint32_t* __restrict__ heads_new, uint64_t np,
                                                             uint64_t* __restrict__ tot, const unsigned int* __restrict__ abort_flag) {
  __shared__ uint64_t s_w[kRankBlock / 32];
  if (ld_relaxed_u32(abort_flag)) return;
  uint32_t ho[kApplyWords], hn[kApplyWords];
  const HeadPair op;
  const uint64_t w0 = (static_cast<uint64_t>(blockIdx.x) * kRankBlock + threadIdx.x) * kApplyWords;
  uint64_t run = apply_run(heads_old, heads_new, np, w0, ho, hn);
  for (int o = 16; o > 0; o >>= 1) run = op(run, __shfl_xor_sync(0xffffffffu, run, o));
  if (lane_id() == 0) s_w[threadIdx.x >> 5] = run;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = s_w[0];
    for (int w = 1; w < kRankBlock / 32; ++w) t = op(t, s_w[w]);
    tot[blockIdx.x] = t;
  }
}
template <bool kRS>
__global__ void __launch_bounds__(kRankBlock) k_refine_apply(const uint32_t* __restrict__ sa, const uint32_t* __restrict__ heads_old,
                                                            const uint32_t* __restrict__ heads_new, uint64_t np,
                                                            uint32_t* __restrict__ level, int full, uint64_t* status,
                                                            uint32_t* counter, const unsigned int* __restrict__ abort_flag,
                                                            const uint64_t* __restrict__ tile_excl) {
  __shared__ uint64_t s_warp[kRankBlock / 32];
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_prefix;
  __shared__ unsigned int s_abort;
  if (threadIdx.x == 0) {
    s_abort = ld_relaxed_u32(abort_flag);
    if constexpr (kRS) {
      s_tile = blockIdx.x;
      s_prefix = s_abort ? 0 : tile_excl[blockIdx.x];
    } else {
      s_tile = atomicAdd(counter, 1u);
    }
  }
  __syncthreads();
  if (s_abort) return;  // this round's detect (or an earlier one) found inversions
  const uint32_t tile = s_tile;
  const uint64_t w0 = (static_cast<uint64_t>(tile) * kRankBlock + threadIdx.x) * kApplyWords;  // first bitmap word
  uint32_t ho[kApplyWords], hn[kApplyWords];
  const uint64_t run = apply_run(heads_old, heads_new, np, w0, ho, hn);  // this thread's last heads (+1; 0 = none)
  const HeadPair op;
  uint64_t total;
  const uint64_t texcl = block_exclusive_scan<uint64_t, HeadPair, kRankBlock>(run, op, &total, s_warp);
  if constexpr (!kRS) {
    if (threadIdx.x < 32) {
      const uint64_t p = tile_lookback<uint64_t, HeadPair>(status, tile, total, op);
      if (threadIdx.x == 0) s_prefix = p;
    }
    __syncthreads();
  }
  const uint64_t pre = op(s_prefix, texcl);
  uint64_t cn = pre >> 31, co = pre & ((1ull << 31) - 1);  // last heads before this run (+1)
#pragma unroll
  for (int u = 0; u < kApplyWords; ++u) {
    const uint64_t base = (w0 + u) * kApplyItems;
    if (base >= np) break;
    const int cnt = static_cast<int>(umin64(kApplyItems, np - base));
    if (!full && hn[u] == ho[u] && cn == co) {  // no head moved in or before this word's groups
      if (hn[u]) cn = co = base + (31 - __clz(hn[u])) + 1;
      continue;
    }
    if (full && cnt == kApplyItems) {  // every rank changes representation: the word's SA in 16-byte loads
#pragma unroll
      for (int q4 = 0; q4 < kApplyItems; q4 += 4) {
        const uint4 v = *reinterpret_cast<const uint4*>(sa + base + q4);
        const uint32_t x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if ((hn[u] >> (q4 + q)) & 1u) cn = base + q4 + q + 1;
          if ((ho[u] >> (q4 + q)) & 1u) co = base + q4 + q + 1;
          level[x[q]] = static_cast<uint32_t>(cn - 1);
        }
      }
      continue;
    }
    for (int q = 0; q < cnt; ++q) {
      if ((hn[u] >> q) & 1u) cn = base + q + 1;
      if ((ho[u] >> q) & 1u) co = base + q + 1;
      if (full || cn != co) level[sa[base + q]] = static_cast<uint32_t>(cn - 1);
    }
  }
}


// ---------------------------------------------------------------- LCP
__global__ void k_phi(const uint32_t* __restrict__ sa, uint64_t np, uint32_t* __restrict__ phi) {
  const uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j < np) phi[sa[j]] = j > 0 ? sa[j - 1] : kNone;
}

struct LiftArgs {
  const int32_t* text;
  uint64_t np;
  const uintptr_t* levels;  // device array of tagged level addresses (rank_at)
  const uint32_t* hs;       // prefix length of each level, ascending, consecutive ones within lift_ratio()
  int nlev;
};

// lcp of suffixes a != b, or `limit` if it is at least that, by lifting over the kept levels: a
// level is applied while the ids agree (at most lift_ratio() - 1 times below a level that did not
// agree), then direct compares below the smallest level
__device__ __forceinline__ uint32_t lcp_lift(const LiftArgs& L, uint64_t a, uint64_t b, uint32_t limit) {
  uint32_t acc = 0;
  for (int r = L.nlev - 1; r >= 0; --r) {
    const uintptr_t lv = L.levels[r];
    const uint32_t hr = L.hs[r];
    while (acc < limit && a < L.np && b < L.np && rank_at(lv, a) == rank_at(lv, b)) {
      a += hr;
      b += hr;
      acc += hr;
    }
  }
  while (acc < limit && a < L.np && b < L.np && __ldg(&L.text[a]) == __ldg(&L.text[b])) ++a, ++b, ++acc;
  return acc;
}

// PLCP capped at `cap` over a SA sorted by the first h_final >= cap symbols (a full SA when every
// group is a singleton).  Suffixes in the same final group share >= h_final symbols: plcp = cap.
// Kasai's carried bound lcp(i-1, phi) - 1 holds across groups (their order is exact) EXCEPT when it
// was capped and i opens its group: then the predecessor lies in another group and the scan
// restarts at 0.  Anything below h_final is exact (direct compares, then lifting).  Proof sketch:
// the carry needs suffix p+1 (p = phi(i-1)) to precede i with every suffix in between sharing
// >= lcp(p+1, i) symbols with i; group order is exact, so this can only fail when p+1 and i share
// a group, i.e. lcp(p, i-1) >= h_final + 1, i.e. i-1 itself took the same-group shortcut.
__global__ void k_plcp(LiftArgs L, const uint32_t* __restrict__ phi, uint32_t* __restrict__ plcp, uint32_t cap) {
  const uint64_t i0 = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * kChunk;
  if (i0 >= L.np) return;
  const uint64_t i1 = min(i0 + kChunk, L.np);
  const uintptr_t top = L.levels[L.nlev - 1];
  uint32_t l = 0;
  bool capped = false;
  for (uint64_t i = i0; i < i1; ++i) {
    const uint32_t p = phi[i];
    if (p == kNone) {
      plcp[i] = 0;
      l = 0;
      capped = false;
      continue;
    }
    if (rank_at(top, i) == rank_at(top, p)) {  // same final group: lcp >= h_final >= cap
      plcp[i] = cap;
      l = cap - 1;
      capped = true;
      continue;
    }
    if (capped) l = 0;
    int steps = 0;
    while (l < cap && i + l < L.np && p + l < L.np && __ldg(&L.text[i + l]) == __ldg(&L.text[p + l])) {
      ++l;
      if (++steps == kLiftAfter) {
        l += lcp_lift(L, i + l, static_cast<uint64_t>(p) + l, cap - l);
        break;
      }
    }
    if (l > cap) l = cap;
    plcp[i] = l;
    capped = false;  // i-1 and phi(i-1) were in different groups: the carry below stays a valid bound
    if (l > 0) --l;
  }
}

// LCP in SA order when the final groups are few (periodic traces: a few groups per rotation
// class): a suffix in its predecessor's final group shares >= h_final >= cap symbols, so its capped
// LCP is cap; a group head's comes from lifting over the kept levels (< h_final).  One thread per
// word of the head bitmap; replaces phi + capped Kasai + gather (three passes with random access).
__global__ void __launch_bounds__(256) k_lcp_heads(LiftArgs L, const uint32_t* __restrict__ sa, const uint32_t* __restrict__ heads,
                                                   uint32_t cap, uint32_t* __restrict__ lcp) {
  // a warp takes 32 consecutive bitmap words (1024 positions): runs without heads are written by the
  // whole warp in coalesced 512-byte rows; words with heads are finished by their own lane
  const unsigned lane = lane_id();
  const uint64_t w = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x);
  const uint64_t wbase = (w - lane) * 32;  // the warp's first position
  if (wbase >= L.np) return;
  const uint64_t base = w * 32;
  uint32_t hb = base < L.np ? __ldg(&heads[w]) : 0u;
  const int cnt = base < L.np ? static_cast<int>(umin64(32, L.np - base)) : 0;
  if (cnt < 32 && cnt > 0) hb &= (1u << cnt) - 1u;
  const bool plain = cnt == 32 && hb == 0 && base > 0;  // all 32 positions: LCP = cap
  const unsigned pm = __ballot_sync(0xffffffffu, plain);
  if (pm == 0xffffffffu) {  // the whole warp's 1024 positions are plain: coalesced stores
    const uint4 c4 = make_uint4(cap, cap, cap, cap);
#pragma unroll
    for (int i = 0; i < 8; ++i) __stcs(reinterpret_cast<uint4*>(lcp + wbase) + i * 32 + lane, c4);
    return;
  }
  if (plain) {
    const uint4 c4 = make_uint4(cap, cap, cap, cap);
#pragma unroll
    for (int q = 0; q < 32; q += 4) __stcs(reinterpret_cast<uint4*>(lcp + base + q), c4);
    return;
  }
  for (int q = 0; q < cnt; ++q) {
    const uint64_t j = base + q;
    uint32_t v = cap;
    if (j == 0) {
      v = 0;
    } else if ((hb >> q) & 1u) {
      const uint32_t l = lcp_lift(L, __ldg(&sa[j - 1]), __ldg(&sa[j]), cap);
      v = l < cap ? l : cap;
    }
    lcp[j] = v;
  }
}

__global__ void k_lcp_gather(const uint32_t* __restrict__ sa, const uint32_t* __restrict__ plcp, uint64_t np,
                             uint32_t* __restrict__ lcp) {
  const uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j < np) lcp[j] = j == 0 ? 0u : plcp[sa[j]];
}

// ---------------------------------------------------------------- batched suffix arrays (C4)
struct BatchDevItem {
  const int32_t* tok;
  uint64_t n;
  uint64_t start;  // first position of this trace in the concatenated text
  uint32_t* sa;    // [n + 1] outputs
  uint32_t* lcp;
};

// concatenated text: trace t's tokens, then its separator vmax + t (unique, above every token)
__global__ void k_batch_concat(const BatchDevItem* __restrict__ items, int32_t vmax, int32_t* __restrict__ text) {
  const BatchDevItem it = items[blockIdx.y];
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i <= it.n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    text[it.start + i] = i < it.n ? __ldg(&it.tok[i]) : vmax + static_cast<int32_t>(blockIdx.y);
}

// trace of each suffix in SA order (for the stable partition by trace)
__global__ void k_batch_trace_of(const uint32_t* __restrict__ sa, uint64_t np, const uint64_t* __restrict__ starts, uint32_t nb,
                                 uint32_t* __restrict__ tid, uint32_t* __restrict__ val) {
  const uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= np) return;
  const uint32_t p = sa[j];
  uint32_t lo = 0, hi = nb;  // largest t with starts[t] <= p
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (starts[mid] <= p) lo = mid;
    else hi = mid;
  }
  tid[j] = lo;
  val[j] = p;
}

// the first suffix of every trace slice has no predecessor of its own trace
__global__ void k_batch_phi_heads(const uint32_t* __restrict__ sa, const uint64_t* __restrict__ starts, uint32_t nb,
                                  uint32_t* __restrict__ phi) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nb) phi[sa[starts[t]]] = kNone;
}

__global__ void k_batch_out(const BatchDevItem* __restrict__ items, const uint32_t* __restrict__ sa,
                            const uint32_t* __restrict__ lcp) {
  const BatchDevItem it = items[blockIdx.y];
  for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k <= it.n;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    it.sa[k] = sa[it.start + k] - static_cast<uint32_t>(it.start);
    it.lcp[k] = lcp[it.start + k];
  }
}

}  // namespace

void build_suffix_array(Ctx* c, const int32_t* tokens, uint64_t n, int32_t term, SuffixState& s, bool want_lcp,
                        radix::Scratch& rs, ScanScratch& scan, uint32_t cap, bool known_alphabet) {
  const uint64_t np = n + 1;
  if (np >= 0xFFFFFFFFull) fail(ITT_E_INVALID_ARGUMENT, "pattern-mining: sequence too long for 32-bit suffix indices");
  s.n = n;
  s.np = np;
  s.levels.clear();
  s.level_tags.clear();
  s.level_h.clear();
  s.rounds = 0;
  // alphabet: codes = value - lo over tokens and the terminator
  int32_t lo = known_alphabet ? 0 : term, hi = term;
  if (n && !known_alphabet) {
    DBuf<int> st(c, 3);
    int init[3] = {INT_MAX, INT_MIN, 0};
    h2d(c, st.p, init, 3);
    const unsigned grid = std::min<unsigned>(grid_for(n, 256), c->sm_count * 8);
    launch(c, "sa_token_stats", n * 4.0, k_token_stats, dim3(grid), dim3(256), 0, tokens, n, term, st.p);
    int h[3];
    readback(c, h, st.p, 3);
    if (h[2] != 0) fail(ITT_E_INVALID_CONFIG, "pattern-mining: terminator symbol occurs in the token sequence");
    lo = std::min(lo, h[0]);
    hi = std::max(hi, h[1]);
  }
  const uint64_t sigma = static_cast<uint64_t>(static_cast<int64_t>(hi) - lo) + 1;
  const int cbits = bits_for(sigma - 1);
  const int k = std::max(1, 32 / cbits);
  s.h0 = static_cast<uint32_t>(k);
  s.lo = lo;
  s.text.alloc(c, np);

  // five rotating buffers: the current SA plus the sort's (keys, vals) double buffer
  DBuf<uint32_t> bufs[5];
  for (auto& b : bufs) b.alloc(c, np);
  uint32_t* ka = bufs[0].p;
  uint32_t* va = bufs[1].p;
  uint32_t* kb = bufs[2].p;
  uint32_t* vb = bufs[3].p;
  uint32_t* spare = bufs[4].p;
  const int init_bits = std::min(32, cbits * k);
  // 8-bit digits: the k-gram codes are spread over the whole key, and a 10-bit pass over them (1024
  // bins) measured 1.12 ms per 100M pairs against 0.82 ms for an 8-bit one — 3 wide passes save nothing
  bool a0;
  if (known_alphabet) {  // keys and the sort's digit histograms in one pass (no host check of trivial passes)
    // 25-27-bit keys (e.g. two 13-bit symbols, V ~ 4K): three 9-bit passes instead of four 8-bit ones
    const bool nine = init_bits > 24 && init_bits <= 27 && !std::getenv("ITT_NO_NINE_BIT_INIT");
    const int rb = nine ? 9 : 8;
    const int passes = (init_bits + rb - 1) / rb;
    DBuf<uint32_t> ihist(c, static_cast<size_t>(passes) << rb);
    ihist.zero();
    const radix::IotaLoader<uint32_t> iota{ka};  // positions are generated by the first pass
    if (nine) {
      launch(c, "sa_init_keys", np * 12.0, k_text_keys_hist<9>, dim3(grid_for((np + 3) / 4, 256, c->sm_count * 8)), dim3(256), 0, tokens,
             n, term, lo, cbits, k, passes, s.text.p, ka, static_cast<uint32_t*>(nullptr), ihist.p);
      a0 = radix_sort_pairs<uint32_t, radix::IotaLoader<uint32_t>, 9>(c, ka, va, kb, vb, np, 0, init_bits, rs, ihist.p, &iota,
                                                                      false);
    } else {
      launch(c, "sa_init_keys", np * 12.0, k_text_keys_hist<8>, dim3(grid_for((np + 3) / 4, 256, c->sm_count * 8)), dim3(256), 0, tokens,
             n, term, lo, cbits, k, passes, s.text.p, ka, static_cast<uint32_t*>(nullptr), ihist.p);
      a0 = radix_sort_pairs<uint32_t, radix::IotaLoader<uint32_t>>(c, ka, va, kb, vb, np, 0, init_bits, rs, ihist.p, &iota,
                                                                   /*skip_trivial=*/false);
    }
  } else {
    launch(c, "sa_init_keys", np * 16.0, k_text_keys, dim3(grid_for(np, 256)), dim3(256), 0, tokens, n, term, lo, cbits, k,
           s.text.p, ka, va);
    a0 = radix_sort_pairs<uint32_t>(c, ka, va, kb, vb, np, 0, init_bits, rs, nullptr,
                                    static_cast<const radix::ArrayLoader<uint32_t>*>(nullptr),
                                    /*skip_trivial=*/!known_alphabet);
  }
  uint32_t* keys = a0 ? kb : ka;
  uint32_t* sa = a0 ? vb : va;
  uint32_t* f1 = a0 ? ka : kb;  // free buffers
  uint32_t* f2 = a0 ? va : vb;

  const int max_passes = (bits_for(np - 1) + 7) / 8;
  constexpr size_t kWideBins = 1u << radix::kWideBits;
  DBuf<uint32_t> gstart(c, std::min<uint64_t>(np, kWideGroups));
  const uint64_t rtiles = (np + kRankBlock * kRankItems - 1) / (kRankBlock * kRankItems);
  // two sets of per-round scratch (histograms of the next round's digits, look-back words): the
  // set for round r+1 and the next sort's radix look-back words are zeroed right after round r's
  // rank update is launched, so the only thing between its group-count readback and the next
  // sort is the host itself
  DBuf<uint32_t> hists[2];  // [kMaxPasses * 256 (8-bit layout) | 2 * 1024 (10-bit layout, k_wide_hist)]
  const size_t hist_words = static_cast<size_t>(kMaxPasses) * 256 + 2 * kWideBins;
  for (auto& hb : hists) hb.alloc(c, hist_words);
  ScanScratch scan2;
  ScanScratch* scans[2] = {&scan, &scan2};
  int cur = 0;
  hists[0].zero();
  scans[0]->prepare(c, rtiles);
  uint32_t* hist_p = nullptr;  // the histograms the latest rank update produced
  // group heads in SA order, one byte per 8 positions: written by every round, read by refinement
  DBuf<uint8_t> heads[2];
  for (auto& hb : heads) hb.alloc(c, rtiles * kRankBlock);
  int hc = 0;
  // one rank update into a new level (u16 when the previous group count suggests the ids fit; if
  // they do not, the update runs again into a u32 level: its inputs are untouched)
  DBuf<unsigned long long> gcount(c, 1);
  // the init level by a text-order fill from a (k-gram -> head) table (k_init_fill); ITT_INIT_MAP=0: the scatter
  bool use_init_map = [] {
    const char* e = std::getenv("ITT_INIT_MAP");
    return !(e && *e == '0');
  }();
  DBuf<unsigned long long> init_map;
  const int init_cbits = cbits, init_k = k;
  auto rank_update = [&](const uint32_t* kk, const uint32_t* ss, uintptr_t rank_old, uint32_t h, bool more,
                         uint64_t g_prev, bool heads_mode) -> uint64_t {
    // only where the arrays outgrow L2 (C2's 40 MB levels stay resident: u16 stores there cost
    // more than they save); ITT_NARROW_MIN_N overrides the size threshold (tests)
    const char* ev = std::getenv("ITT_NARROW_MIN_N");
    const uint64_t min_n = ev && *ev ? std::strtoull(ev, nullptr, 10) : (1ull << 24);
    bool narrow = !heads_mode && g_prev <= kNarrowTry && np >= min_n;
    for (;;) {
      s.levels.emplace_back(c, narrow ? (np + 1) / 2 : np);
      const uintptr_t lvl = reinterpret_cast<uintptr_t>(s.levels.back().p) | (narrow ? 1u : 0u);
      ScanScratch& sc = *scans[cur];
      hist_p = hists[cur].p;
      const bool map_init = heads_mode && !rank_old && use_init_map && !narrow;
      if (map_init) {
        init_map.alloc(c, size_t{1} << kInitMapBits);
        init_map.zero();
      }
      if (map_init) {
        gcount.zero();
        launch(c, "sa_rank_update", np * 4.0, k_init_heads, dim3(grid_for((np + kRankItems - 1) / kRankItems, 256)), dim3(256), 0,
               kk, np, heads[hc ^ 1].p, gcount.p, init_map.p, (1u << kInitMapBits) - 1);
      } else if (heads_mode) {
        gcount.zero();
        launch(c, "sa_rank_update", np * (rank_old ? 20.0 : 12.0), k_rank_update<true>,
               dim3(static_cast<unsigned>(rtiles)), dim3(kRankBlock), 0, kk, ss, rank_old, h, np, lvl, hist_p, max_passes,
               nullptr, sc.buf.p + 1, reinterpret_cast<uint32_t*>(sc.buf.p), 0u, heads[hc ^ 1].p, gcount.p,
               map_init ? init_map.p : nullptr, (1u << kInitMapBits) - 1);
      } else {
        launch(c, "sa_rank_update", np * (rank_old ? 20.0 : 12.0), k_rank_update<false>, dim3(static_cast<unsigned>(rtiles)),
               dim3(kRankBlock), 0, kk, ss, rank_old, h, np, lvl, hist_p, max_passes, gstart.p, sc.buf.p + 1,
               reinterpret_cast<uint32_t*>(sc.buf.p), 0u, heads[hc ^ 1].p, nullptr, nullptr, 0u);
      }
      // group count G: the last tile's inclusive word (dense ids) or the head counter, copied out
      // and waited on by event, so the next round's scratch zeroing (queued after the copy) runs
      // while the host wakes up
      ++StageTimer::syncs();
      uint64_t* word = static_cast<uint64_t*>(c->deferred_block()) + 8;  // [0, 64) holds the order verdict
      ITT_CUDA(cudaMemcpyAsync(word, heads_mode ? reinterpret_cast<const uint64_t*>(gcount.p) : sc.buf.p + rtiles, 8,
                               cudaMemcpyDeviceToHost, c->stream));
      ITT_CUDA(cudaEventRecord(c->deferred_ev, c->stream));
      if (more) {
        hists[cur ^ 1].zero();
        scans[cur ^ 1]->prepare(c, rtiles);
        radix_prezero_status(c, rs, np, max_passes, 0);  // a wide sort zeroes its own (rare, larger)
      }
      ITT_CUDA(cudaEventSynchronize(c->deferred_ev));
      uint64_t total = heads_mode ? *word : (*word & kValMask);
      if (map_init) {
        if (total >> 63) {  // more distinct k-grams than the table holds: the scatter after all
          use_init_map = false;
          s.levels.pop_back();
          hists[cur].zero();
          sc.prepare(c, rtiles);
          continue;
        }
        launch(c, "sa_init_fill", np * 8.0, k_init_fill, dim3(grid_for((np + 3) / 4, 256, c->sm_count * 16)), dim3(256), 0,
               s.text.p, np, init_cbits, init_k, init_map.p, (1u << kInitMapBits) - 1, reinterpret_cast<uint32_t*>(lvl));
      }
      if (narrow && total > kNarrowGroups) {  // the ids did not fit 16 bits: redo into u32
        s.levels.pop_back();
        hists[cur].zero();
        sc.prepare(c, rtiles);
        narrow = false;
        continue;
      }
      s.level_tags.push_back(lvl);
      // the level before the previous one is read by nothing queued after this launch
      if (!s.keep_levels && s.levels.size() >= 3) s.levels[s.levels.size() - 3].release();
      cur ^= 1;
      hc ^= 1;
      return total;
    }
  };
  static const int refine_mode = [] {  // ITT_SA_REFINE=0: full rounds only (A/B, tests)
    const char* e = std::getenv("ITT_SA_REFINE");
    return e && *e ? std::atoi(e) : 1;
  }();
  // the first level holds group heads when refinement may follow: a periodic text (few, large
  // k-gram groups) then goes straight into refinement rounds with no dense-to-head conversion
  const bool init_heads = refine_mode > 0 && np < (1ull << 31) && s.h0 < cap;
  uint64_t g = rank_update(keys, sa, 0, 0, s.h0 < cap, 0, init_heads);
  s.level_h.push_back(s.h0);
  uint32_t h = s.h0;  // prefix length the newest level separates
  bool dense = !init_heads;  // the newest level holds dense ids (else group-head positions)
  bool try_refine = init_heads && g * 16 < np;  // then decided after each full round from the groups it added
  int cooldown = 0;
  DBuf<unsigned long long> rcount(c, 4);  // two rounds' (groups, inversions): one round of lookahead
  DBuf<unsigned int> abort_flag(c, 1);    // set by a detect that counted inversions: later rounds' kernels return
  abort_flag.zero();
  DBuf<uint32_t> head_hist;
  ScanScratch rscan[2];
  DBuf<uint64_t> rtot;  // reduce-then-scan apply: per-tile totals, then their exclusive scan
  // Refinement rounds run one round ahead of the host: round r+1's kernels are queued before the
  // host reads round r's verdict (its readback overlaps round r+1 on the device).  A round whose
  // detect counts inversions sets abort_flag, so everything queued after it returns at once; the
  // host then restores the state from before that round and sorts it instead.
  struct Snapshot {
    int hc;
    bool dense;
    uint32_t h;
    int rounds;
    size_t n_levels, n_tags;
    std::vector<uint32_t> level_h;
  };
  struct Pending {
    bool on = false;
    int slot = 0;
    Snapshot before;
  } pend;
  int rslot = 0;
  unsigned long long* host_cnt = static_cast<unsigned long long*>(c->deferred_block()) + 16;  // [16, 20): two rounds' counts
  cudaEvent_t rev[2] = {nullptr, nullptr};
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() {
      for (int i = 0; i < 2; ++i)
        if (e[i]) cudaEventDestroy(e[i]);
    }
  } rev_guard{rev};
  for (auto& e : rev) ITT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  // the pending round's verdict: commit its group count, or undo it and everything after it
  auto resolve = [&]() -> bool {  // true: the pending round had inversions (state restored)
    if (!pend.on) return false;
    pend.on = false;
    ++StageTimer::syncs();
    ITT_CUDA(cudaEventSynchronize(rev[pend.slot]));
    const unsigned long long* cnt = host_cnt + 2 * pend.slot;
    if (cnt[1] == 0) {
      g = cnt[0];
      return false;
    }
    const Snapshot& b = pend.before;
    hc = b.hc, dense = b.dense, h = b.h, s.rounds = b.rounds;
    s.levels.resize(b.n_levels);
    s.level_tags.resize(b.n_tags);
    s.level_h = b.level_h;
    ITT_CUDA(cudaMemsetAsync(abort_flag.p, 0, 4, c->stream));
    cooldown = 2;  // inversions: sort this round, try again two rounds later
    return true;
  };
  // stop when every suffix is alone, or when the groups already separate `cap` symbols (mining
  // never looks deeper than its L_max; see k_plcp for why the capped LCP stays exact below cap)
  for (;;) {
    if (!(g < np && h < cap)) {
      if (!pend.on) break;
      resolve();  // the last speculative round: commit it, or undo it and sort it
      continue;
    }
    if (try_refine && cooldown == 0) {
      // ---- refinement round: no sort when every group is already ordered by its second key
      const uintptr_t rank = s.level_tags.back();
      Snapshot before{hc, dense, h, s.rounds, s.levels.size(), s.level_tags.size(), s.level_h};
      unsigned long long* dcnt = rcount.p + 2 * rslot;
      ITT_CUDA(cudaMemsetAsync(dcnt, 0, 16, c->stream));
      launch(c, "sa_refine_detect", np * 9.125, k_refine_detect, dim3(static_cast<unsigned>(rtiles)), dim3(kRankBlock), 0, sa,
             heads[hc].p, rank, h, np, heads[hc ^ 1].p, dcnt, abort_flag.p);
      const bool full = dense;  // dense ids: every rank changes representation
      // the input level is updated in place unless LCP lifting keeps it: kept levels stay within
      // lift_ratio() of each other, so most refinement rounds skip the level copy (C3: 12 -> 3 copies of
      // 400 MB, step -1.1 ms; lifting repeats a level up to 15 times, lcp_plcp unchanged)
      const size_t nl = s.level_h.size();
      const uint64_t below = nl >= 2 ? s.level_h[nl - 2] : 1;
      const bool dispensable = !s.keep_levels || below * lift_ratio() >= 2ull * h;
      uint32_t* lvl;
      if (!full && dispensable) {  // nothing reads the old level again: update it in place
        lvl = reinterpret_cast<uint32_t*>(rank);
        s.level_h.back() = static_cast<uint32_t>(std::min<uint64_t>(2ull * h, 0xFFFFFFFFull));
      } else {
        s.levels.emplace_back(c, np);
        lvl = s.levels.back().p;
        if (!full) ITT_CUDA(cudaMemcpyAsync(lvl, reinterpret_cast<const uint32_t*>(rank), np * 4, cudaMemcpyDeviceToDevice,
                                            c->stream));
        s.level_tags.push_back(reinterpret_cast<uintptr_t>(lvl));
        s.level_h.push_back(static_cast<uint32_t>(std::min<uint64_t>(2ull * h, 0xFFFFFFFFull)));
        // (older levels are not released here: an undone round may need them)
      }
      const uint64_t atiles = (np + kRankBlock * kApplyItems * kApplyWords - 1) / (kRankBlock * kApplyItems * kApplyWords);
      // ITT_APPLY_RS=1: reduce-then-scan apply (A/B at C3, both with 16-byte bitmap loads: 0.47 ms in three
      // launches vs 0.375 ms for the look-back kernel, whose chain over ~1.5K tiles is short)
      static const bool apply_rs = [] {
        const char* e = std::getenv("ITT_APPLY_RS");
        return e && *e == '1';
      }();
      const uint32_t* h_old = reinterpret_cast<const uint32_t*>(heads[hc].p);
      const uint32_t* h_new = reinterpret_cast<const uint32_t*>(heads[hc ^ 1].p);
      if (apply_rs) {  // tile totals, one-block scan, apply from known prefixes (stream order reuses rtot)
        if (rtot.n < atiles) rtot.alloc(c, atiles);
        launch(c, "sa_refine_totals", np * 0.25, k_refine_totals, dim3(static_cast<unsigned>(atiles)), dim3(kRankBlock), 0,
               h_old, h_new, np, rtot.p, abort_flag.p);
        launch(c, "sa_refine_scan", atiles * 16.0, k_scan_tile_totals<uint64_t, HeadPair>, dim3(1), dim3(1024), 0, rtot.p,
               atiles);
        launch(c, "sa_refine_apply", full ? np * 8.25 : np * 0.25, k_refine_apply<true>, dim3(static_cast<unsigned>(atiles)),
               dim3(kRankBlock), 0, sa, h_old, h_new, np, lvl, full ? 1 : 0, static_cast<uint64_t*>(nullptr),
               static_cast<uint32_t*>(nullptr), abort_flag.p, static_cast<const uint64_t*>(rtot.p));
      } else {
        rscan[rslot].prepare(c, atiles);
        launch(c, "sa_refine_apply", full ? np * 8.25 : np * 0.25, k_refine_apply<false>, dim3(static_cast<unsigned>(atiles)),
               dim3(kRankBlock), 0, sa, h_old, h_new, np, lvl, full ? 1 : 0, rscan[rslot].buf.p + 1,
               reinterpret_cast<uint32_t*>(rscan[rslot].buf.p), abort_flag.p, static_cast<const uint64_t*>(nullptr));
      }
      ITT_CUDA(cudaMemcpyAsync(host_cnt + 2 * rslot, dcnt, 16, cudaMemcpyDeviceToHost, c->stream));
      ITT_CUDA(cudaEventRecord(rev[rslot], c->stream));
      // this round is queued; now the verdict of the one before it
      const bool undone = resolve();
      if (undone) continue;  // state is back before the failed round (this one returned at once on the device)
      hc ^= 1;
      dense = false;
      ++s.rounds;
      pend.on = true;
      pend.slot = rslot;
      pend.before = std::move(before);
      rslot ^= 1;
      if (static_cast<uint64_t>(h) * 2 > 0xFFFFFFFFull) {
        resolve();
        break;
      }
      h *= 2;
      continue;
    }
    if (resolve()) continue;  // a full round needs the pending round's verdict (and its exact state)
    const uintptr_t rank = s.level_tags.back();
    // ---- full round: stable sort of E_j = SA_j - h by rank_h (the E trick) + rank update
    const int b = dense ? bits_for(g - 1) : bits_for(np - 1);
    const EmitLoader ld{sa, rank, np, h};
    // the SA buffer is read by the first pass, so the sort only writes the other buffers:
    // pass 1: loader(sa) -> (f1, f2); pass 2: (f1, f2) -> (kx, vx); pass 3: -> (f1, f2) ...
    uint32_t* kx = keys;  // the previous round's sorted keys are dead now
    uint32_t* vx = spare;
    // 10-bit digits when they save a pass (e.g. the 9-bit ids of a periodic trace: one pass, not two)
    static const bool no_wide = [] {
      const char* e = std::getenv("ITT_NO_WIDE_DIGITS");
      return e && *e && *e != '0';
    }();
    const bool wide = !no_wide && (!dense || g <= kWideGroups) &&
                      (b + radix::kWideBits - 1) / radix::kWideBits < (b + 7) / 8;
    const uint32_t* hist8 = hist_p;
    uint32_t* whist = hist_p + kMaxPasses * 256;
    if (!dense) {  // keys are head positions: digit histograms straight from the level
      const int rb = wide ? radix::kWideBits : 8;
      const int passes = (b + rb - 1) / rb;
      head_hist.alloc(c, static_cast<size_t>(passes) << rb);
      head_hist.zero();
      const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((np + 255) / 256, static_cast<uint64_t>(c->sm_count) * 8));
      const size_t smem = (static_cast<size_t>(passes) << rb) * 4;
      if (wide) {
        smem_optin(c, radix::k_hist<uint32_t, radix::kWideBits>, smem);
        launch(c, "radix_hist", np * 4.0, radix::k_hist<uint32_t, radix::kWideBits>, dim3(grid), dim3(256), smem,
               reinterpret_cast<const uint32_t*>(rank), np, 0, passes, head_hist.p);
        whist = head_hist.p;
      } else {
        smem_optin(c, radix::k_hist<uint32_t, 8>, smem);
        launch(c, "radix_hist", np * 4.0, radix::k_hist<uint32_t, 8>, dim3(grid), dim3(256), smem,
               reinterpret_cast<const uint32_t*>(rank), np, 0, passes, head_hist.p);
        hist8 = head_hist.p;
      }
    } else if (wide) {
      const int pw = (b + radix::kWideBits - 1) / radix::kWideBits;
      launch(c, "sa_wide_hist", g * 8.0, k_wide_hist, dim3(grid_for(g, 256, c->sm_count * 4)), dim3(256), 0, gstart.p, g, np, pw,
             whist);
    }
    const bool alt = wide ? radix_sort_pairs<uint32_t, EmitLoader, radix::kWideBits>(c, kx, vx, f1, f2, np, 0, b, rs, whist,
                                                                                       &ld, false, false)
                          : radix_sort_pairs<uint32_t, EmitLoader>(c, kx, vx, f1, f2, np, 0, b, rs, hist8, &ld, false,
                                                                   /*status_zeroed=*/true);
    uint32_t* nkeys = alt ? f1 : kx;
    uint32_t* nsa = alt ? f2 : vx;
    uint32_t* other_k = alt ? kx : f1;
    uint32_t* other_v = alt ? vx : f2;
    const uint64_t g_old = g;
    g = rank_update(nkeys, nsa, rank, h, static_cast<uint64_t>(h) * 2 < cap, g, false);
    s.level_h.push_back(static_cast<uint32_t>(std::min<uint64_t>(2ull * h, 0xFFFFFFFFull)));
    dense = true;
    ++s.rounds;
    if (cooldown > 0) --cooldown;
    // few new groups: the structure has settled (a periodic trace) — try refinement next round
    try_refine = refine_mode > 0 && np < (1ull << 31) && (g - g_old) * 16 < np;
    // rotate: new SA / keys; the old SA and the unused pair become free
    spare = sa;
    sa = nsa;
    keys = nkeys;
    f1 = other_k;
    f2 = other_v;
    if (static_cast<uint64_t>(h) * 2 > 0xFFFFFFFFull) break;
    h *= 2;
  }
  if (g != np && h < cap) fail(ITT_E_CUDA, "internal: prefix doubling did not converge");
  s.h_final = h;
  s.cap = g == np ? 0xFFFFFFFFu : cap;
  s.sa.alloc(c, np);
  ITT_CUDA(cudaMemcpyAsync(s.sa.p, sa, np * 4, cudaMemcpyDeviceToDevice, c->stream));
  if (!want_lcp) return;

  // ---- LCP
  const std::vector<uintptr_t>& lv = s.level_tags;
  DBuf<uintptr_t> dlv(c, lv.size());
  h2d(c, dlv.p, lv.data(), lv.size());
  DBuf<uint32_t> dlh(c, s.level_h.size());
  h2d(c, dlh.p, s.level_h.data(), s.level_h.size());
  LiftArgs L{s.text.p, np, dlv.p, dlh.p, static_cast<int>(lv.size())};
  const char* hl_env = std::getenv("ITT_LCP_HEADS");  // 0: always phi + capped Kasai (A/B, tests)
  const int heads_lcp = hl_env && *hl_env ? std::atoi(hl_env) : 1;
  if (heads_lcp && g < np && g * kHeadsLcpRatio < np) {  // few final groups: LCP from the head bitmap
    s.lcp.alloc(c, np);
    const uint64_t words = (np + 31) / 32;
    launch(c, "lcp_heads", np * 4.0 + words * 4.0 + g * 8.0, k_lcp_heads, dim3(grid_for(words, 256)), dim3(256), 0, L, s.sa.p,
           reinterpret_cast<const uint32_t*>(heads[hc].p), s.cap, s.lcp.p);
    return;
  }
  DBuf<uint32_t> phi(c, np), plcp(c, np);
  launch(c, "lcp_phi", np * 12.0, k_phi, dim3(grid_for(np, 256)), dim3(256), 0, s.sa.p, np, phi.p);
  const uint64_t chunks = (np + kChunk - 1) / kChunk;
  launch(c, "lcp_plcp", np * 16.0, k_plcp, dim3(grid_for(chunks, 128)), dim3(128), 0, L, phi.p, plcp.p, s.cap);
  s.lcp.alloc(c, np);
  launch(c, "lcp_gather", np * 12.0, k_lcp_gather, dim3(grid_for(np, 256)), dim3(256), 0, s.sa.p, plcp.p, np, s.lcp.p);
  // dlv is released stream-ordered (or lives in the call's arena): no host wait needed
}

}  // namespace itt

namespace itt {

// Suffix arrays + capped LCP of many traces in one doubling sequence (one sort per
// round for all resident traces).  The traces are concatenated with distinct separators vmax + t
// above every token, so each trace's suffixes keep their own relative order (a comparison
// within trace t is decided at the latest by its unique separator, exactly as by its own
// terminator) and LCPs of two suffixes of one trace stop at it.  A stable partition of the
// global suffix array by trace gives every trace its own slice; LCP runs on the partitioned
// array with each slice's head cut off.  cap >= every trace's L_max + 1 (a larger cap than a
// trace needs only makes its LCP more exact: mining is unchanged).
void build_batched_sa(Ctx* c, const std::vector<BatchSAItem>& items, int32_t vmax, uint32_t cap, radix::Scratch& rs,
                      ScanScratch& scan) {
  const uint32_t nb = static_cast<uint32_t>(items.size());
  if (nb == 0) return;
  std::vector<BatchDevItem> host(nb);
  std::vector<uint64_t> starts(nb + 1, 0);
  uint64_t maxn = 0;
  for (uint32_t t = 0; t < nb; ++t) {
    host[t] = BatchDevItem{items[t].tokens, items[t].n, starts[t], items[t].sa, items[t].lcp};
    starts[t + 1] = starts[t] + items[t].n + 1;
    maxn = std::max(maxn, items[t].n + 1);
  }
  const uint64_t np = starts[nb];
  if (np >= 0xFFFFFFFFull) fail(ITT_E_INVALID_ARGUMENT, "pattern-mining: batch too long for 32-bit suffix indices");
  DBuf<BatchDevItem> ditems(c, nb);
  h2d(c, ditems.p, host.data(), nb);
  DBuf<uint64_t> dstarts(c, nb + 1);
  h2d(c, dstarts.p, starts.data(), nb + 1);
  DBuf<int32_t> text(c, np);
  const dim3 g2(std::min<unsigned>(grid_for(maxn, 256), 64), nb);
  launch(c, "sa_batch_concat", np * 8.0, k_batch_concat, g2, dim3(256), 0, ditems.p, vmax, text.p);
  // the last separator is the global terminator
  SuffixState s;
  build_suffix_array(c, text.p, np - 1, vmax + static_cast<int32_t>(nb) - 1, s, false, rs, scan, cap, true);
  text.release();
  // per-trace slices: stable partition of the suffix array by trace
  DBuf<uint32_t> k0(c, np), v0(c, np), k1(c, np), v1(c, np);
  launch(c, "sa_batch_trace", np * 12.0, k_batch_trace_of, dim3(grid_for(np, 256)), dim3(256), 0, s.sa.p, np, dstarts.p, nb,
         k0.p, v0.p);
  const bool alt = radix_sort_pairs<uint32_t>(c, k0.p, v0.p, k1.p, v1.p, np, 0, bits_for(nb > 1 ? nb - 1 : 1), rs, nullptr,
                                              static_cast<const radix::ArrayLoader<uint32_t>*>(nullptr), false);
  ITT_CUDA(cudaMemcpyAsync(s.sa.p, alt ? v1.p : v0.p, np * 4, cudaMemcpyDeviceToDevice, c->stream));
  k0.release(), v0.release(), k1.release(), v1.release();
  // LCP over the partitioned array (sa.cu's phi / capped Kasai / gather), slice heads cut off
  DBuf<uint32_t> phi(c, np), plcp(c, np);
  launch(c, "lcp_phi", np * 12.0, k_phi, dim3(grid_for(np, 256)), dim3(256), 0, s.sa.p, np, phi.p);
  launch(c, "sa_batch_heads", nb * 8.0, k_batch_phi_heads, dim3(grid_for(nb, 256)), dim3(256), 0, s.sa.p, dstarts.p, nb, phi.p);
  const std::vector<uintptr_t>& lv = s.level_tags;
  DBuf<uintptr_t> dlv(c, lv.size());
  h2d(c, dlv.p, lv.data(), lv.size());
  DBuf<uint32_t> dlh(c, s.level_h.size());
  h2d(c, dlh.p, s.level_h.data(), s.level_h.size());
  LiftArgs L{s.text.p, np, dlv.p, dlh.p, static_cast<int>(lv.size())};
  const uint64_t chunks = (np + kChunk - 1) / kChunk;
  launch(c, "lcp_plcp", np * 16.0, k_plcp, dim3(grid_for(chunks, 128)), dim3(128), 0, L, phi.p, plcp.p, s.cap);
  s.lcp.alloc(c, np);
  launch(c, "lcp_gather", np * 12.0, k_lcp_gather, dim3(grid_for(np, 256)), dim3(256), 0, s.sa.p, plcp.p, np, s.lcp.p);
  launch(c, "sa_batch_out", np * 16.0, k_batch_out, g2, dim3(256), 0, ditems.p, s.sa.p, s.lcp.p);
  c->sync();  // the outputs belong to other contexts' calls: complete before they resume
}

}  // namespace itt
