// mine.cu — LCP-interval enumeration (all nearest smaller values) and the repeat mining
// reduction, sm_100a.
//
// enumerate_repeats (mine.hpp:46-60) visits every internal suffix-tree node; here a node is
// the LCP interval represented by its leftmost position k with value l = LCP[k] > 0:
//   lb  = previous j < k with LCP[j] <= l     (if LCP[lb] == l, k is not leftmost: skip)
//   nsv = next j > k with LCP[j] < l          (n' past the end)
//   count = nsv - lb, parent depth = max(LCP[lb], LCP[nsv]), first_leaf = min SA[lb, nsv).
// Searches run in two levels: inside a 1024-wide tile through a shared-memory sparse table
// (binary lifting), across tiles through a sparse table of tile minima plus a binary search
// over the target tile's prefix/suffix minima.
//
// mine_pattern_impl (mine.hpp:75-111) tries epsilon = eps0 * 2^p for p = 0, 1, ... and
// returns the preferred candidate (mine.hpp:69-73) of the first pass that has one.  A
// candidate (count c) first qualifies at pass p(c) = min{p : iters - eps_p + 1 <= c}, so the
// answer is the max over all candidates of (-p(c), len, count, -first_leaf): one reduction
// plus a min-SA pass over the (disjoint) intervals tied on (p, len, count).
#include <algorithm>
#include <cstring>

#include "pipeline.cuh"

namespace itt {

namespace {

constexpr int kTileA = 1024;
constexpr int kLogTileA = 10;
constexpr int kAnsvBlock = 256;

// sparse table over tile minima: st[l * nt + t] = min(tmin[t, t + 2^l))
__global__ void k_sparse_level(uint32_t* st, uint32_t nt, int l) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nt) return;
  const uint32_t half = 1u << (l - 1);
  const uint32_t* prev = st + static_cast<uint64_t>(l - 1) * nt;
  uint32_t v = prev[t];
  if (t + half < nt) v = min(v, prev[t + half]);
  st[static_cast<uint64_t>(l) * nt + t] = v;
}

// all sparse-table levels in one CTA (small tile counts): one launch instead of one per level
__global__ void __launch_bounds__(1024) k_sparse_all(uint32_t* st, uint32_t nt, int levels) {
  for (int l = 1; l < levels; ++l) {
    const uint32_t half = 1u << (l - 1);
    const uint32_t* prev = st + static_cast<uint64_t>(l - 1) * nt;
    uint32_t* cur = st + static_cast<uint64_t>(l) * nt;
    for (uint32_t t = threadIdx.x; t < nt; t += blockDim.x) {
      uint32_t v = prev[t];
      if (t + half < nt) v = min(v, prev[t + half]);
      cur[t] = v;
    }
    __syncthreads();  // level l complete (global writes visible to the block)
  }
}

struct AnsvArgs {
  const uint32_t* lcp;
  const uint32_t* bmin;  // minimum per 32-position block
  const uint32_t* tst;  // tile sparse table
  uint32_t nt;
  int tlevels;
  uint64_t np;
  uint32_t* cnt;
  uint32_t* par;
  uint32_t* lb;
  // list mode (mining): only intervals that can be a mining candidate — count >= 2 and
  // min(LCP, max_len) > parent depth — are appended as (LCP, count, parent, lb); no dense arrays
  uint4* list;
  unsigned int* n_list;
  uint32_t max_len;
  __device__ __forceinline__ void emit(uint64_t k, uint32_t l, uint32_t c, uint32_t p, uint32_t b) const {
    if (!list) {
      cnt[k] = c;
      par[k] = p;
      lb[k] = b;
      return;
    }
    const bool want = c >= 2 && min(l, max_len) > p;
    const unsigned act = __activemask();
    const unsigned w = __ballot_sync(act, want);  // one atomic per warp
    if (!w) return;
    const int leader = __ffs(w) - 1;
    unsigned base = 0;
    if (static_cast<int>(lane_id()) == leader) base = atomicAdd(n_list, static_cast<unsigned>(__popc(w)));
    base = __shfl_sync(act, base, leader);
    if (want) list[base + __popc(w & lanemask_lt())] = make_uint4(l, c, p, b);
  }
};

// last j in tile t with LCP[j] <= thr (the tile's min is known to be <= thr): the last 32-block
// whose minimum qualifies, then the last position in it
__device__ __forceinline__ uint64_t last_le_in_tile(const AnsvArgs& a, uint32_t t, uint32_t thr) {
  const uint64_t t0 = static_cast<uint64_t>(t) * kTileA;
  int b = static_cast<int>((umin64(t0 + kTileA, a.np) - 1 - t0) >> 5);
  while (b > 0 && a.bmin[static_cast<uint64_t>(t) * 32 + b] > thr) --b;
  uint64_t j = umin64(t0 + (static_cast<uint64_t>(b) + 1) * 32, a.np) - 1;
  while (a.lcp[j] > thr) --j;
  return j;
}
// first j in tile t with LCP[j] < thr (the tile's min is known to be < thr)
__device__ __forceinline__ uint64_t first_lt_in_tile(const AnsvArgs& a, uint32_t t, uint32_t thr) {
  const uint64_t t0 = static_cast<uint64_t>(t) * kTileA;
  int b = 0;
  while (a.bmin[static_cast<uint64_t>(t) * 32 + b] >= thr) ++b;
  uint64_t j = t0 + static_cast<uint64_t>(b) * 32;
  while (a.lcp[j] >= thr) ++j;
  return j;
}

// Most positions are decided by their neighbours alone: LCP[k-1] == l (k is not leftmost),
// or LCP[k-1] < l (the PSE is k-1) with LCP[k+1] < l (the NSV is k+1).  Pass 1 (every tile; 4 KiB
// of shared memory, so many tiles overlap their loads) loads the tile with 16-byte loads, writes
// its 32-position block minima and its minimum (what the cross-tile searches need; no separate
// minima pass over the LCP array) and emits every decided position; a tile with undecided ones
// goes on a list.  Pass 2 runs over the listed tiles only, after the tile sparse table exists.
__global__ void __launch_bounds__(kAnsvBlock) k_ansv_fast(AnsvArgs a, uint32_t* __restrict__ bmin, uint32_t* __restrict__ tmin,
                                                          uint32_t* __restrict__ search_tiles, unsigned int* __restrict__ n_search) {
  __shared__ __align__(16) uint32_t st0[kTileA];
  __shared__ uint32_t s_w[kAnsvBlock / 32];
  const uint32_t t = blockIdx.x;
  const uint64_t base = static_cast<uint64_t>(t) * kTileA;
  const uint32_t len = static_cast<uint32_t>(umin64(kTileA, a.np - base));
  const uint32_t x0 = threadIdx.x * 4;  // 4 consecutive positions per thread
  uint4 v = make_uint4(~0u, ~0u, ~0u, ~0u);
  if (x0 + 4 <= len) {
    v = __ldcs(reinterpret_cast<const uint4*>(a.lcp + base + x0));
  } else {
    if (x0 < len) v.x = a.lcp[base + x0];
    if (x0 + 1 < len) v.y = a.lcp[base + x0 + 1];
    if (x0 + 2 < len) v.z = a.lcp[base + x0 + 2];
  }
  *reinterpret_cast<uint4*>(&st0[x0]) = v;
  uint32_t m = min(min(v.x, v.y), min(v.z, v.w));  // 32-position block minima: 8 threads each
  m = min(m, __shfl_xor_sync(0xffffffffu, m, 1));
  m = min(m, __shfl_xor_sync(0xffffffffu, m, 2));
  m = min(m, __shfl_xor_sync(0xffffffffu, m, 4));
  if ((threadIdx.x & 7) == 0) bmin[static_cast<uint64_t>(t) * 32 + (threadIdx.x >> 3)] = m;
  const uint32_t wm = __reduce_min_sync(0xffffffffu, m);
  if (lane_id() == 0) s_w[threadIdx.x >> 5] = wm;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t tm = s_w[0];
    for (int w = 1; w < kAnsvBlock / 32; ++w) tm = min(tm, s_w[w]);
    tmin[t] = tm;
  }
  bool any_search = false;
  for (uint32_t x = threadIdx.x; x < len; x += kAnsvBlock) {
    const uint64_t k = base + x;
    const uint32_t l = st0[x];
    uint32_t cnt = 0, par = 0, lbv = 0;
    bool search = false;
    if (k > 0 && l > 0) {
      const uint32_t lp = x > 0 ? st0[x - 1] : a.lcp[k - 1];
      if (lp > l) {
        search = true;
      } else if (lp < l) {  // leftmost, PSE = k - 1
        const uint32_t ln = k + 1 >= a.np ? 0u : (x + 1 < len ? st0[x + 1] : a.lcp[k + 1]);
        if (ln < l) {
          cnt = 2;  // [k - 1, k + 1)
          par = max(lp, ln);
          lbv = static_cast<uint32_t>(k - 1);
        } else {
          search = true;
        }
      }
    }
    any_search |= search;
    if (!search) a.emit(k, l, cnt, par, lbv);
  }
  if (__syncthreads_or(any_search) && threadIdx.x == 0) search_tiles[atomicAdd(n_search, 1u)] = t;
}

__global__ void __launch_bounds__(kAnsvBlock) k_ansv_search(AnsvArgs a, const uint32_t* __restrict__ search_tiles,
                                                            const unsigned int* __restrict__ n_search) {
  __shared__ uint32_t st[kLogTileA][kTileA];  // st[l][x] = min(LCP[x, x + 2^l)) within the tile
  const uint32_t ns = *n_search;
  for (uint32_t qt = blockIdx.x; qt < ns; qt += gridDim.x) {
  const uint32_t t = search_tiles[qt];
  const uint64_t base = static_cast<uint64_t>(t) * kTileA;
  const uint32_t len = static_cast<uint32_t>(umin64(kTileA, a.np - base));
  __syncthreads();  // the previous tile's table is consumed
  for (uint32_t x = threadIdx.x; x < kTileA; x += kAnsvBlock) st[0][x] = x < len ? a.lcp[base + x] : 0xFFFFFFFFu;
  __syncthreads();
  for (int l = 1; l < kLogTileA; ++l) {
    const uint32_t half = 1u << (l - 1);
    for (uint32_t x = threadIdx.x; x < kTileA; x += kAnsvBlock)
      st[l][x] = x + half < kTileA ? min(st[l - 1][x], st[l - 1][x + half]) : st[l - 1][x];
    __syncthreads();
  }
    for (uint32_t x = threadIdx.x; x < len; x += kAnsvBlock) {
      const uint64_t k = base + x;
      const uint32_t l = st[0][x];
      if (k == 0 || l == 0) continue;
      {  // the positions the first pass decided
        const uint32_t lp = x > 0 ? st[0][x - 1] : a.lcp[k - 1];
        if (lp == l) continue;
        if (lp < l) {
          const uint32_t ln = k + 1 >= a.np ? 0u : (x + 1 < len ? st[0][x + 1] : a.lcp[k + 1]);
          if (ln < l) continue;
        }
      }
      uint32_t cnt = 0, par = 0, lbv = 0;
      {
        // ---- previous j < k with LCP[j] <= l
        uint32_t pos = x;
  #pragma unroll
        for (int lv = kLogTileA - 1; lv >= 0; --lv) {
          const uint32_t w = 1u << lv;
          if (pos >= w && st[lv][pos - w] > l) pos -= w;
        }
        uint64_t pse;
        if (pos > 0) {
          pse = base + pos - 1;
        } else {  // cross-tile: last tile before t whose min <= l (tile 0 holds LCP[0] = 0)
          uint32_t tp = t;
          for (int lv = a.tlevels - 1; lv >= 0; --lv) {
            const uint32_t w = 1u << lv;
            if (tp >= w && a.tst[static_cast<uint64_t>(lv) * a.nt + tp - w] > l) tp -= w;
          }
          pse = last_le_in_tile(a, tp - 1, l);
        }
        const uint32_t lp = pse - base < kTileA && pse >= base ? st[0][pse - base] : a.lcp[pse];
        if (lp < l) {  // k is the leftmost position of its interval
          // ---- next j > k with LCP[j] < l
          uint32_t q = x + 1;
  #pragma unroll
          for (int lv = kLogTileA - 1; lv >= 0; --lv) {
            const uint32_t w = 1u << lv;
            if (q + w <= len && st[lv][q] >= l) q += w;
          }
          uint64_t nsv;
          uint32_t ln = 0;
          if (q < len) {
            nsv = base + q;
            ln = st[0][q];
          } else {
            uint32_t tn = t + 1;
            for (int lv = a.tlevels - 1; lv >= 0; --lv) {
              const uint32_t w = 1u << lv;
              if (tn + w <= a.nt && a.tst[static_cast<uint64_t>(lv) * a.nt + tn] >= l) tn += w;
            }
            if (tn < a.nt) {
              nsv = first_lt_in_tile(a, tn, l);
              ln = a.lcp[nsv];
            } else {
              nsv = a.np;
              ln = 0;
            }
          }
          cnt = static_cast<uint32_t>(nsv - pse);
          par = max(lp, ln);
          lbv = static_cast<uint32_t>(pse);
        }
      }
      a.emit(k, l, cnt, par, lbv);
    }
  }
}

// ---------------------------------------------------------------- mining reduction
struct MineArgs {
  const uint32_t* lcp;
  const uint32_t* cnt;
  const uint32_t* par;
  uint64_t np;
  int64_t iters;
  int64_t max_len;
  int npass;
  int64_t min_count[64];  // iters - eps_p + 1 per pass
};
struct Best {
  unsigned long long hi;  // (63 - pass) << 32 | len
  unsigned long long lo;  // count
};
__device__ __forceinline__ bool better(const Best& a, const Best& b) { return a.hi != b.hi ? a.hi > b.hi : a.lo > b.lo; }

__device__ __forceinline__ bool candidate_key(const MineArgs& a, uint64_t k, Best& out) {
  const uint32_t c = a.cnt[k];
  if (c == 0) return false;
  const uint32_t l = a.lcp[k];
  const int64_t len = imin64(static_cast<int64_t>(l), a.max_len);
  if (len <= static_cast<int64_t>(a.par[k])) return false;  // mid-edge truncation stays below the node
  if (static_cast<int64_t>(c) > a.iters) return false;
  int p = 0;
  while (p < a.npass && static_cast<int64_t>(c) < a.min_count[p]) ++p;
  if (p == a.npass) return false;
  out.hi = (static_cast<unsigned long long>(63 - p) << 32) | static_cast<unsigned long long>(len);
  out.lo = c;
  return true;
}

__global__ void __launch_bounds__(256) k_mine_reduce(MineArgs a, Best* block_best) {
  Best b{0, 0};
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < a.np; k += stride) {
    Best x;
    if (candidate_key(a, k, x) && better(x, b)) b = x;
  }
  for (int o = 16; o > 0; o >>= 1) {
    Best y{__shfl_xor_sync(0xffffffffu, b.hi, o), __shfl_xor_sync(0xffffffffu, b.lo, o)};
    if (better(y, b)) b = y;
  }
  __shared__ Best sw[8];
  if (lane_id() == 0) sw[threadIdx.x >> 5] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w)
      if (better(sw[w], b)) b = sw[w];
    block_best[blockIdx.x] = b;
  }
}

// the same over an interval list (lcp_intervals in list mode): entries (LCP, count, parent, lb)
__device__ __forceinline__ bool candidate_entry(const MineArgs& a, const uint4& e, Best& out) {
  const int64_t len = imin64(static_cast<int64_t>(e.x), a.max_len);
  if (len <= static_cast<int64_t>(e.z)) return false;
  const uint32_t c = e.y;
  if (static_cast<int64_t>(c) > a.iters) return false;
  int p = 0;
  while (p < a.npass && static_cast<int64_t>(c) < a.min_count[p]) ++p;
  if (p == a.npass) return false;
  out.hi = (static_cast<unsigned long long>(63 - p) << 32) | static_cast<unsigned long long>(len);
  out.lo = c;
  return true;
}
__global__ void __launch_bounds__(256) k_mine_reduce_list(MineArgs a, const uint4* __restrict__ list,
                                                          const unsigned int* __restrict__ n_list, Best* block_best) {
  Best b{0, 0};
  const uint64_t nl = *n_list;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nl; i += stride) {
    Best x;
    if (candidate_entry(a, list[i], x) && better(x, b)) b = x;
  }
  for (int o = 16; o > 0; o >>= 1) {
    Best y{__shfl_xor_sync(0xffffffffu, b.hi, o), __shfl_xor_sync(0xffffffffu, b.lo, o)};
    if (better(y, b)) b = y;
  }
  __shared__ Best sw[8];
  if (lane_id() == 0) sw[threadIdx.x >> 5] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w)
      if (better(sw[w], b)) b = sw[w];
    block_best[blockIdx.x] = b;
  }
}

__global__ void k_best_final(const Best* bb, uint32_t nb, Best* out) {
  Best b{0, 0};
  for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x)
    if (better(bb[i], b)) b = bb[i];
  for (int o = 16; o > 0; o >>= 1) {
    Best y{__shfl_xor_sync(0xffffffffu, b.hi, o), __shfl_xor_sync(0xffffffffu, b.lo, o)};
    if (better(y, b)) b = y;
  }
  if (threadIdx.x == 0) *out = b;
}

// min SA over the intervals tied on the winning (pass, len, count): they are disjoint.  Small
// intervals are reduced by the thread that finds them; wide ones are listed for k_tied_wide.
constexpr uint32_t kTiedSerial = 256;
constexpr uint32_t kTiedChunk = 4096;
__global__ void __launch_bounds__(256) k_tied_min_sa(MineArgs a, const uint32_t* __restrict__ lb,
                                                     const uint32_t* __restrict__ sa, const Best* best,
                                                     unsigned int* __restrict__ result, uint32_t* __restrict__ wide,
                                                     unsigned int* __restrict__ n_wide) {
  const Best w = *best;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < a.np; k += stride) {
    Best x;
    if (!candidate_key(a, k, x) || x.hi != w.hi || x.lo != w.lo) continue;
    const uint32_t l0 = lb[k], c = a.cnt[k];
    if (c > kTiedSerial) {
      const unsigned q = atomicAdd(n_wide, 1u);
      wide[2 * q] = l0;
      wide[2 * q + 1] = c;
      continue;
    }
    uint32_t m = 0xFFFFFFFFu;
    for (uint32_t q = 0; q < c; ++q) m = min(m, sa[l0 + q]);
    atomicMin(result, m);
  }
}

__global__ void __launch_bounds__(256) k_tied_min_sa_list(MineArgs a, const uint4* __restrict__ list,
                                                          const unsigned int* __restrict__ n_list, const uint32_t* __restrict__ sa,
                                                          const Best* best, unsigned int* __restrict__ result,
                                                          uint32_t* __restrict__ wide, unsigned int* __restrict__ n_wide) {
  const Best w = *best;
  const uint64_t nl = *n_list;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nl; i += stride) {
    const uint4 e = list[i];
    Best x;
    if (!candidate_entry(a, e, x) || x.hi != w.hi || x.lo != w.lo) continue;
    const uint32_t l0 = e.w, c = e.y;
    if (c > kTiedSerial) {
      const unsigned q = atomicAdd(n_wide, 1u);
      wide[2 * q] = l0;
      wide[2 * q + 1] = c;
      continue;
    }
    uint32_t m = 0xFFFFFFFFu;
    for (uint32_t q = 0; q < c; ++q) m = min(m, sa[l0 + q]);
    atomicMin(result, m);
  }
}

// wide tied intervals in kTiedChunk pieces spread over all blocks
__global__ void __launch_bounds__(256) k_tied_wide(const uint32_t* __restrict__ wide, const unsigned int* __restrict__ n_wide,
                                                   const uint32_t* __restrict__ sa, unsigned int* __restrict__ result) {
  const unsigned nw = *n_wide;
  uint32_t m = 0xFFFFFFFFu;
  uint64_t chunk0 = 0;  // global chunk numbering across the listed intervals
  for (unsigned e = 0; e < nw; ++e) {
    const uint32_t l0 = wide[2 * e], c = wide[2 * e + 1];
    const uint64_t nch = (c + kTiedChunk - 1) / kTiedChunk;
    for (uint64_t ch = (blockIdx.x + gridDim.x - chunk0 % gridDim.x) % gridDim.x; ch < nch; ch += gridDim.x) {
      const uint32_t b = l0 + static_cast<uint32_t>(ch * kTiedChunk);
      const uint32_t end = l0 + min(c, static_cast<uint32_t>((ch + 1) * kTiedChunk));
      for (uint32_t q = b + threadIdx.x; q < end; q += blockDim.x) m = min(m, sa[q]);
    }
    chunk0 += nch;
  }
  for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane_id() == 0 && m != 0xFFFFFFFFu) atomicMin(result, m);
}

// Result of one loop in one buffer (a single host round trip): the winning key, the pattern's
// first occurrence and its tokens (text codes + lo).  out = [best.hi, best.lo, start, tokens...]
__global__ void k_pattern_out(const Best* __restrict__ best, const unsigned int* __restrict__ start,
                              const int32_t* __restrict__ text, int32_t lo, uint32_t max_out,
                              uint32_t* __restrict__ out) {
  const Best b = *best;
  const uint32_t st = *start;
  const uint32_t len = static_cast<uint32_t>(b.hi & 0xFFFFFFFFull);
  if (threadIdx.x == 0) {
    reinterpret_cast<unsigned long long*>(out)[0] = b.hi;
    reinterpret_cast<unsigned long long*>(out)[1] = b.lo;
    out[4] = st;
    out[5] = 0;
  }
  if (b.hi == 0 && b.lo == 0) return;
  for (uint32_t q = threadIdx.x; q < len && q < max_out; q += blockDim.x)
    out[6 + q] = static_cast<uint32_t>(text[st + q] + lo);
}

}  // namespace

void lcp_intervals(Ctx* c, const SuffixState& s, IntervalState& iv, uint32_t list_max_len) {
  const uint64_t np = s.np;
  const uint32_t nt = static_cast<uint32_t>((np + kTileA - 1) / kTileA);
  DBuf<uint32_t> bmin(c, static_cast<size_t>(nt) * 32);
  int tlevels = 1;
  while ((1u << tlevels) <= nt) ++tlevels;
  DBuf<uint32_t> tst(c, static_cast<size_t>(tlevels) * nt);
  DBuf<uint32_t> stiles(c, nt);
  DBuf<unsigned int> nsearch(c, 1);
  AnsvArgs a{s.lcp.p, bmin.p, tst.p, nt, tlevels, np, nullptr, nullptr, nullptr, nullptr, nullptr, 0};
  Fills fz(c);
  fz.add(nsearch.p, 4, 0);
  if (list_max_len) {  // mining: the candidate intervals only (no host sync: the kernels read the count)
    iv.list.alloc(c, np);
    iv.n_list.alloc(c, 1);
    fz.add(iv.n_list.p, 4, 0);
    a.list = iv.list.p;
    a.n_list = iv.n_list.p;
    a.max_len = list_max_len;
  } else {
    iv.cnt.alloc(c, np);
    iv.par.alloc(c, np);
    iv.lb.alloc(c, np);
    a.cnt = iv.cnt.p, a.par = iv.par.p, a.lb = iv.lb.p;
  }
  fz.flush();
  launch(c, "ansv_intervals", np * (list_max_len ? 4.0 : 16.0) + nt * 132.0, k_ansv_fast, dim3(nt), dim3(kAnsvBlock), 0, a,
         bmin.p, tst.p, stiles.p, nsearch.p);
  if (nt <= 65536) {
    if (tlevels > 1)
      launch(c, "ansv_sparse", nt * 12.0 * (tlevels - 1), k_sparse_all, dim3(1), dim3(1024), 0, tst.p, nt, tlevels);
  } else {
    for (int l = 1; l < tlevels; ++l)
      launch(c, "ansv_sparse", nt * 12.0, k_sparse_level, dim3(grid_for(nt, 256)), dim3(256), 0, tst.p, nt, l);
  }
  launch(c, "ansv_search", 0.0, k_ansv_search, dim3(std::min<uint32_t>(nt, c->sm_count * 5)), dim3(kAnsvBlock), 0, a,
         stiles.p, nsearch.p);
}

MinedPattern mine_one(Ctx* c, const SuffixState& s, const IntervalState& iv, const itt_mining_cfg& cfg,
                      const std::string& label) {
  MinedPattern r;
  const int64_t iters = cfg.iterations, eps0 = cfg.epsilon0;
  const int64_t n = static_cast<int64_t>(s.n);
  if (iters < 2 || eps0 < 1 || eps0 >= iters) {
    r.status = ITT_E_INVALID_ITERATION_COUNT;
    r.error = "pattern-mining" + label + ": need iterations >= 2 and 1 <= epsilon0 < iterations (got iterations=" +
              std::to_string(iters) + ", epsilon0=" + std::to_string(eps0) + ")";
    return r;
  }
  if (n < iters) {
    r.status = ITT_E_INVALID_ITERATION_COUNT;
    r.error = "pattern-mining" + label + ": sequence of " + std::to_string(n) + " operations cannot contain " +
              std::to_string(iters) + " iterations";
    return r;
  }
  const int64_t cap = cfg.epsilon_cap > 0 ? cfg.epsilon_cap : iters;
  const int64_t max_len = (n - 1) / iters;  // mine.hpp:64-67
  MineArgs a{};
  a.lcp = s.lcp.p;
  a.cnt = iv.cnt.p;
  a.par = iv.par.p;
  a.np = s.np;
  a.iters = iters;
  a.max_len = max_len;
  std::vector<int64_t> eps;
  for (int64_t e = eps0; e < cap && eps.size() < 63; e *= 2) eps.push_back(e);
  a.npass = static_cast<int>(eps.size());
  for (size_t p = 0; p < eps.size(); ++p) a.min_count[p] = iters - eps[p] + 1;
  auto no_pattern = [&]() {
    r.status = ITT_E_NO_PATTERN_FOUND;
    r.error = "pattern-mining" + label +
              ": no repeated substring satisfies the repetition and length criteria for iterations=" +
              std::to_string(iters) + " (epsilon exhausted at cap " + std::to_string(cap) +
              "); the trace may not be iterative at the declared count";
  };
  if (max_len < 1 || a.npass == 0) {  // enumerate_repeats is empty (mine.hpp:50)
    no_pattern();
    return r;
  }
  const unsigned grid = std::min<unsigned>(grid_for(s.np, 256), c->sm_count * 4);
  DBuf<Best> bb(c, grid + 1);
  if (iv.list.p)
    launch(c, "mine_reduce", 0.0, k_mine_reduce_list, dim3(grid), dim3(256), 0, a, iv.list.p, iv.n_list.p, bb.p);
  else
    launch(c, "mine_reduce", s.np * 12.0, k_mine_reduce, dim3(grid), dim3(256), 0, a, bb.p);
  launch(c, "mine_final", grid * 16.0, k_best_final, dim3(1), dim3(32), 0, bb.p, grid, bb.p + grid);
  // the tie-break kernels run whether or not a candidate exists (no candidate key equals the
  // empty key), so the whole result comes back in one round trip
  DBuf<unsigned int> start(c, 2);
  Fills fz(c);  // (min SA = none, wide count = 0) in one launch
  fz.add(start.p, 4, 0xFF);
  fz.add(start.p + 1, 4, 0);
  fz.flush();
  const size_t wide_cap = s.np / (kTiedSerial + 1) + 2;  // disjoint intervals wider than kTiedSerial
  DBuf<uint32_t> wide(c, 2 * wide_cap);
  if (iv.list.p)
    launch(c, "mine_tied_min_sa", 0.0, k_tied_min_sa_list, dim3(grid), dim3(256), 0, a, iv.list.p, iv.n_list.p, s.sa.p,
           bb.p + grid, start.p, wide.p, start.p + 1);
  else
    launch(c, "mine_tied_min_sa", s.np * 12.0, k_tied_min_sa, dim3(grid), dim3(256), 0, a, iv.lb.p, s.sa.p, bb.p + grid,
           start.p, wide.p, start.p + 1);
  launch(c, "mine_tied_wide", 0.0, k_tied_wide, dim3(static_cast<unsigned>(c->sm_count) * 4), dim3(256), 0, wide.p, start.p + 1,
         s.sa.p, start.p);
  constexpr uint32_t kFirstRead = 16384;  // pattern tokens read back with the key; longer ones need a second trip
  const uint32_t max_out = static_cast<uint32_t>(std::min<int64_t>(max_len, 0xFFFFFFF));
  DBuf<uint32_t> res(c, 6 + static_cast<size_t>(max_out));
  launch(c, "mine_pattern_out", max_out * 8.0, k_pattern_out, dim3(1), dim3(256), 0, bb.p + grid, start.p, s.text.p, s.lo,
         max_out, res.p);
  std::vector<uint32_t> h(6 + std::min(max_out, kFirstRead));
  readback(c, h.data(), res.p, h.size());
  Best best;
  std::memcpy(&best.hi, &h[0], 8);
  std::memcpy(&best.lo, &h[2], 8);
  if (best.hi == 0 && best.lo == 0) {
    no_pattern();
    return r;
  }
  const uint32_t st = h[4];
  const int64_t len = static_cast<int64_t>(best.hi & 0xFFFFFFFFull);
  const int pass = 63 - static_cast<int>(best.hi >> 32);
  r.count = static_cast<int64_t>(best.lo);
  r.first_token = st;
  r.epsilon_used = eps[static_cast<size_t>(pass)];
  r.tokens.resize(static_cast<size_t>(len));
  if (len > static_cast<int64_t>(kFirstRead)) {
    std::vector<uint32_t> all(static_cast<size_t>(len));
    readback(c, all.data(), res.p + 6, static_cast<size_t>(len));
    std::memcpy(r.tokens.data(), all.data(), static_cast<size_t>(len) * 4);
  } else {
    std::memcpy(r.tokens.data(), &h[6], static_cast<size_t>(len) * 4);
  }
  return r;
}

std::vector<MinedPattern> mine_loops(Ctx* c, const SuffixState& s, const IntervalState& iv,
                                     const std::vector<itt_mining_cfg>& loops, bool multi) {
  std::vector<MinedPattern> out;
  for (size_t k = 0; k < loops.size(); ++k) {
    const std::string label = multi ? " (loop " + std::to_string(k + 1) + ")" : "";
    out.push_back(mine_one(c, s, iv, loops[k], label));
    if (out.back().status) return out;
  }
  return out;
}

}  // namespace itt
