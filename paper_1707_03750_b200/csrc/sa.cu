// sa.cu — suffix array by prefix doubling + LCP by phi / chunked Kasai, sm_100a.
//
// Replaces the Ukkonen suffix tree (suffix_tree.hpp:21-190, built by mine.hpp:38-40): the
// tree's leaves in child-key order are the suffixes of tokens+[terminator] in sorted
// order (SA), internal nodes are the LCP intervals, depth = LCP value, leaf_count =
// interval width, first_leaf = min SA over the interval.
//
// Doubling (h -> 2h) with group-head ranks:
//   1. init: key_i = the first k symbols of suffix i packed into 32 bits (k = 32 / bits per
//      symbol), one onesweep sort, ranks = index of the first suffix of each key group.
//   2. round h: the sequence E_j = SA_j - h (or SA_j + n' - h for SA_j < h, which are
//      singletons) lists every suffix i ordered by the rank of i + h.  A STABLE sort of E
//      by rank_i (b = log2 n' bits, ceil(b/8) passes instead of 2b/8) yields SA ordered by
//      (rank_i, rank_{i+h}).  New ranks = max-scan of group-start flags (decoupled look-back).
//   3. stop when every group is a singleton.
// Every round's rank array is kept: level r identifies equal (k * 2^r)-prefixes, so
// lcp(i, j) = sum of the levels where the ranks agree (binary lifting) + < k direct compares.
//
// LCP: phi[SA_j] = SA_{j-1}; PLCP by Kasai in chunks of kChunk text positions per thread
// (each chunk restarts at l = 0); any direct comparison longer than kLiftAfter symbols
// switches to lifting, so periodic traces (Sum LCP ~ n^2/2) cost O(n log n) at worst;
// LCP_j = PLCP[SA_j].
#include <algorithm>

#include "pipeline.cuh"

namespace itt {

namespace {

constexpr int kChunk = 64;
constexpr int kLiftAfter = 24;
constexpr int kRankBlock = 256;
constexpr int kRankItems = 8;

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

// codes: tokens - lo, terminator appended at n
__global__ void k_text_codes(const int32_t* __restrict__ tok, uint64_t n, int32_t term, int32_t lo, int32_t* __restrict__ text) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) text[i] = tok[i] - lo;
  else if (i == n) text[n] = term - lo;
}

__global__ void k_init_keys(const int32_t* __restrict__ text, uint64_t np, int bits, int k, uint32_t* __restrict__ keys,
                            uint32_t* __restrict__ vals) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= np) return;
  uint32_t key = 0;
  for (int q = 0; q < k; ++q) {
    const uint32_t c = i + q < np ? static_cast<uint32_t>(text[i + q]) : 0u;  // padding past the unique terminator is never decisive
    key = (key << bits) | c;
  }
  keys[i] = key;
  vals[i] = static_cast<uint32_t>(i);
}

// E_j: suffix whose (i + h) is SA_j; the h suffixes with i + h >= n' (already singletons) take
// the slots of SA_j < h.  key = rank_i.
__global__ void k_emit(const uint32_t* __restrict__ sa, const uint32_t* __restrict__ rank, uint64_t np, uint32_t h,
                       uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= np) return;
  const uint32_t x = sa[j];
  const uint32_t i = x >= h ? x - h : static_cast<uint32_t>(x + np - h);
  keys[j] = rank[i];
  vals[j] = i;
}

__global__ void k_second_key(const uint32_t* __restrict__ sa, const uint32_t* __restrict__ rank, uint64_t np, uint32_t h,
                             uint32_t* __restrict__ r2) {
  const uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= np) return;
  const uint64_t x = static_cast<uint64_t>(sa[j]) + h;
  r2[j] = x < np ? rank[x] : kNone;
}

// New group-head ranks: flag_j = (key, r2) differs from j-1; head_j = max-scan(flag ? j : 0);
// rank_new[SA_j] = head_j.  r2 may be null (init round).  groups += number of flags.
__global__ void __launch_bounds__(kRankBlock) k_rank_update(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ r2,
                                                            const uint32_t* __restrict__ sa, uint64_t np,
                                                            uint32_t* __restrict__ rank_new, uint64_t* status, uint32_t* counter,
                                                            unsigned long long* groups) {
  __shared__ uint32_t s_warp[kRankBlock / 32];
  __shared__ uint32_t s_tile, s_prefix;
  __shared__ uint32_t s_cnt;
  if (threadIdx.x == 0) {
    s_tile = atomicAdd(counter, 1u);
    s_cnt = 0;
  }
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t base = static_cast<uint64_t>(tile) * (kRankBlock * kRankItems) + static_cast<uint64_t>(threadIdx.x) * kRankItems;
  uint32_t head[kRankItems];
  uint32_t run = 0, flags = 0;
  uint32_t pk = 0, pr = 0;
  if (base < np && base > 0) {
    pk = keys[base - 1];
    pr = r2 ? r2[base - 1] : 0;
  }
#pragma unroll
  for (int q = 0; q < kRankItems; ++q) {
    const uint64_t j = base + q;
    uint32_t v = 0;
    if (j < np) {
      const uint32_t k = keys[j];
      const uint32_t r = r2 ? r2[j] : 0;
      const bool f = j == 0 || k != pk || r != pr;
      flags += f;
      v = f ? static_cast<uint32_t>(j) : 0u;
      pk = k;
      pr = r;
    }
    run = max(run, v);
    head[q] = run;
  }
  uint32_t total;
  const uint32_t texcl = block_exclusive_scan<uint32_t, MaxOp<uint32_t>, kRankBlock>(run, MaxOp<uint32_t>(), &total, s_warp);
  if (threadIdx.x < 32) {
    const uint32_t p = tile_lookback<uint32_t, MaxOp<uint32_t>>(status, tile, total, MaxOp<uint32_t>());
    if (threadIdx.x == 0) s_prefix = p;
  }
  // flags count: warp reduce then one shared atomic per warp
  uint32_t fc = flags;
  for (int o = 16; o > 0; o >>= 1) fc += __shfl_xor_sync(0xffffffffu, fc, o);
  if (lane_id() == 0 && fc) atomicAdd(&s_cnt, fc);
  __syncthreads();
  const uint32_t pre = max(s_prefix, texcl);
#pragma unroll
  for (int q = 0; q < kRankItems; ++q) {
    const uint64_t j = base + q;
    if (j < np) rank_new[sa[j]] = max(pre, head[q]);
  }
  if (threadIdx.x == 0 && s_cnt) atomicAdd(groups, static_cast<unsigned long long>(s_cnt));
}

// ---------------------------------------------------------------- LCP
__global__ void k_phi(const uint32_t* __restrict__ sa, uint64_t np, uint32_t* __restrict__ phi) {
  const uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j < np) phi[sa[j]] = j > 0 ? sa[j - 1] : kNone;
}

struct LiftArgs {
  const int32_t* text;
  uint64_t np;
  const uint32_t* const* levels;  // device array of level pointers
  int nlev;
  uint32_t h0;
};

// lcp of suffixes a != b (both < np) by binary lifting over the doubling levels
__device__ __forceinline__ uint32_t lcp_lift(const LiftArgs& L, uint64_t a, uint64_t b) {
  uint32_t acc = 0;
  for (int r = L.nlev - 1; r >= 0; --r) {
    const uint32_t* lv = L.levels[r];
    if (a < L.np && b < L.np && __ldg(&lv[a]) == __ldg(&lv[b])) {
      const uint32_t hr = L.h0 << r;
      a += hr;
      b += hr;
      acc += hr;
    }
  }
  while (a < L.np && b < L.np && __ldg(&L.text[a]) == __ldg(&L.text[b])) ++a, ++b, ++acc;
  return acc;
}

__global__ void k_plcp(LiftArgs L, const uint32_t* __restrict__ phi, uint32_t* __restrict__ plcp) {
  const uint64_t i0 = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * kChunk;
  if (i0 >= L.np) return;
  const uint64_t i1 = min(i0 + kChunk, L.np);
  uint32_t l = 0;
  for (uint64_t i = i0; i < i1; ++i) {
    const uint32_t p = phi[i];
    if (p == kNone) {
      plcp[i] = 0;
      l = 0;
      continue;
    }
    int steps = 0;
    bool lifted = false;
    while (i + l < L.np && p + l < L.np && __ldg(&L.text[i + l]) == __ldg(&L.text[p + l])) {
      ++l;
      if (++steps == kLiftAfter) {
        l += lcp_lift(L, i + l, static_cast<uint64_t>(p) + l);
        lifted = true;
        break;
      }
    }
    (void)lifted;
    plcp[i] = l;
    if (l > 0) --l;
  }
}

__global__ void k_lcp_gather(const uint32_t* __restrict__ sa, const uint32_t* __restrict__ plcp, uint64_t np,
                             uint32_t* __restrict__ lcp) {
  const uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j < np) lcp[j] = j == 0 ? 0u : plcp[sa[j]];
}

}  // namespace

void build_suffix_array(Ctx* c, const int32_t* tokens, uint64_t n, int32_t term, SuffixState& s, bool want_lcp,
                        radix::Scratch& rs, ScanScratch& scan) {
  const uint64_t np = n + 1;
  if (np >= 0xFFFFFFFFull) fail(ITT_E_INVALID_ARGUMENT, "pattern-mining: sequence too long for 32-bit suffix indices");
  s.n = n;
  s.np = np;
  s.levels.clear();
  s.rounds = 0;
  // alphabet: codes = value - lo over tokens and the terminator
  int32_t lo = term, hi = term;
  if (n) {
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
  launch(c, "sa_text", np * 8.0, k_text_codes, dim3(grid_for(np, 256)), dim3(256), 0, tokens, n, term, lo, s.text.p);

  DBuf<uint32_t> ka(c, np), kb(c, np), va(c, np), vb(c, np);
  launch(c, "sa_init_keys", np * (4.0 * k + 8.0), k_init_keys, dim3(grid_for(np, 256)), dim3(256), 0, s.text.p, np, cbits, k,
         ka.p, va.p);
  const int init_bits = std::min(32, cbits * k);
  bool alt = radix_sort_pairs<uint32_t>(c, ka.p, va.p, kb.p, vb.p, np, 0, init_bits, rs);
  uint32_t* keys = alt ? kb.p : ka.p;
  uint32_t* sa = alt ? vb.p : va.p;
  uint32_t* keys_o = alt ? ka.p : kb.p;  // the other buffer pair is scratch for the next sort
  uint32_t* sa_o = alt ? va.p : vb.p;

  DBuf<unsigned long long> groups(c, 1);
  const uint64_t rtiles = (np + kRankBlock * kRankItems - 1) / (kRankBlock * kRankItems);
  auto rank_update = [&](const uint32_t* kk, const uint32_t* r2, const uint32_t* ss, uint32_t* rank_new) -> uint64_t {
    groups.zero();
    scan.prepare(c, rtiles);
    launch(c, "sa_rank_update", np * (r2 ? 16.0 : 12.0), k_rank_update, dim3(static_cast<unsigned>(rtiles)), dim3(kRankBlock),
           0, kk, r2, ss, np, rank_new, scan.buf.p + 1, reinterpret_cast<uint32_t*>(scan.buf.p), groups.p);
    return read1(c, groups.p);
  };
  s.levels.emplace_back(c, np);
  uint64_t g = rank_update(keys, nullptr, sa, s.levels.back().p);
  const int b = bits_for(np - 1);
  DBuf<uint32_t> r2(c, np);
  uint32_t h = s.h0;
  while (g < np) {
    const uint32_t* rank = s.levels.back().p;
    // E sorted stably by rank_i
    launch(c, "sa_emit", np * 16.0, k_emit, dim3(grid_for(np, 256)), dim3(256), 0, sa, rank, np, h, keys_o, sa_o);
    const bool a2 = radix_sort_pairs<uint32_t>(c, keys_o, sa_o, keys, sa, np, 0, b, rs);
    if (!a2) {  // result landed in (keys_o, sa_o)
      std::swap(keys, keys_o);
      std::swap(sa, sa_o);
    }
    launch(c, "sa_second_key", np * 12.0, k_second_key, dim3(grid_for(np, 256)), dim3(256), 0, sa, rank, np, h, r2.p);
    s.levels.emplace_back(c, np);
    g = rank_update(keys, r2.p, sa, s.levels.back().p);
    ++s.rounds;
    if (static_cast<uint64_t>(h) * 2 > 0xFFFFFFFFull) break;
    h *= 2;
  }
  if (g != np) fail(ITT_E_CUDA, "internal: prefix doubling did not converge");
  // SA into its own buffer
  s.sa.alloc(c, np);
  ITT_CUDA(cudaMemcpyAsync(s.sa.p, sa, np * 4, cudaMemcpyDeviceToDevice, c->stream));
  if (!want_lcp) return;

  // ---- LCP
  DBuf<uint32_t> phi(c, np), plcp(c, np);
  launch(c, "lcp_phi", np * 12.0, k_phi, dim3(grid_for(np, 256)), dim3(256), 0, s.sa.p, np, phi.p);
  std::vector<const uint32_t*> lv;
  for (auto& d : s.levels) lv.push_back(d.p);
  DBuf<const uint32_t*> dlv(c, lv.size());
  h2d(c, dlv.p, lv.data(), lv.size());
  LiftArgs L{s.text.p, np, dlv.p, static_cast<int>(lv.size()), s.h0};
  const uint64_t chunks = (np + kChunk - 1) / kChunk;
  launch(c, "lcp_plcp", np * 16.0, k_plcp, dim3(grid_for(chunks, 128)), dim3(128), 0, L, phi.p, plcp.p);
  s.lcp.alloc(c, np);
  launch(c, "lcp_gather", np * 12.0, k_lcp_gather, dim3(grid_for(np, 256)), dim3(256), 0, s.sa.p, plcp.p, np, s.lcp.p);
  c->sync();  // dlv must outlive the kernels
}

}  // namespace itt
