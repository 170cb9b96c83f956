// match.cu — approximate occurrences of the mined pattern (iteration boundaries), sm_100a.
//
// approx_match (match.hpp:41-85) is a sequential greedy scan.  It decomposes exactly into
//   (1) per anchor a (tokens[a] == P[0], match.hpp:51-54): the budgeted greedy walk from a
//       gives (ok, last, extra) independently of every other anchor — one warp per anchor,
//       32 pattern symbols compared per step with a ballot, one skip per mismatch;
//   (2) the scan visits anchors in order, jumping to last(a) + 1 after a success
//       (match.hpp:77-82): the spans are the chain  a_0 = first ok anchor,
//       a_{s+1} = first ok anchor >= last(a_s) + 1.  When no success overlaps the next ok
//       anchor (the common case) the chain is every ok anchor; otherwise the chain is
//       enumerated by binary lifting over succ().
#include <algorithm>

#include "pipeline.cuh"

namespace itt {

namespace {

struct AnchorF {  // compaction of anchor positions
  const int32_t* tok;
  int32_t head;
  uint32_t* out;
  __device__ __forceinline__ uint32_t load(uint64_t i) const { return tok[i] == head ? 1u : 0u; }
  __device__ __forceinline__ void store(uint64_t i, uint32_t excl, uint32_t v) const {
    if (v) out[excl] = static_cast<uint32_t>(i);
  }
};

// one warp per anchor: greedy budgeted subsequence walk (match.hpp:56-76)
__global__ void k_anchor_eval(const int32_t* __restrict__ tok, uint64_t n, const int32_t* __restrict__ pat, uint64_t m,
                              int64_t k0, const uint32_t* __restrict__ anchors, uint32_t n_anchors,
                              uint8_t* __restrict__ ok, uint32_t* __restrict__ last_out, uint32_t* __restrict__ extra_out) {
  const uint64_t w = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (w >= n_anchors) return;
  const unsigned lane = lane_id();
  const uint64_t a = anchors[w];
  uint64_t pos = a, j = 0, last = a;
  int64_t extra = 0;
  bool good = false;
  for (;;) {
    if (j == m) {
      good = true;
      break;
    }
    if (pos >= n) break;  // ran off the sequence before completing (match.hpp:61-64)
    // 128 symbols per step (four 32-symbol ballots, all loads in flight together): the walk over a
    // matching iteration advances 128 at a time instead of 32
    const uint64_t cnt = umin64(128, umin64(m - j, n - pos));
    unsigned mk[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t q = lane + 32u * u;
      mk[u] = __ballot_sync(0xffffffffu, q < cnt && __ldg(&tok[pos + q]) == __ldg(&pat[j + q]));
    }
    uint64_t f = 0;  // leading matches
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (mk[u] == 0xffffffffu) {
        f += 32;
        continue;
      }
      f += static_cast<uint64_t>(__ffs(~mk[u]) - 1);
      break;
    }
    if (f > cnt) f = cnt;
    if (f > 0) {
      pos += f;
      j += f;
      last = pos - 1;
    }
    if (j == m) {
      good = true;
      break;
    }
    if (f < cnt) {  // tokens[pos] != P[j]: skip it against the budget (match.hpp:70-75)
      if (++extra > k0) break;
      ++pos;
    }
  }
  if (lane == 0) {
    ok[w] = good;
    last_out[w] = static_cast<uint32_t>(last);
    extra_out[w] = static_cast<uint32_t>(extra);
  }
}

struct OkF {  // compaction of successful anchors
  const uint8_t* ok;
  const uint32_t* anchors;
  const uint32_t* last;
  const uint32_t* extra;
  uint32_t* o_pos;
  uint32_t* o_last;
  uint32_t* o_extra;
  __device__ __forceinline__ uint32_t load(uint64_t i) const { return ok[i]; }
  __device__ __forceinline__ void store(uint64_t i, uint32_t excl, uint32_t v) const {
    if (v) {
      o_pos[excl] = anchors[i];
      o_last[excl] = last[i];
      o_extra[excl] = extra[i];
    }
  }
};

// succ(x) = first ok anchor >= last(x) + 1; flags a conflict when succ(x) != x + 1
// n_ok comes from the ok-compaction scan's last status word (inclusive total), so this kernel is
// launched over all anchors and the host reads n_ok and the conflict flag in one round trip
__global__ void k_succ(const uint32_t* __restrict__ o_pos, const uint32_t* __restrict__ o_last,
                       const uint64_t* __restrict__ scan_last, uint32_t* __restrict__ succ,
                       uint32_t* __restrict__ conflict /* [0] flag, [1] n_ok */) {
  const uint32_t n_ok = static_cast<uint32_t>(*scan_last & kValMask);
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x == 0) conflict[1] = n_ok;
  if (x >= n_ok) return;
  const uint64_t target = static_cast<uint64_t>(o_last[x]) + 1;
  uint32_t lo = x + 1, hi = n_ok;  // ok anchors after x; positions strictly increase
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (o_pos[mid] < target) lo = mid + 1;
    else hi = mid;
  }
  succ[x] = lo;
  if (lo != x + 1) atomicOr(conflict, 1u);
}

__global__ void k_jump(const uint32_t* __restrict__ prev, uint32_t n_ok, uint32_t* __restrict__ next) {
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x > n_ok) return;
  const uint32_t y = x < n_ok ? prev[x] : n_ok;
  next[x] = y < n_ok ? prev[y] : n_ok;
}

// number of chain steps from node 0 (single thread)
__global__ void k_chain_length(const uint32_t* const* __restrict__ levels, int nlev, uint32_t n_ok, uint32_t* out) {
  uint32_t x = 0, t = 0;
  for (int r = nlev - 1; r >= 0; --r) {
    const uint32_t y = levels[r][x];
    if (y < n_ok) {
      x = y;
      t += 1u << r;
    }
  }
  *out = t + 1;
}

__global__ void k_chain_nodes(const uint32_t* const* __restrict__ levels, int nlev, uint32_t len,
                              const uint32_t* __restrict__ o_pos, const uint32_t* __restrict__ o_last,
                              const uint32_t* __restrict__ o_extra, uint32_t* __restrict__ s_start,
                              uint32_t* __restrict__ s_end, uint32_t* __restrict__ s_extra) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= len) return;
  uint32_t x = 0;
  for (int r = 0; r < nlev; ++r)
    if ((s >> r) & 1u) x = levels[r][x];
  s_start[s] = o_pos[x];
  s_end[s] = o_last[x];
  s_extra[s] = o_extra[x];
}

}  // namespace

void approx_match_dev(Ctx* c, const int32_t* tokens, uint64_t n, const int32_t* pattern_dev, int32_t head, uint64_t m,
                      int64_t k0, SpanState& out, ScanScratch& scan) {
  out.n = 0;
  if (m == 0 || n < m) return;  // match.hpp:47
  DBuf<uint32_t> anchors(c, n);
  DBuf<uint32_t> cnt(c, 1);
  device_scan<uint32_t, SumOp<uint32_t>>(c, "match_anchors", n * 4.0, AnchorF{tokens, head, anchors.p}, n, scan);
  const uint32_t na = static_cast<uint32_t>(scan.total(c));
  if (na == 0) return;
  DBuf<uint8_t> ok(c, na);
  DBuf<uint32_t> last(c, na), extra(c, na);
  const uint64_t threads = static_cast<uint64_t>(na) * 32;
  launch(c, "match_anchor_eval", static_cast<double>(na) * (m + 32) * 4.0, k_anchor_eval, dim3(grid_for(threads, 256)),
         dim3(256), 0, tokens, n, pattern_dev, m, k0, anchors.p, na, ok.p, last.p, extra.p);
  DBuf<uint32_t> o_pos(c, na), o_last(c, na), o_extra(c, na);
  device_scan<uint32_t, SumOp<uint32_t>>(c, "match_ok", na * 13.0,
                                         OkF{ok.p, anchors.p, last.p, extra.p, o_pos.p, o_last.p, o_extra.p}, na, scan);
  DBuf<uint32_t> succ(c, na + 1);
  DBuf<uint32_t> conflict(c, 2);
  conflict.zero();
  launch(c, "match_succ", na * 16.0, k_succ, dim3(grid_for(na, 256)), dim3(256), 0, o_pos.p, o_last.p,
         scan.buf.p + scan.tiles, succ.p, conflict.p);
  uint32_t hc[2];
  readback(c, hc, conflict.p, 2);
  const uint32_t n_ok = hc[1];
  if (n_ok == 0) return;
  if (hc[0] == 0) {  // chain = every ok anchor
    out.n = n_ok;
    out.start = std::move(o_pos);
    out.end = std::move(o_last);
    out.extra = std::move(o_extra);
    return;
  }
  // binary lifting: levels[r][x] = succ^(2^r)(x), n_ok absorbing
  std::vector<DBuf<uint32_t>> lv;
  lv.emplace_back(std::move(succ));
  ITT_CUDA(cudaMemcpyAsync(lv[0].p + n_ok, &n_ok, 4, cudaMemcpyHostToDevice, c->stream));
  c->sync();
  int nlev = 1;
  while ((1ull << nlev) <= n_ok) {
    lv.emplace_back(c, n_ok + 1);
    launch(c, "match_jump", n_ok * 12.0, k_jump, dim3(grid_for(n_ok + 1, 256)), dim3(256), 0, lv[nlev - 1].p, n_ok,
           lv[nlev].p);
    ++nlev;
  }
  std::vector<const uint32_t*> ptrs;
  for (auto& d : lv) ptrs.push_back(d.p);
  DBuf<const uint32_t*> dp(c, ptrs.size());
  h2d(c, dp.p, ptrs.data(), ptrs.size());
  launch(c, "match_chain_len", 0.0, k_chain_length, dim3(1), dim3(1), 0, dp.p, nlev, n_ok, cnt.p);
  const uint32_t len = read1(c, cnt.p);
  out.n = len;
  out.start.alloc(c, len);
  out.end.alloc(c, len);
  out.extra.alloc(c, len);
  launch(c, "match_chain_nodes", len * 24.0, k_chain_nodes, dim3(grid_for(len, 256)), dim3(256), 0, dp.p, nlev, len, o_pos.p,
         o_last.p, o_extra.p, out.start.p, out.end.p, out.extra.p);
  c->sync();
}

}  // namespace itt
