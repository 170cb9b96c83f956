// dist.cu — per-rank device steps of the distributed suffix array (SURVEY §8e, config C5 on
// G GPUs): prefix doubling over (rank_i, rank_{i+h}) pairs with a sample-sort all-to-all, and
// the capped Kasai LCP with phi routed to the owners of text positions.
//
// One trace's suffixes are block-partitioned by text position: rank r owns [lo_r, hi_r) and the
// rank array of those positions (global dense group ids, as in sa.cu).  The exchanges
// themselves (all-to-all of records, all-gather of samples / boundary keys) are the host
// driver's (paper_1707_03750_b200/dist_sa.py: NCCL through torch.distributed, or in-process
// virtual ranks); every per-element step is one of the kernels below, behind the C-ABI
// itt_dsa_* (include/itertrace_cuda.h).  Replaces the same functionality as the single-GPU
// build_suffix_array (sa.cu) — i.e. the reference's SuffixTree (suffix_tree.hpp:21-190) leaf
// order and node depths — for traces whose sort buffers do not fit one device.
//
// Records moved between ranks are (u64 a, u32 b) pairs:
//   doubling   a = (rank_i << b) | (rank_{i+h} + 1) (0 = past the end), b = i
//   ranks back a = (id << 32) | i                    (owner of i)
//   LCP ask    a = (k << 32) | SA_k, b = SA_{k-1} | same-group bit 31   (owner of SA_k)
//   LCP back   a = (plcp << 32) | k                  (owner of sorted position k)
#include <algorithm>
#include <climits>

#include "pipeline.cuh"

namespace itt {
namespace dsa {

namespace {

constexpr uint32_t kSameBit = 0x80000000u;
constexpr int kIdsBlock = 256;
constexpr int kIdsItems = 8;
constexpr int kKasaiChunk = 64;

// init keys (rank == null): the first k symbols of suffix i packed with `bits` per symbol;
// round keys: (rank_i << b) | (rank_{i+h} + 1), rank2[j] for j < n2, else 0 (suffix i+h past the end)
__global__ void k_keys(const int32_t* __restrict__ text, uint64_t np, uint64_t lo, uint64_t cnt, int bits, int k,
                       const uint32_t* __restrict__ rank, const uint32_t* __restrict__ rank2, uint64_t n2, int b,
                       uint64_t* __restrict__ a, uint32_t* __restrict__ v) {
  const uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= cnt) return;
  const uint64_t i = lo + j;
  uint64_t key = 0;
  if (!rank) {
    for (int q = 0; q < k; ++q) {
      const uint64_t c = i + q < np ? static_cast<uint32_t>(text[i + q]) : 0u;
      key = (key << bits) | c;
    }
  } else {
    const uint64_t r2 = j < n2 ? static_cast<uint64_t>(rank2[j]) + 1 : 0;
    key = (static_cast<uint64_t>(rank[j]) << b) | r2;
  }
  a[j] = key;
  v[j] = static_cast<uint32_t>(i);
}

// destination of each record: mode 0 = number of splitters <= (a, b) (lexicographic);
// mode 1 = owner of position (u32)a: the q with bounds[q] <= pos < bounds[q+1]
__global__ void k_dest(const uint64_t* __restrict__ a, const uint32_t* __restrict__ b, uint64_t cnt, int mode,
                       const uint64_t* __restrict__ spl_a, const uint32_t* __restrict__ spl_b, uint32_t nspl,
                       const uint64_t* __restrict__ bounds, uint32_t P, uint32_t* __restrict__ dest,
                       uint32_t* __restrict__ idx) {
  extern __shared__ uint64_t sh[];
  const uint32_t m = mode == 0 ? nspl : P + 1;
  for (uint32_t t = threadIdx.x; t < m; t += blockDim.x) {
    if (mode == 0) {
      sh[2 * t] = spl_a[t];
      sh[2 * t + 1] = spl_b[t];
    } else {
      sh[t] = bounds[t];
    }
  }
  __syncthreads();
  const uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= cnt) return;
  uint32_t lo = 0, hi = 0;
  if (mode == 0) {
    const uint64_t ka = a[j];
    const uint32_t kb = b[j];
    lo = 0, hi = nspl;  // count splitters <= key
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      const uint64_t sa = sh[2 * mid];
      const uint32_t sb = static_cast<uint32_t>(sh[2 * mid + 1]);
      if (sa < ka || (sa == ka && sb <= kb)) lo = mid + 1;
      else hi = mid;
    }
  } else {
    const uint64_t pos = static_cast<uint32_t>(a[j]);
    lo = 0, hi = P;  // largest q with bounds[q] <= pos
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (sh[mid] <= pos) lo = mid;
      else hi = mid;
    }
  }
  dest[j] = lo;
  idx[j] = static_cast<uint32_t>(j);
}

__global__ void k_gather(const uint64_t* __restrict__ a, const uint32_t* __restrict__ b, const uint32_t* __restrict__ perm,
                         uint64_t cnt, uint64_t* __restrict__ oa, uint32_t* __restrict__ ob) {
  const uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= cnt) return;
  const uint32_t p = perm[j];
  oa[j] = a[p];
  if (ob) ob[j] = b[p];
}

// counts[q] = number of sorted dests equal to q (P threads, binary search)
__global__ void k_dest_counts(const uint32_t* __restrict__ sorted_dest, uint64_t cnt, uint32_t P, uint64_t* __restrict__ counts) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= P) return;
  auto lower = [&](uint32_t x) {
    uint64_t lo = 0, hi = cnt;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (sorted_dest[mid] < x) lo = mid + 1;
      else hi = mid;
    }
    return lo;
  };
  counts[q] = lower(q + 1) - lower(q);
}

// new dense ids over the rank's slice of the globally sorted records: flag_j = a_j != a_{j-1}
// (a_{-1} = prev, the previous non-empty rank's last key, when has_prev); id_j = offset +
// (inclusive flag count) - 1; out_j = (id_j << 32) | b_j.  Decoupled look-back scan.
__global__ void __launch_bounds__(kIdsBlock) k_ids(const uint64_t* __restrict__ a, const uint32_t* __restrict__ b, uint64_t cnt,
                                                   int has_prev, uint64_t prev, uint32_t offset, uint64_t* __restrict__ out,
                                                   uint64_t* status, uint32_t* counter) {
  __shared__ uint32_t s_warp[kIdsBlock / 32];
  __shared__ uint32_t s_tile, s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t base = static_cast<uint64_t>(tile) * (kIdsBlock * kIdsItems) + static_cast<uint64_t>(threadIdx.x) * kIdsItems;
  uint64_t pk = 0;
  bool have = false;
  if (base < cnt) {
    if (base > 0) pk = a[base - 1], have = true;
    else if (has_prev) pk = prev, have = true;
  }
  uint32_t fmask = 0;
#pragma unroll
  for (int q = 0; q < kIdsItems; ++q) {
    const uint64_t j = base + q;
    if (j < cnt) {
      const uint64_t k = a[j];
      if (!have || k != pk) fmask |= 1u << q;
      pk = k;
      have = true;
    }
  }
  uint32_t total;
  const uint32_t texcl = block_exclusive_scan<uint32_t, SumOp<uint32_t>, kIdsBlock>(__popc(fmask), SumOp<uint32_t>(), &total, s_warp);
  if (threadIdx.x < 32) {
    const uint32_t p = tile_lookback<uint32_t, SumOp<uint32_t>>(status, tile, total, SumOp<uint32_t>());
    if (threadIdx.x == 0) s_prefix = p;
  }
  __syncthreads();
  const uint32_t pre = s_prefix + texcl;
#pragma unroll
  for (int q = 0; q < kIdsItems; ++q) {
    const uint64_t j = base + q;
    if (j < cnt) {
      const uint32_t id = offset + pre + __popc(fmask & ((2u << q) - 1u)) - 1;
      out[j] = (static_cast<uint64_t>(id) << 32) | b[j];
    }
  }
}

// dst[(u32)p - lo] = p >> 32
__global__ void k_scatter_hi(const uint64_t* __restrict__ p, uint64_t cnt, uint64_t lo, uint32_t* __restrict__ dst) {
  const uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= cnt) return;
  const uint64_t v = p[j];
  dst[static_cast<uint32_t>(v) - lo] = static_cast<uint32_t>(v >> 32);
}

// LCP requests from the sorted slice (packed (id << 32) | SA): a = (k << 32) | SA_k, b = SA_{k-1}
// (0x7FFFFFFF at k = 0) | kSameBit when SA_{k-1} is in the same final group
__global__ void k_lcp_requests(const uint64_t* __restrict__ packed, uint64_t cnt, uint64_t kbase, int has_prev, uint64_t prev,
                               uint64_t* __restrict__ a, uint32_t* __restrict__ b) {
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= cnt) return;
  const uint64_t cur = packed[t];
  const bool hp = t > 0 || has_prev;
  const uint64_t pv = t > 0 ? packed[t - 1] : prev;
  a[t] = ((kbase + t) << 32) | static_cast<uint32_t>(cur);
  b[t] = hp ? (static_cast<uint32_t>(pv) | ((pv >> 32) == (cur >> 32) ? kSameBit : 0u)) : 0x7FFFFFFFu;
}

// requests land at the owner of SA_k: phi, same flag and sorted position per own text position
__global__ void k_lcp_place(const uint64_t* __restrict__ a, const uint32_t* __restrict__ b, uint64_t cnt, uint64_t lo,
                            uint32_t* __restrict__ phi, uint32_t* __restrict__ kpos) {
  const uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= cnt) return;
  const uint64_t v = a[j];
  const uint32_t i = static_cast<uint32_t>(v) - static_cast<uint32_t>(lo);
  phi[i] = b[j];
  kpos[i] = static_cast<uint32_t>(v >> 32);
}

// capped Kasai over own text positions [lo, lo+cnt) in chunks (sa.cu k_plcp's argument: suffixes
// in the same final group share >= cap symbols; after such a shortcut the carried bound is not
// valid and the scan restarts).  The text is replicated on every rank.  Output (plcp << 32) | k.
__global__ void k_kasai(const int32_t* __restrict__ text, uint64_t np, uint64_t lo, uint64_t cnt, const uint32_t* __restrict__ phi,
                        const uint32_t* __restrict__ kpos, uint32_t cap, uint64_t* __restrict__ out) {
  const uint64_t c0 = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * kKasaiChunk;
  if (c0 >= cnt) return;
  const uint64_t c1 = umin64(c0 + kKasaiChunk, cnt);
  uint32_t l = 0;
  bool capped = false;
  for (uint64_t j = c0; j < c1; ++j) {
    const uint64_t i = lo + j;
    const uint32_t pw = phi[j];
    uint32_t v;
    if (pw == 0x7FFFFFFFu) {  // SA_0
      v = 0, l = 0, capped = false;
    } else if (pw & kSameBit) {
      v = cap, l = cap - 1, capped = true;
    } else {
      const uint64_t p = pw;
      if (capped) l = 0;
      while (l < cap && i + l < np && p + l < np && __ldg(&text[i + l]) == __ldg(&text[p + l])) ++l;
      v = l;
      capped = false;
      if (l > 0) --l;
    }
    out[j] = (static_cast<uint64_t>(v) << 32) | kpos[j];
  }
}

// pseudo-random positions (splitmix64): evenly spaced samples would alias with the period of
// a periodic trace and see one key
__global__ void k_sample(const uint64_t* __restrict__ a, const uint32_t* __restrict__ b, uint64_t cnt, uint32_t s,
                         uint64_t* __restrict__ oa, uint32_t* __restrict__ ob) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= s) return;
  uint64_t z = static_cast<uint64_t>(t) + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  const uint64_t j = z % cnt;
  oa[t] = a[j];
  ob[t] = b[j];
}

}  // namespace

void keys(Ctx* c, const int32_t* text, uint64_t np, uint64_t lo, uint64_t cnt, int bits, int k, const uint32_t* rank,
          const uint32_t* rank2, uint64_t n2, int b, uint64_t* a, uint32_t* v) {
  if (!cnt) return;
  launch(c, "dsa_keys", cnt * 24.0, k_keys, dim3(grid_for(cnt, 256)), dim3(256), 0, text, np, lo, cnt, bits, k, rank, rank2, n2,
         b, a, v);
}

// stable partition of (a, b) by destination into (oa, ob); counts[P] to the host
void partition(Ctx* c, const uint64_t* a, const uint32_t* b, uint64_t cnt, int mode, const uint64_t* spl_a,
               const uint32_t* spl_b, uint32_t nspl, const uint64_t* bounds, uint32_t P, uint64_t* oa, uint32_t* ob,
               uint64_t* counts_host) {
  std::fill(counts_host, counts_host + P, 0);
  if (!cnt) return;
  DBuf<uint32_t> d0(c, cnt), i0(c, cnt), d1(c, cnt), i1(c, cnt);
  const size_t smem = (mode == 0 ? 2 * static_cast<size_t>(nspl) : P + 1) * 8;
  launch(c, "dsa_dest", cnt * 24.0, k_dest, dim3(grid_for(cnt, 256)), dim3(256), smem, a, b, cnt, mode, spl_a, spl_b, nspl,
         bounds, P, d0.p, i0.p);
  const int bits = bits_for(P > 1 ? P - 1 : 1);
  radix::Scratch rs;
  const bool alt = radix_sort_pairs<uint32_t>(c, d0.p, i0.p, d1.p, i1.p, cnt, 0, bits, rs);
  const uint32_t* sd = alt ? d1.p : d0.p;
  const uint32_t* si = alt ? i1.p : i0.p;
  launch(c, "dsa_gather", cnt * 28.0, k_gather, dim3(grid_for(cnt, 256)), dim3(256), 0, a, b, si, cnt, oa, ob);
  DBuf<uint64_t> cd(c, P);
  launch(c, "dsa_counts", 0.0, k_dest_counts, dim3(grid_for(P, 128)), dim3(128), 0, sd, cnt, P, cd.p);
  readback(c, counts_host, cd.p, P);
}

// stable sort of (a, b) by the low `bits` bits of a, in place
void sort(Ctx* c, uint64_t* a, uint32_t* b, uint64_t cnt, int bits) {
  if (cnt < 2) return;
  DBuf<uint64_t> a1(c, cnt);
  DBuf<uint32_t> b1(c, cnt);
  radix::Scratch rs;
  bits = std::max(1, bits);
  // 10-bit digits when they save a pass (e.g. 42-bit pair keys: 5 passes instead of 6)
  const bool wide = (bits + radix::kWideBits - 1) / radix::kWideBits < (bits + 7) / 8;
  const bool alt = wide ? radix_sort_pairs<uint64_t, radix::ArrayLoader<uint64_t>, radix::kWideBits>(c, a, b, a1.p, b1.p, cnt, 0,
                                                                                                      bits, rs)
                        : radix_sort_pairs<uint64_t>(c, a, b, a1.p, b1.p, cnt, 0, bits, rs);
  if (alt) {
    ITT_CUDA(cudaMemcpyAsync(a, a1.p, cnt * 8, cudaMemcpyDeviceToDevice, c->stream));
    ITT_CUDA(cudaMemcpyAsync(b, b1.p, cnt * 4, cudaMemcpyDeviceToDevice, c->stream));
  }
}

uint64_t ids(Ctx* c, const uint64_t* a, const uint32_t* b, uint64_t cnt, bool has_prev, uint64_t prev, uint32_t offset,
             uint64_t* out) {
  if (!cnt) return 0;
  constexpr uint64_t TILE = kIdsBlock * kIdsItems;
  const uint64_t tiles = (cnt + TILE - 1) / TILE;
  ScanScratch sc;
  sc.prepare(c, tiles);
  launch(c, "dsa_ids", cnt * 20.0, k_ids, dim3(static_cast<unsigned>(tiles)), dim3(kIdsBlock), 0, a, b, cnt, has_prev ? 1 : 0, prev,
         offset, out, sc.buf.p + 1, reinterpret_cast<uint32_t*>(sc.buf.p));
  return sc.total(c);
}

void scatter_hi(Ctx* c, const uint64_t* p, uint64_t cnt, uint64_t lo, uint32_t* dst) {
  if (!cnt) return;
  launch(c, "dsa_scatter", cnt * 12.0, k_scatter_hi, dim3(grid_for(cnt, 256)), dim3(256), 0, p, cnt, lo, dst);
}

void lcp_requests(Ctx* c, const uint64_t* packed, uint64_t cnt, uint64_t kbase, bool has_prev, uint64_t prev, uint64_t* a,
                  uint32_t* b) {
  if (!cnt) return;
  launch(c, "dsa_lcp_requests", cnt * 20.0, k_lcp_requests, dim3(grid_for(cnt, 256)), dim3(256), 0, packed, cnt, kbase,
         has_prev ? 1 : 0, prev, a, b);
}

void kasai(Ctx* c, const int32_t* text, uint64_t np, uint64_t lo, uint64_t cnt, const uint64_t* req_a, const uint32_t* req_b,
           uint32_t cap, uint64_t* out) {
  if (!cnt) return;
  DBuf<uint32_t> phi(c, cnt), kpos(c, cnt);
  launch(c, "dsa_lcp_place", cnt * 20.0, k_lcp_place, dim3(grid_for(cnt, 256)), dim3(256), 0, req_a, req_b, cnt, lo, phi.p, kpos.p);
  const uint64_t chunks = (cnt + kKasaiChunk - 1) / kKasaiChunk;
  launch(c, "dsa_kasai", cnt * 24.0, k_kasai, dim3(grid_for(chunks, 128)), dim3(128), 0, text, np, lo, cnt, phi.p, kpos.p, cap, out);
}

void sample(Ctx* c, const uint64_t* a, const uint32_t* b, uint64_t cnt, uint32_t s, uint64_t* oa, uint32_t* ob) {
  if (!cnt || !s) return;
  launch(c, "dsa_sample", 0.0, k_sample, dim3(grid_for(s, 256)), dim3(256), 0, a, b, cnt, s, oa, ob);
}

}  // namespace dsa
}  // namespace itt
