// intern.cu — records -> (start,row) order -> GPU name dictionary -> census -> main-stream
// token string in first-appearance order.
//
// Replaces, on the device:
//   ingest.hpp:396-400      stable sort by (start, row)            (K1: radix sort of start)
//   trace.hpp:103-113       classify_op_kind per record            (per distinct name, then a lookup)
//   streams.hpp:60-81       summarize_streams                      (warp-aggregated census)
//   streams.hpp:179-207     filter_majority_device                 (device census + keep mask)
//   streams.hpp:147-169     build_token_sequence                   (hash dictionary + first appearance)
//   streams.hpp:212-221     count_interval_overlaps
// The dictionary is exact: a 64-bit hash only picks the slot; every record's name bytes are
// then compared with the slot representative's bytes, and a mismatch (a true hash
// collision) re-runs the dictionary with another seed.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <thread>

#include "pipeline.cuh"

namespace itt {

namespace {

constexpr int kHashBlock = 128;
constexpr int kWarpBuf = 4096;  // staged name bytes per warp
constexpr uint32_t kDevSmem = 64;
constexpr uint32_t kStreamTableCap = 4096;
constexpr uint32_t kBlockStreams = 64;

// classify bits of a name (trace.hpp:103-113 needs memcpy+{htod,dtoh,dtod}, memset)
enum : uint8_t { NB_MEMCPY = 1, NB_HTOD = 2, NB_DTOH = 4, NB_DTOD = 8, NB_MEMSET = 16 };

__device__ __forceinline__ int kind_from(uint8_t nb, bool has_tp) {
  if (nb & NB_MEMCPY) {
    if (nb & NB_HTOD) return ITT_KIND_HTOD;
    if (nb & NB_DTOH) return ITT_KIND_DTOH;
    if (nb & NB_DTOD) return ITT_KIND_DTOD;
  }
  if (nb & NB_MEMSET) return ITT_KIND_MEMSET;
  return has_tp ? ITT_KIND_OTHER : ITT_KIND_KERNEL;
}

// low n (< 8) bytes of w, or w
__device__ __forceinline__ uint64_t low_bytes(uint64_t w, uint32_t n) {
  return n >= 8 ? w : (w & ((1ull << (8 * n)) - 1ull));
}

__device__ __forceinline__ uint64_t fmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}
// Name hash: NH (two 32x32->64 products per 16-byte chunk, keys from the seed) summed over the
// name's 16-byte chunks, then fmix64 with the length.  The sum does not depend on the order the
// chunks are visited in, so eight lanes hash one name at once (one chunk each, a 3-step shuffle
// reduction) — coalesced shared-memory reads instead of one lane walking each name.  A new seed
// draws new keys, so a collision (caught by the byte compare) does not survive a re-run.
__device__ __forceinline__ uint32_t nh_key(uint64_t seed, uint32_t idx) {
  return static_cast<uint32_t>(fmix64(seed ^ ((static_cast<uint64_t>(idx) + 1) * 0x9E3779B97F4A7C15ull)));
}
__device__ __forceinline__ void nh_keys(uint64_t seed, uint32_t chunk, uint32_t (&k)[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) k[i] = nh_key(seed, chunk * 4 + i);
}
__device__ __forceinline__ uint64_t nh_chunk(const uint32_t (&x)[4], const uint32_t (&k)[4]) {
  return static_cast<uint64_t>(x[0] + k[0]) * (x[1] + k[1]) + static_cast<uint64_t>(x[2] + k[2]) * (x[3] + k[3]);
}
__device__ __forceinline__ uint64_t nh_final(uint64_t sum, uint32_t len, uint64_t seed) {
  const uint64_t h = fmix64(sum ^ seed ^ (static_cast<uint64_t>(len) * 0xC2B2AE3D27D4EB4Full));
  return h ? h : 1;  // 0 marks an empty slot
}
// keep the first v (0..16) bytes of a chunk, zero the rest
__device__ __forceinline__ void mask_chunk(uint32_t (&x)[4], int v) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int b = v - 4 * i;
    x[i] = b >= 4 ? x[i] : (b <= 0 ? 0u : x[i] & ((1u << (8 * b)) - 1u));
  }
}

// Stage the name bytes of rows [g0, g1) into a per-warp shared buffer with 16-byte cp.async
// copies (L2-only: the names are streamed once); the caller commits and waits.  Returns false when
// they do not fit (the caller then reads global memory directly).
__device__ __forceinline__ bool stage_issue(const uint8_t* __restrict__ bytes, uint64_t total, uint64_t b0, uint64_t b1,
                                            uint8_t* buf, uint64_t& base) {
  const uint64_t a0 = b0 & ~15ull, a1 = (b1 + 15) & ~15ull;
  base = a0;
  if (a1 - a0 > static_cast<uint64_t>(kWarpBuf)) return false;
  const bool aligned = (reinterpret_cast<uintptr_t>(bytes) & 15) == 0;
  if (aligned && a1 <= total) {  // every chunk in bounds: 32-bit shared offsets, one cp.async each
    const uint32_t nch = static_cast<uint32_t>((a1 - a0) >> 4);
    const uint32_t dst0 = static_cast<uint32_t>(__cvta_generic_to_shared(buf));
    const uint8_t* src0 = bytes + a0;
    for (uint32_t ch = lane_id(); ch < nch; ch += 32)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst0 + ch * 16), "l"(src0 + ch * 16) : "memory");
  } else {
    for (uint64_t o = a0 + lane_id() * 16; o < a1; o += 512) {
      if (aligned && o + 16 <= total) {
        const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(buf + (o - a0)));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(bytes + o) : "memory");
      } else {
        for (int j = 0; j < 16; ++j) buf[o - a0 + j] = o + j < total ? bytes[o + j] : 0;
      }
    }
  }
  return true;
}

// ------------------------------------------------------------------ K1: order
// Sort each 256-row block by (start, row) — unique keys because the row breaks ties, so the
// result is the stable order — and record the block's start range and whether the source order
// has a descent.  Bitonic network with one row per thread: the 30 stages whose partner is in the
// same warp exchange through shuffles; only the 6 cross-warp stages (j >= 32) go through shared
// memory.  Global min/max and the descent flag are folded in k_order_check (no same-address
// atomics per block).
constexpr int kOrderBlock = 256;

// Any descent start[i] < start[i-1] in source order?  8 rows per thread (16-byte loads); the block
// sort and its check run only when one exists (profiler exports of one stream, and the synthetic
// C3 / C5 traces, arrive in start order: the 256-row bitonic sorts would be pure overhead).
__global__ void __launch_bounds__(256) k_order_descent(const int64_t* __restrict__ start, uint64_t n,
                                                       unsigned int* __restrict__ any) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x * 8;
  bool d = false;
  for (uint64_t i0 = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 8; i0 < n; i0 += stride) {
    long long v[8];
    if (i0 + 8 <= n) {
#pragma unroll
      for (int q = 0; q < 8; q += 2) {
        const longlong2 w = __ldcs(reinterpret_cast<const longlong2*>(start + i0 + q));
        v[q] = w.x, v[q + 1] = w.y;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = i0 + q < n ? start[i0 + q] : LLONG_MAX;
    }
    long long prev = i0 > 0 ? start[i0 - 1] : LLONG_MIN;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      d |= v[q] < prev;
      prev = v[q];
    }
  }
  if (__any_sync(0xffffffffu, d) && lane_id() == 0) atomicOr(any, 1u);
}

__global__ void __launch_bounds__(kOrderBlock) k_order_block_sort(const int64_t* __restrict__ start, uint64_t n,
                                                                  uint32_t* __restrict__ perm, int64_t* __restrict__ bmin,
                                                                  int64_t* __restrict__ bmax, uint8_t* __restrict__ bdesc,
                                                                  const unsigned int* __restrict__ any) {
  if (*any == 0) return;  // already in (start, row) order: one small grid exits at once
  __shared__ long long s[kOrderBlock];
  __shared__ uint32_t r[kOrderBlock];
  __shared__ long long wmn[kOrderBlock / 32], wmx[kOrderBlock / 32];
  const uint64_t nb = (n + kOrderBlock - 1) / kOrderBlock;
  const uint32_t t = threadIdx.x;
  for (uint64_t blk = blockIdx.x; blk < nb; blk += gridDim.x) {  // grid-stride over the 256-row blocks
    __syncthreads();  // the previous block's shared arrays are consumed
    const uint64_t base = blk * kOrderBlock;
    const uint32_t len = static_cast<uint32_t>(umin64(kOrderBlock, n - base));
    long long a = t < len ? __ldcs(&start[base + t]) : LLONG_MAX;  // padding rows sort last
    uint32_t ra = t;
    s[t] = a;
    long long mn = a, mx = t < len ? a : LLONG_MIN;
    for (int o = 16; o > 0; o >>= 1) {
      mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane_id() == 0) wmn[t >> 5] = mn, wmx[t >> 5] = mx;
    __syncthreads();
    // descent in the source order: against the previous row of the block / of the previous block
    const long long prev = t > 0 ? s[t - 1] : (base > 0 ? start[base - 1] : LLONG_MIN);
    const int any_desc = __syncthreads_or(t < len && prev > a);
    long long bmn = wmn[0], bmx = wmx[0];
    for (int w = 1; w < kOrderBlock / 32; ++w) bmn = min(bmn, wmn[w]), bmx = max(bmx, wmx[w]);
    if (t == 0) {
      bmin[blk] = bmn;
      bmax[blk] = bmx;
      bdesc[blk] = any_desc ? 1 : 0;
    }
    if (static_cast<unsigned long long>(bmx) - static_cast<unsigned long long>(bmn) < (1ull << 24)) {
      // narrow block (the usual case: 256 consecutive records span far less than 16.7 ms): sort one
      // 32-bit key (start - min) << 8 | row — one shuffle per stage instead of three, and the row
      // in the low bits breaks ties exactly like (start, row); padding rows sort last
      uint32_t key = t < len ? (static_cast<uint32_t>(a - bmn) << 8) | t : 0xFFFFFFFFu;
      for (uint32_t k = 2; k <= kOrderBlock; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
          uint32_t b;
          if (j >= 32) {
            __syncthreads();
            r[t] = key;
            __syncthreads();
            b = r[t ^ j];
          } else {
            b = __shfl_xor_sync(0xffffffffu, key, j);
          }
          const bool lower = (t & j) == 0, ascending = (t & k) == 0;
          if ((lower == ascending) == (key > b)) key = b;
        }
      }
      if (t < len) perm[base + t] = static_cast<uint32_t>(base + (key & 0xFFu));
      continue;
    }
    for (uint32_t k = 2; k <= kOrderBlock; k <<= 1) {
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        long long b;
        uint32_t rb;
        if (j >= 32) {
          __syncthreads();
          s[t] = a;
          r[t] = ra;
          __syncthreads();
          b = s[t ^ j];
          rb = r[t ^ j];
        } else {
          b = __shfl_xor_sync(0xffffffffu, a, j);
          rb = __shfl_xor_sync(0xffffffffu, ra, j);
        }
        const bool a_gt_b = a > b || (a == b && ra > rb);
        const bool lower = (t & j) == 0, ascending = (t & k) == 0;
        if ((lower == ascending) == a_gt_b) a = b, ra = rb;  // lower keeps the min when ascending
      }
    }
    if (t < len) perm[base + t] = static_cast<uint32_t>(base + ra);
  }
}

// Fold the per-block results: stats = [min start, max start, any descent, overlapping block
// boundaries]; block b's largest start must not exceed block b+1's smallest (equal starts stay in
// row order).  One set of atomics per CTA.
__global__ void __launch_bounds__(256) k_order_check(const int64_t* __restrict__ bmin, const int64_t* __restrict__ bmax,
                                                     const uint8_t* __restrict__ bdesc, uint64_t nb,
                                                     unsigned long long* stats, const unsigned int* __restrict__ any) {
  if (*any == 0) return;  // no descent: stats keep "no descent" (the blocks were not sorted)
  const uint64_t b = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  long long mn = LLONG_MAX, mx = LLONG_MIN;
  unsigned desc = 0, bad = 0;
  if (b < nb) {
    mn = bmin[b];
    mx = bmax[b];
    desc = bdesc[b];
    bad = b + 1 < nb && mx > bmin[b + 1];
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  desc = __reduce_or_sync(0xffffffffu, desc);
  bad = __reduce_add_sync(0xffffffffu, bad);
  __shared__ long long smn[8], smx[8];
  __shared__ unsigned sd[8], sb[8];
  if (lane_id() == 0) smn[threadIdx.x >> 5] = mn, smx[threadIdx.x >> 5] = mx, sd[threadIdx.x >> 5] = desc, sb[threadIdx.x >> 5] = bad;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) mn = min(mn, smn[w]), mx = max(mx, smx[w]), desc |= sd[w], bad += sb[w];
    atomicMin(reinterpret_cast<long long*>(&stats[0]), mn);
    atomicMax(reinterpret_cast<long long*>(&stats[1]), mx);
    if (desc) atomicAdd(&stats[2], 1ull);
    if (bad) atomicAdd(&stats[3], static_cast<unsigned long long>(bad));
  }
}

__global__ void k_order_keys(const int64_t* __restrict__ start, uint64_t n, int64_t mn, uint64_t* __restrict__ keys,
                             uint32_t* __restrict__ vals) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) {
    keys[i] = static_cast<uint64_t>(start[i] - mn);
    vals[i] = static_cast<uint32_t>(i);
  }
}

// ------------------------------------------------------------------ K2: dictionary
// 4 bytes at an arbitrary address from two aligned words (callers keep the read in bounds)
// explicit address spaces: an address rebuilt from an integer would otherwise compile to a
// generic LD (long-scoreboard, LSU path) even when it points into shared memory
struct SharedBytes {
  uint32_t base;  // shared-window address
  __device__ __forceinline__ explicit SharedBytes(const uint8_t* p)
      : base(static_cast<uint32_t>(__cvta_generic_to_shared(p))) {}
  __device__ __forceinline__ uint32_t word(uint32_t a) const {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
  }
  __device__ __forceinline__ uint32_t load4(uint32_t i) const {
    const uint32_t a = base + i;
    return __funnelshift_r(word(a & ~3u), word((a & ~3u) + 4), (a & 3) * 8);
  }
  __device__ __forceinline__ uint8_t byte(uint32_t i) const {
    uint16_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(base + i));
    return static_cast<uint8_t>(v);
  }
};
// Sequential 4-byte reads of an unaligned run in shared memory: one aligned LDS per step (the
// previous aligned word is reused), instead of two per unaligned 4-byte read.  Reads at most
// one aligned word past the run (the staging buffers are padded).
struct SharedStream {
  uint32_t addr;  // next aligned word to load
  uint32_t sh;    // byte misalignment in bits
  uint32_t cur;
  __device__ __forceinline__ static uint32_t lds(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
  }
  __device__ __forceinline__ explicit SharedStream(const SharedBytes& p)
      : addr((p.base & ~3u) + 4), sh((p.base & 3u) * 8), cur(lds(p.base & ~3u)) {}
  __device__ __forceinline__ uint32_t next4() {
    const uint32_t nw = lds(addr);
    addr += 4;
    const uint32_t v = __funnelshift_r(cur, nw, sh);
    cur = nw;
    return v;
  }
};
struct GlobalBytes {
  const uint8_t* p;
  __device__ __forceinline__ explicit GlobalBytes(const uint8_t* q) : p(q) {}
  __device__ __forceinline__ uint32_t load4(uint32_t i) const {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p + i);
    const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~static_cast<uintptr_t>(3));
    return __funnelshift_r(__ldg(w), __ldg(w + 1), static_cast<uint32_t>(a & 3) * 8);
  }
  __device__ __forceinline__ uint8_t byte(uint32_t i) const { return __ldg(p + i); }
};
// byte equality of two names; words while 8 bytes remain (keeps the aligned-word reads inside
// the name's buffer), then bytes
template <typename A, typename B>
__device__ __forceinline__ bool same_bytes(const A& p, const B& q, uint32_t len) {
  uint32_t i = 0;
  for (; i + 8 <= len; i += 4)
    if (p.load4(i) != q.load4(i)) return false;
  for (; i < len; ++i)
    if (p.byte(i) != q.byte(i)) return false;
  return true;
}
// both runs in shared memory: two streams, one LDS per side per 4 bytes, 8 bytes per step; the
// 0-7 byte tail as one masked 8-byte compare (staging buffers are padded)
__device__ __forceinline__ bool same_bytes(const SharedBytes& p, const SharedBytes& q, uint32_t len) {
  SharedStream a(p), b(q);
  uint32_t i = 0;
  uint32_t diff = 0;
  for (; i + 8 <= len; i += 8) {
    const uint32_t x0 = a.next4(), y0 = b.next4();
    const uint32_t x1 = a.next4(), y1 = b.next4();
    diff |= (x0 ^ y0) | (x1 ^ y1);
  }
  const uint32_t x0 = a.next4(), y0 = b.next4();
  const uint32_t x1 = a.next4(), y1 = b.next4();
  const uint64_t d = (static_cast<uint64_t>(x0 ^ y0) | (static_cast<uint64_t>(x1 ^ y1) << 32));
  return diff == 0 && low_bytes(d, len - i) == 0;
}

struct HashArgs {
  const uint64_t* name_off;
  const uint8_t* bytes;  // bytes[o] is name byte o for o in [lo, total)
  uint64_t lo;           // 0, or the first byte of a streamed chunk window (16-byte aligned)
  uint64_t total;
  uint64_t row0;         // rows [row0, n) in this launch
  uint64_t n;
  const uint8_t* arena;  // streamed names: bytes of the slot representatives of earlier chunks
  const uint64_t* arena_off;
  const uint16_t* device;
  uint64_t* tkey;  // (32-bit hash fragment | 1) << 32 | row of the slot's first inserter; 0 = empty
  uint64_t* tready;  // (128-byte unit of the slot's copy in `copies` + 1) << 32 | name length; 0 = not yet
  uint8_t* copies;   // representatives' names, 128-byte aligned, zero-padded to whole 16-byte chunks
  uint64_t copies_cap;
  unsigned long long* copies_top;
  uint32_t mask;
  uint64_t seed;
  uint32_t* slot_out;
  uint32_t* used;
  uint32_t* used_count;  // [0] = count, [1] = overflow flag, [2] = collision flag
  unsigned long long* dev_counts;  // [65536]
  uint32_t* dev_max;
};

// name-relative bytes [q, q + 16) of a name staged at shared address `s`: five aligned words,
// funnel-shifted (the staging buffer is padded, so the fifth word is always in bounds)
__device__ __forceinline__ void chunk_shared(uint32_t s, uint32_t q, uint32_t (&x)[4]) {
  const uint32_t a = s + q, w = a & ~3u, sh = (a & 3u) * 8;
  uint32_t v[5];
#pragma unroll
  for (int i = 0; i < 5; ++i) v[i] = SharedStream::lds(w + 4 * i);
#pragma unroll
  for (int i = 0; i < 4; ++i) x[i] = __funnelshift_r(v[i], v[i + 1], sh);
}
// the same from global memory, byte by byte (groups too long to stage)
__device__ __forceinline__ void chunk_global(const uint8_t* p, int v, uint32_t (&x)[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint32_t w = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (4 * i + j < v) w |= static_cast<uint32_t>(__ldg(p + 4 * i + j)) << (8 * j);
    x[i] = w;
  }
}
__device__ __forceinline__ uint4 ld_cg_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

// One warp per group of 32 consecutive rows.  The group's name bytes are staged into shared
// memory (one contiguous cp.async range); then
//   1. hash: sub-warp `sub` (8 lanes) hashes name 4*it + sub in round `it`, one 16-byte chunk per
//      lane, and the hash moves to the name's own lane;
//   2. probe (lane per row): find the slot or claim it with one 64-bit CAS of (hash fragment, row);
//      the claimer also reserves a 16-byte aligned copy of its name in `copies`;
//   3. verify (sub-warp per name again): a claimer writes its copy and publishes it in tready; any
//      other row whose slot copy is published compares its chunks (still in registers from step 1
//      for names up to 128 bytes) with the copy — one coalesced 16-byte load per lane; rows whose
//      slot copy is not yet published (its claimer is still in flight) compare with the
//      representative row's own bytes, lane by lane.
// A byte mismatch means two different names landed in one slot: the collision flag makes the host
// re-run with another seed, so a hash never decides equality on its own.  Device census: one
// ballot round per distinct device id in the warp.
#ifndef ITT_HASH_MINB
#define ITT_HASH_MINB 4  // 4 CTAs per SM: more warps hide the probe and copy latency (C3: 6.9 -> 5.8 ms)
#endif
__global__ void __launch_bounds__(kHashBlock, ITT_HASH_MINB) k_hash_insert(HashArgs a) {
  // double-buffered names; padded so a lane past its name's end still reads inside the buffer
  __shared__ __align__(16) uint8_t s_buf[kHashBlock / 32][2][kWarpBuf + 144];
  __shared__ __align__(16) uint64_t s_part[kHashBlock / 32][8][32];  // per-lane NH partial sums
  __shared__ uint4 s_mask[17];  // s_mask[v]: keep the first v bytes of a 16-byte chunk
  __shared__ uint2 s_nm[kHashBlock / 32][32];  // per row of the group: (length, offset) / (mode, copy)
  __shared__ unsigned int s_dev[kDevSmem];
  __shared__ uint32_t s_devmax;
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const unsigned sub = lane >> 3, t = lane & 7;
  for (unsigned i = threadIdx.x; i < kDevSmem; i += blockDim.x) s_dev[i] = 0;
  if (threadIdx.x == 0) s_devmax = 0;
  uint32_t dev_hi = 0;  // largest device id this thread counted
  if (threadIdx.x < 17) {
    uint32_t x[4] = {~0u, ~0u, ~0u, ~0u};
    mask_chunk(x, static_cast<int>(threadIdx.x));
    s_mask[threadIdx.x] = make_uint4(x[0], x[1], x[2], x[3]);
  }
  __syncthreads();
  if (a.total == ~0ull) a.total = __ldg(&a.name_off[a.n]);  // resident names: end of the byte buffer
  uint32_t key0[4];  // NH keys of this lane's chunk in the first 128 bytes of a name
  nh_keys(a.seed, t, key0);
  const uint64_t groups = (a.n - a.row0 + 31) / 32;
  const uint64_t gstride = static_cast<uint64_t>(gridDim.x) * (blockDim.x / 32);
  bool bad = false;
  // name offsets: one load per lane (+ lane 31 the group's end), issued two groups ahead
  auto offsets = [&](uint64_t g, uint64_t& off, uint64_t& nxt) {
    const uint64_t r0 = a.row0 + g * 32;
    off = g < groups ? __ldg(&a.name_off[umin64(r0 + lane, a.n)]) : 0;
    nxt = g < groups && lane == 31 ? __ldg(&a.name_off[umin64(r0 + 32, a.n)]) : 0;
  };
  // a group's name ends and byte span; its names go into buffer `b` (one group ahead of use)
  auto stage = [&](uint64_t g, uint64_t off, uint64_t nxt, int b, uint64_t& end, uint64_t& base) -> bool {
    const uint64_t g0 = a.row0 + g * 32, cnt = umin64(32, a.n - g0);
    const uint64_t down = __shfl_down_sync(0xffffffffu, off, 1);
    end = lane == 31 ? nxt : down;  // name_off[row + 1]
    const uint64_t b0 = __shfl_sync(0xffffffffu, off, 0);
    const uint64_t b1 = __shfl_sync(0xffffffffu, end, static_cast<int>(cnt - 1));
    return stage_issue(a.bytes, a.total, b0, b1, s_buf[warp][b], base);
  };
  uint64_t g = static_cast<uint64_t>(blockIdx.x) * (blockDim.x / 32) + warp;
  uint64_t my_off = 0, my_end = 0, cur_base = 0, off_n = 0, end_n = 0;
  bool cur_staged = false;
  int cur = 0;
  if (g < groups) {
    uint64_t nxt;
    offsets(g, my_off, nxt);
    cur_staged = stage(g, my_off, nxt, 0, my_end, cur_base);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  offsets(g + gstride, off_n, end_n);
  for (; g < groups; g += gstride) {
    const uint64_t g0 = a.row0 + g * 32, g1 = min(g0 + 32, a.n);
    const uint64_t row = g0 + lane;
    const bool valid = row < a.n;
    // the next group's names into the other buffer while this group is processed
    uint64_t nx_end = 0, nx_base = 0, nx_off = off_n;
    bool nx_staged = false;
    if (g + gstride < groups) nx_staged = stage(g + gstride, off_n, end_n, cur ^ 1, nx_end, nx_base);
    asm volatile("cp.async.commit_group;" ::: "memory");
    offsets(g + 2 * gstride, off_n, end_n);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncwarp();
    uint8_t* buf = s_buf[warp][cur];
    const uint32_t sbuf = static_cast<uint32_t>(__cvta_generic_to_shared(buf));
    const uint64_t base = cur_base;
    const bool staged = cur_staged;
    const uint32_t len = valid ? static_cast<uint32_t>(my_end - my_off) : 0u;

    // ---- 1. hash, 8 lanes per name; each lane's partial sum goes through shared memory, and the
    // name's own lane adds its eight partials
    const uint32_t rel = static_cast<uint32_t>(my_off - base);  // staged: the name's offset in buf
    const bool short_names = __all_sync(0xffffffffu, len <= 128);
    uint32_t xw[8][4];  // this lane's chunk of the first 128 bytes of name 4*it + sub
    if (staged && short_names) {  // the common case: one chunk per lane, straight-line code
      s_nm[warp][lane] = make_uint2(len, rel);
      __syncwarp();
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const uint2 nm = s_nm[warp][4 * it + sub];  // (length, offset in buf) of this sub-warp's name
        const int vb = static_cast<int>(nm.x) - static_cast<int>(16 * t);  // valid bytes of this lane's chunk
        uint32_t x[4];
        chunk_shared(sbuf + nm.y, 16 * t, x);  // in bounds: the buffer is padded past a chunk
        const uint4 m = s_mask[min(max(vb, 0), 16)];
        x[0] &= m.x, x[1] &= m.y, x[2] &= m.z, x[3] &= m.w;
        const uint64_t c = nh_chunk(x, key0);
#pragma unroll
        for (int i = 0; i < 4; ++i) xw[it][i] = x[i];
        s_part[warp][it][lane] = vb > 0 ? c : 0ull;
      }
    } else {
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int j = 4 * it + static_cast<int>(sub);
        const uint32_t lj = __shfl_sync(0xffffffffu, len, j);
        uint32_t relj = 0;
        uint64_t oj = 0;
        if (staged) relj = __shfl_sync(0xffffffffu, rel, j);
        else oj = __shfl_sync(0xffffffffu, my_off, j);
        uint64_t acc = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) xw[it][i] = 0;
        for (uint32_t q = 16 * t; q < lj; q += 128) {
          uint32_t x[4];
          const int v = static_cast<int>(min(16u, lj - q));
          if (staged) chunk_shared(sbuf + relj, q, x);
          else chunk_global(a.bytes + oj + q, v, x);
          const uint4 m = s_mask[v];
          x[0] &= m.x, x[1] &= m.y, x[2] &= m.z, x[3] &= m.w;
          if (q < 128) {
#pragma unroll
            for (int i = 0; i < 4; ++i) xw[it][i] = x[i];
            acc += nh_chunk(x, key0);
          } else {
            uint32_t kk[4];
            nh_keys(a.seed, q / 16, kk);
            acc += nh_chunk(x, kk);
          }
        }
        s_part[warp][it][lane] = acc;
      }
    }
    __syncwarp();
    uint64_t my_h;
    {
      const ulonglong2* pp = reinterpret_cast<const ulonglong2*>(&s_part[warp][lane >> 2][8 * (lane & 3)]);
      uint64_t sum = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const ulonglong2 v = pp[i];
        sum += v.x + v.y;
      }
      my_h = nh_final(sum, len, a.seed);
    }
    __syncwarp();  // s_part is rewritten by the next group
    if (a.seed == 0) my_h = 1;  // test hook (ITT_TEST_FORCE_COLLISION): every name in one slot
    // ---- 2. probe, lane per row
    uint32_t s = 0, rep = static_cast<uint32_t>(row);
    uint64_t ready = 0, copy_at = ~0ull;
    bool claimed = false;
    if (valid) {
      const uint64_t frag = ((my_h >> 32) | 1ull) << 32;  // nonzero: 0 marks an empty slot
      s = static_cast<uint32_t>(my_h) & a.mask;
      for (uint32_t probe = 0;; ++probe) {
        if (probe > a.mask) {
          atomicOr(&a.used_count[1], 1u);
          break;
        }
        uint64_t k = ld_relaxed_u64(&a.tkey[s]);
        const uint64_t rd = ld_relaxed_u64(&a.tready[s]);  // a published copy is final: read with the key
        if (k == 0) {
          k = atomicCAS(reinterpret_cast<unsigned long long*>(&a.tkey[s]), 0ull, frag | row);
          if (k == 0) {  // claimed: this row represents the slot
            claimed = true;
            a.used[atomicAdd(&a.used_count[0], 1u)] = s;
            // 128-byte aligned copies: an L1 line never holds bytes of a copy not yet published
            const uint64_t need = (static_cast<uint64_t>(len) + 127) & ~127ull;
            const unsigned long long at = atomicAdd(a.copies_top, static_cast<unsigned long long>(need));
            if (at + need <= a.copies_cap) copy_at = at;  // else the slot keeps no copy (the slow compare)
            break;
          }
        }
        if ((k & 0xFFFFFFFF00000000ull) == frag) {
          rep = static_cast<uint32_t>(k);
          ready = rd;
          break;
        }
        s = (s + 1) & a.mask;
      }
      a.slot_out[row] = s;
    }

    // ---- 3. verify: 0 nothing, 1 write the slot copy, 2 compare with the copy, 3 slow compare
    uint32_t mode = 0;
    uint64_t at = 0;
    if (valid) {
      if (claimed) {
        if (copy_at != ~0ull) mode = 1, at = copy_at;
      } else if (ready != 0) {
        if (static_cast<uint32_t>(ready) != len) bad = true;  // different lengths: different names
        else mode = 2, at = ((ready >> 32) - 1) << 7;
      } else if (rep != row) {
        mode = 3;
      }
      if (len >= (1u << 30)) mode = mode == 1 ? 0u : (mode == 2 ? 3u : mode);  // keep `pk` exact
    }
    // mode and length in one word, the copy's offset in 128-byte units (copies_cap < 2^38 bytes)
    const uint32_t pk = mode | (len << 2);
    const uint32_t atu = static_cast<uint32_t>(at >> 7);
    if (__any_sync(0xffffffffu, mode == 1)) {  // claimers write their copies, then publish them
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int j = 4 * it + static_cast<int>(sub);
        const uint32_t pj = __shfl_sync(0xffffffffu, pk, j);
        const uint32_t aj = __shfl_sync(0xffffffffu, atu, j);
        const uint32_t lj = pj >> 2;
        uint32_t relj = 0;
        uint64_t oj = 0;
        if (staged) relj = __shfl_sync(0xffffffffu, rel, j);
        else oj = __shfl_sync(0xffffffffu, my_off, j);
        if ((pj & 3u) == 1u) {
          for (uint32_t q = 16 * t; q < lj; q += 128) {
            uint32_t x[4];
            if (q < 128) {
#pragma unroll
              for (int i = 0; i < 4; ++i) x[i] = xw[it][i];
            } else {
              const int v = static_cast<int>(min(16u, lj - q));
              if (staged) chunk_shared(sbuf + relj, q, x);
              else chunk_global(a.bytes + oj + q, v, x);
              if (v < 16) mask_chunk(x, v);
            }
            *reinterpret_cast<uint4*>(a.copies + (static_cast<uint64_t>(aj) << 7) + q) = make_uint4(x[0], x[1], x[2], x[3]);
          }
        }
      }
      __threadfence();
      __syncwarp();
      if (mode == 1) st_relaxed_u64(&a.tready[s], ((static_cast<uint64_t>(atu) + 1) << 32) | len);
    }
    if (short_names) {  // every name <= 128 bytes: one chunk per lane, four loads in flight at a time
      s_nm[warp][lane] = make_uint2(pk, atu);
      __syncwarp();
      uint32_t diff = 0;
#pragma unroll
      for (int h2 = 0; h2 < 8; h2 += 4) {
        uint4 y[4];
        bool use[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint2 nm = s_nm[warp][4 * (h2 + u) + sub];  // (mode | length << 2, copy unit)
          use[u] = (nm.x & 3u) == 2u && 16 * t < (nm.x >> 2);
          y[u] = make_uint4(0, 0, 0, 0);
          if (use[u]) y[u] = *reinterpret_cast<const uint4*>(a.copies + (static_cast<uint64_t>(nm.y) << 7) + 16 * t);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t d = (xw[h2 + u][0] ^ y[u].x) | (xw[h2 + u][1] ^ y[u].y) | (xw[h2 + u][2] ^ y[u].z) |
                             (xw[h2 + u][3] ^ y[u].w);
          diff |= use[u] ? d : 0u;
        }
      }
      __syncwarp();  // s_nm is rewritten by the next group
      if (diff) bad = true;
    } else {
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int j = 4 * it + static_cast<int>(sub);
        const uint32_t pj = __shfl_sync(0xffffffffu, pk, j);
        const uint32_t aj = __shfl_sync(0xffffffffu, atu, j);
        const uint32_t lj = pj >> 2;
        uint32_t relj = 0;
        uint64_t oj = 0;
        if (staged) relj = __shfl_sync(0xffffffffu, rel, j);
        else oj = __shfl_sync(0xffffffffu, my_off, j);
        uint32_t diff = 0;
        if ((pj & 3u) == 2u) {
          for (uint32_t q = 16 * t; q < lj; q += 128) {
            uint32_t x[4];
            if (q < 128) {
#pragma unroll
              for (int i = 0; i < 4; ++i) x[i] = xw[it][i];
            } else {
              const int v = static_cast<int>(min(16u, lj - q));
              if (staged) chunk_shared(sbuf + relj, q, x);
              else chunk_global(a.bytes + oj + q, v, x);
              if (v < 16) mask_chunk(x, v);
            }
            const uint4 yy = *reinterpret_cast<const uint4*>(a.copies + (static_cast<uint64_t>(aj) << 7) + q);
            diff |= (x[0] ^ yy.x) | (x[1] ^ yy.y) | (x[2] ^ yy.z) | (x[3] ^ yy.w);
          }
        }
        if (diff) bad = true;
      }
    }
    if (mode == 3) {  // the slot's copy is not published yet: compare with the representative row
      const uint64_t o = my_off;
      const uint64_t ro = a.name_off[rep];
      const uint32_t rlen = static_cast<uint32_t>(a.name_off[rep + 1] - ro);
      bool same = rlen == len;
      if (same) {
        if (rep < a.row0) {  // streamed: the representative's chunk is gone, its bytes are in the arena
          const GlobalBytes rb(a.arena + a.arena_off[s]);
          same = staged ? same_bytes(SharedBytes(buf + (o - base)), rb, len) : same_bytes(GlobalBytes(a.bytes + o), rb, len);
        } else if (staged && rep >= g0 && rep < g1) {
          same = same_bytes(SharedBytes(buf + (o - base)), SharedBytes(buf + (ro - base)), len);
        } else if (staged) {
          same = same_bytes(SharedBytes(buf + (o - base)), GlobalBytes(a.bytes + ro), len);
        } else {
          same = same_bytes(GlobalBytes(a.bytes + o), GlobalBytes(a.bytes + ro), len);
        }
      }
      if (!same) bad = true;
    }
    // device census (filter_majority_device): one ballot round per distinct id in the warp
    if (a.device) {
      uint32_t d = valid ? a.device[row] : 0xFFFFFu;
      unsigned todo = __ballot_sync(0xffffffffu, valid);
      while (todo) {
        const uint32_t d0 = __shfl_sync(0xffffffffu, d, __ffs(todo) - 1);
        const unsigned m = __ballot_sync(0xffffffffu, valid && d == d0) & todo;
        if (lane == static_cast<unsigned>(__ffs(m) - 1)) {
          if (d0 < kDevSmem) atomicAdd(&s_dev[d0], static_cast<unsigned>(__popc(m)));
          else atomicAdd(&a.dev_counts[d0], static_cast<unsigned long long>(__popc(m)));
          dev_hi = max(dev_hi, d0);
        }
        todo &= ~m;
      }
    }
    __syncwarp();
    my_off = nx_off, my_end = nx_end, cur_base = nx_base, cur_staged = nx_staged;
    cur ^= 1;
  }
  if (bad) atomicOr(&a.used_count[2], 1u);
  if (a.device) atomicMax(&s_devmax, dev_hi);
  __syncthreads();
  if (a.device) {
    for (unsigned i = threadIdx.x; i < kDevSmem; i += blockDim.x)
      if (s_dev[i]) atomicAdd(&a.dev_counts[i], static_cast<unsigned long long>(s_dev[i]));
    if (threadIdx.x == 0) atomicMax(a.dev_max, s_devmax);
  }
}

// Streamed names: after each chunk, copy the names of the slots it claimed (used[snap..count))
// into the arena, so later chunks verify against them and the classifier reads them.
__global__ void k_save_reps(const uint32_t* __restrict__ used, const uint32_t* __restrict__ snap,
                            const uint32_t* __restrict__ count, const uint64_t* __restrict__ tkey,
                            const uint64_t* __restrict__ name_off, const uint8_t* __restrict__ bytes, uint8_t* arena,
                            uint64_t arena_cap, uint64_t* __restrict__ arena_off, unsigned long long* top,
                            uint32_t* overflow) {
  const uint32_t u0 = *snap, u1 = *count;
  for (uint32_t u = u0 + blockIdx.x * blockDim.x + threadIdx.x; u < u1; u += gridDim.x * blockDim.x) {
    const uint32_t s = used[u];
    const uint32_t r = static_cast<uint32_t>(tkey[s]);
    const uint64_t o = name_off[r], len = name_off[r + 1] - o;
    const unsigned long long at = atomicAdd(top, static_cast<unsigned long long>(len));
    if (at + len > arena_cap) {
      atomicOr(overflow, 1u);
      continue;
    }
    for (uint64_t i = 0; i < len; ++i) arena[at + i] = bytes[o + i];
    arena_off[s] = at;
  }
}

// classify each distinct name once (trace.hpp:103-113): one warp per name, the lanes testing
// different start positions of each needle
__device__ __forceinline__ bool warp_contains_ci(const uint8_t* h, uint32_t hl, const char* needle, uint32_t nl) {
  bool hit = false;
  for (uint32_t base = 0; base + nl <= hl; base += 32) {  // uniform trip count across the warp
    const uint32_t i = base + lane_id();
    if (i + nl <= hl) {
      uint32_t j = 0;
      while (j < nl) {
        uint8_t ch = h[i + j];
        if (ch >= 'A' && ch <= 'Z') ch += 32;
        if (ch != static_cast<uint8_t>(needle[j])) break;
        ++j;
      }
      hit |= j == nl;
    }
  }
  return __any_sync(0xffffffffu, hit);
}

__global__ void k_classify_slots(const uint32_t* __restrict__ used, uint32_t n_used, const uint64_t* __restrict__ tkey,
                                 const uint64_t* __restrict__ name_off, const uint8_t* __restrict__ bytes,
                                 const uint8_t* __restrict__ arena, const uint64_t* __restrict__ arena_off,
                                 uint8_t* __restrict__ tflags) {
  const uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (u >= n_used) return;  // whole warps exit together
  const uint32_t s = used[u];
  const uint32_t r = static_cast<uint32_t>(tkey[s]);  // first inserter's row
  const uint8_t* p = arena ? arena + arena_off[s] : bytes + name_off[r];
  const uint32_t len = static_cast<uint32_t>(name_off[r + 1] - name_off[r]);
  uint8_t f = 0;
  if (warp_contains_ci(p, len, "memcpy", 6)) f |= NB_MEMCPY;
  if (warp_contains_ci(p, len, "htod", 4)) f |= NB_HTOD;
  if (warp_contains_ci(p, len, "dtoh", 4)) f |= NB_DTOH;
  if (warp_contains_ci(p, len, "dtod", 4)) f |= NB_DTOD;
  if (warp_contains_ci(p, len, "memset", 6)) f |= NB_MEMSET;
  if (lane_id() == 0) tflags[s] = f;
}

__global__ void k_name_bounds(const uint64_t* __restrict__ name_off, uint64_t n, uint64_t rows_per_chunk,
                              uint64_t chunks, uint64_t* __restrict__ out) {
  const uint64_t c = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c <= chunks) out[c] = name_off[min(c * rows_per_chunk, n)];
}

// kind per record and the smallest source row per slot.  Four consecutive rows per thread (one
// 16-byte slot load, one 4-byte kind store); the representative check reads trep through L1
// (ld.ca) — a stale value only costs a redundant atomicMin, which is the authority.
__global__ void k_kinds_minrow(const uint32_t* __restrict__ slot, const uint8_t* __restrict__ rflags, uint64_t n,
                               const uint8_t* __restrict__ tflags, uint8_t* __restrict__ kind, uint32_t* trep) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  // the caller's flags column may sit at any byte address: quads only when it is 4-byte aligned
  const uint64_t quads = (reinterpret_cast<uintptr_t>(rflags) & 3u) ? 0 : n / 4;
  // two quads per iteration (q, q + stride): both streaming loads are in flight before the
  // dependent table lookups
  const auto one = [&](uint64_t q, uint4 sl, uint32_t fl) {
    const uint64_t i = q * 4;
    const uint32_t s4[4] = {sl.x, sl.y, sl.z, sl.w};
    uint32_t kd = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t s = s4[u];
      kd |= static_cast<uint32_t>(kind_from(__ldg(&tflags[s]), ((fl >> (8 * u)) & ITT_REC_HAS_THROUGHPUT) != 0)) << (8 * u);
      if (__ldca(&trep[s]) > i + u) atomicMin(&trep[s], static_cast<uint32_t>(i + u));
    }
    reinterpret_cast<uint32_t*>(kind)[q] = kd;
  };
  uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; q + stride < quads; q += 2 * stride) {
    const uint4 sa = __ldcs(reinterpret_cast<const uint4*>(slot) + q);
    const uint4 sb = __ldcs(reinterpret_cast<const uint4*>(slot) + q + stride);
    const uint32_t fa = __ldcs(reinterpret_cast<const uint32_t*>(rflags) + q);
    const uint32_t fb = __ldcs(reinterpret_cast<const uint32_t*>(rflags) + q + stride);
    one(q, sa, fa);
    one(q + stride, sb, fb);
  }
  if (q < quads) one(q, __ldcs(reinterpret_cast<const uint4*>(slot) + q), __ldcs(reinterpret_cast<const uint32_t*>(rflags) + q));
  for (uint64_t i = quads * 4 + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t s = slot[i];
    kind[i] = static_cast<uint8_t>(kind_from(__ldg(&tflags[s]), (rflags[i] & ITT_REC_HAS_THROUGHPUT) != 0));
    if (__ldca(&trep[s]) > i) atomicMin(&trep[s], static_cast<uint32_t>(i));
  }
}

// The same for dictionaries of up to kKindsSmemCap slots: the slot flags and a per-CTA smallest row
// per slot in shared memory (random table reads as LDS instead of L1 wavefronts of up to 32 lines),
// folded into trep once per CTA.  1024-thread CTAs, two per SM.
constexpr uint32_t kKindsSmemCap = 16384;
__global__ void __launch_bounds__(1024) k_kinds_minrow_smem(const uint32_t* __restrict__ slot, const uint8_t* __restrict__ rflags,
                                                           uint64_t n, const uint8_t* __restrict__ tflags, uint32_t cap,
                                                           uint8_t* __restrict__ kind, uint32_t* trep) {
  extern __shared__ __align__(16) uint8_t k_sm[];
  uint32_t* s_rep = reinterpret_cast<uint32_t*>(k_sm);
  uint8_t* s_fl = k_sm + static_cast<size_t>(cap) * 4;
  for (uint32_t i = threadIdx.x; i < cap; i += blockDim.x) {
    s_rep[i] = 0xFFFFFFFFu;
    s_fl[i] = tflags[i];
  }
  __syncthreads();
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t quads = (reinterpret_cast<uintptr_t>(rflags) & 3u) ? 0 : n / 4;
  for (uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < quads; q += stride) {
    const uint64_t i = q * 4;
    const uint4 sl = __ldcs(reinterpret_cast<const uint4*>(slot) + q);
    const uint32_t fl = __ldcs(reinterpret_cast<const uint32_t*>(rflags) + q);
    const uint32_t s4[4] = {sl.x, sl.y, sl.z, sl.w};
    uint32_t kd = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t s = s4[u];
      kd |= static_cast<uint32_t>(kind_from(s_fl[s], ((fl >> (8 * u)) & ITT_REC_HAS_THROUGHPUT) != 0)) << (8 * u);
      if (s_rep[s] > i + u) atomicMin(&s_rep[s], static_cast<uint32_t>(i + u));
    }
    reinterpret_cast<uint32_t*>(kind)[q] = kd;
  }
  for (uint64_t i = quads * 4 + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t s = slot[i];
    kind[i] = static_cast<uint8_t>(kind_from(s_fl[s], (rflags[i] & ITT_REC_HAS_THROUGHPUT) != 0));
    if (s_rep[s] > i) atomicMin(&s_rep[s], static_cast<uint32_t>(i));
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < cap; i += blockDim.x)
    if (s_rep[i] != 0xFFFFFFFFu) atomicMin(&trep[i], s_rep[i]);
}

// ------------------------------------------------------------------ stream census
struct StreamEntry {
  unsigned long long key;  // stream + 1 (0 = empty)
  unsigned long long counts[6];
  unsigned long long min_start;  // order-preserving u64 of int64
  unsigned long long max_end;
};
__device__ __forceinline__ unsigned long long ord64(int64_t v) {
  return static_cast<unsigned long long>(v) ^ 0x8000000000000000ull;
}
__host__ __device__ inline int64_t unord64(unsigned long long u) { return static_cast<int64_t>(u ^ 0x8000000000000000ull); }

__device__ uint32_t global_stream_slot(StreamEntry* table, uint32_t* list, uint32_t* count, unsigned long long key) {
  uint32_t s = static_cast<uint32_t>(key * 0x9E3779B1u) & (kStreamTableCap - 1);
  for (uint32_t probe = 0; probe < kStreamTableCap; ++probe) {
    unsigned long long k = atomicAdd(&table[s].key, 0ull);
    if (k == 0) {
      k = atomicCAS(&table[s].key, 0ull, key);
      if (k == 0) {
        list[atomicAdd(count, 1u)] = s;
        return s;
      }
    }
    if (k == key) return s;
    s = (s + 1) & (kStreamTableCap - 1);
  }
  return kNone;
}

struct CensusArgs {
  uint64_t n;
  const uint32_t* stream;
  const uint16_t* device;
  int filter;  // keep only device == majority
  uint16_t majority;
  const uint8_t* kind;
  const int64_t* start;
  const int64_t* dur;
  StreamEntry* table;
  uint32_t* list;
  uint32_t* count;
};

__global__ void __launch_bounds__(256) k_stream_census(CensusArgs a) {
  __shared__ unsigned long long s_key[kBlockStreams];
  __shared__ unsigned int s_cnt[kBlockStreams][6];
  __shared__ unsigned long long s_min[kBlockStreams], s_max[kBlockStreams];
  for (unsigned i = threadIdx.x; i < kBlockStreams; i += blockDim.x) {
    s_key[i] = 0;
    s_min[i] = ~0ull;
    s_max[i] = 0;
    for (int k = 0; k < 6; ++k) s_cnt[i][k] = 0;
  }
  __syncthreads();
  const unsigned lane = lane_id();
  // one row per lane per round: the stream's block slot by match_any, counts / min start / max end
  // reduced over the lanes of the same stream
  const auto row = [&](bool valid, uint32_t st, int kd, int64_t s0, int64_t e0) {
    const unsigned long long key = static_cast<unsigned long long>(st) + 1ull;
    uint32_t bs = kNone;
    const unsigned peers = __match_any_sync(0xffffffffu, valid ? key : 0ull);
    const int leader = __ffs(peers) - 1;
    if (valid && static_cast<int>(lane) == leader) {
      uint32_t s = static_cast<uint32_t>(key * 0x9E3779B1u) & (kBlockStreams - 1);
      for (uint32_t probe = 0; probe < kBlockStreams; ++probe) {
        unsigned long long k = s_key[s];
        if (k == 0) {
          k = atomicCAS(&s_key[s], 0ull, key);
          if (k == 0) k = key;
        }
        if (k == key) {
          bs = s;
          break;
        }
        s = (s + 1) & (kBlockStreams - 1);
      }
    }
    bs = __shfl_sync(0xffffffffu, bs, leader);
    if (!valid) return;
    if (bs == kNone) {  // block table overflow: update the global table directly
      const uint32_t gs = global_stream_slot(a.table, a.list, a.count, key);
      if (gs != kNone) {
        atomicAdd(&a.table[gs].counts[kd], 1ull);
        atomicMin(&a.table[gs].min_start, ord64(s0));
        atomicMax(&a.table[gs].max_end, ord64(e0));
      }
      return;
    }
    const unsigned kp = __match_any_sync(peers, static_cast<unsigned>(kd));
    if (static_cast<int>(lane) == __ffs(kp) - 1) atomicAdd(&s_cnt[bs][kd], static_cast<unsigned>(__popc(kp)));
    // min start / max end over the stream's lanes: reduce 32-bit halves
    const unsigned long long us = ord64(s0), ue = ord64(e0);
    const unsigned hs = __reduce_min_sync(peers, static_cast<unsigned>(us >> 32));
    const unsigned ls = __reduce_min_sync(peers, static_cast<unsigned>(us >> 32) == hs ? static_cast<unsigned>(us) : ~0u);
    const unsigned he = __reduce_max_sync(peers, static_cast<unsigned>(ue >> 32));
    const unsigned le = __reduce_max_sync(peers, static_cast<unsigned>(ue >> 32) == he ? static_cast<unsigned>(ue) : 0u);
    if (static_cast<int>(lane) == leader) {
      atomicMin(&s_min[bs], (static_cast<unsigned long long>(hs) << 32) | ls);
      atomicMax(&s_max[bs], (static_cast<unsigned long long>(he) << 32) | le);
    }
  };
  // four consecutive rows per thread with 16-byte loads when the columns are aligned
  const bool vec = ((reinterpret_cast<uintptr_t>(a.stream) | reinterpret_cast<uintptr_t>(a.start) |
                     (a.dur ? reinterpret_cast<uintptr_t>(a.dur) : 0)) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(a.kind) & 3) == 0 &&
                   (!a.filter || (reinterpret_cast<uintptr_t>(a.device) & 7) == 0);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x * 4;
  for (uint64_t b = static_cast<uint64_t>(blockIdx.x) * blockDim.x * 4; b < a.n; b += stride) {
    const uint64_t i0 = b + threadIdx.x * 4;
    uint32_t st[4] = {0, 0, 0, 0};
    int kd[4] = {0, 0, 0, 0};
    int64_t s0[4] = {0, 0, 0, 0}, e0[4] = {0, 0, 0, 0};
    bool valid[4];
    if (vec && i0 + 4 <= a.n) {
      const uint4 sv = __ldcs(reinterpret_cast<const uint4*>(a.stream + i0));
      const uint32_t kv = __ldcs(reinterpret_cast<const uint32_t*>(a.kind + i0));
      const longlong2 t0 = __ldcs(reinterpret_cast<const longlong2*>(a.start + i0));
      const longlong2 t1 = __ldcs(reinterpret_cast<const longlong2*>(a.start + i0 + 2));
      st[0] = sv.x, st[1] = sv.y, st[2] = sv.z, st[3] = sv.w;
      s0[0] = t0.x, s0[1] = t0.y, s0[2] = t1.x, s0[3] = t1.y;
      if (a.dur) {
        const longlong2 d0 = __ldcs(reinterpret_cast<const longlong2*>(a.dur + i0));
        const longlong2 d1 = __ldcs(reinterpret_cast<const longlong2*>(a.dur + i0 + 2));
        e0[0] = s0[0] + d0.x, e0[1] = s0[1] + d0.y, e0[2] = s0[2] + d1.x, e0[3] = s0[3] + d1.y;
      } else {  // no durations yet (late): ends come later
#pragma unroll
        for (int e = 0; e < 4; ++e) e0[e] = s0[e];
      }
      uint2 dv = make_uint2(0, 0);
      if (a.filter) dv = __ldcs(reinterpret_cast<const uint2*>(a.device + i0));
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        kd[e] = static_cast<int>((kv >> (8 * e)) & 0xFFu);
        const uint32_t dev = ((e < 2 ? dv.x : dv.y) >> (16 * (e & 1))) & 0xFFFFu;
        valid[e] = !(a.filter && dev != a.majority);
      }
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint64_t i = i0 + e;
        valid[e] = i < a.n;
        if (valid[e] && a.filter && a.device[i] != a.majority) valid[e] = false;
        if (valid[e]) {
          st[e] = a.stream[i];
          kd[e] = a.kind[i];
          s0[e] = a.start[i];
          e0[e] = a.dur ? s0[e] + a.dur[i] : s0[e];
        }
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) row(valid[e], valid[e] ? st[e] : 0u, kd[e], s0[e], e0[e]);
  }
  __syncthreads();
  for (unsigned i = threadIdx.x; i < kBlockStreams; i += blockDim.x) {
    if (!s_key[i]) continue;
    const uint32_t gs = global_stream_slot(a.table, a.list, a.count, s_key[i]);
    if (gs == kNone) continue;
    for (int k = 0; k < 6; ++k)
      if (s_cnt[i][k]) atomicAdd(&a.table[gs].counts[k], static_cast<unsigned long long>(s_cnt[i][k]));
    atomicMin(&a.table[gs].min_start, s_min[i]);
    atomicMax(&a.table[gs].max_end, s_max[i]);
  }
}

// dense copy of the used census entries: out[0].key = count, out[1 + u] = entry of list slot u
__global__ void k_pack_streams(const StreamEntry* __restrict__ table, const uint32_t* __restrict__ list,
                               StreamEntry* __restrict__ out) {
  const uint32_t ns = list[0];
  if (threadIdx.x == 0) out[0].key = ns;
  for (uint32_t u = threadIdx.x; u < ns; u += blockDim.x) out[1 + u] = table[list[1 + u]];
}

__global__ void k_init_stream_table(StreamEntry* t, uint32_t* list, uint32_t list_n) {  // + zeroes the list
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < list_n; i += gridDim.x * blockDim.x) list[i] = 0;
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < kStreamTableCap) {
    t[i].key = 0;
    for (int k = 0; k < 6; ++k) t[i].counts[k] = 0;
    t[i].min_start = ~0ull;
    t[i].max_end = 0;
  }
}

// ------------------------------------------------------------------ K3: compaction
struct CompactF {
  uint64_t n;
  const uint32_t* perm;  // sorted position -> row (null: identity)
  const uint32_t* stream;
  const uint16_t* device;
  int filter;
  uint16_t majority;
  uint32_t main_stream;
  const uint8_t* kind;
  const uint32_t* slot;
  const int64_t* start;
  const int64_t* dur;
  const int64_t* size;
  const uint8_t* rflags;
  uint32_t* tok_slot;
  int64_t* tok_start;
  int64_t* tok_end;
  uint8_t* tok_kind;
  uint64_t* tok_record;  // optional
  uint32_t* tfirst;
  int64_t* htod_start;
  int64_t* htod_end;
  int64_t* htod_size;
  unsigned long long* htod_range;
  int ends_only;  // late durations: only tok_end / htod_end and the HtoD end range (the rest is written)
  __device__ __forceinline__ uint32_t row(uint64_t k) const { return perm ? perm[k] : static_cast<uint32_t>(k); }
  __device__ __forceinline__ uint64_t load(uint64_t k) const {
    const uint32_t i = row(k);
    if (filter && device[i] != majority) return 0;
    const uint64_t m = stream[i] == main_stream ? 1ull : 0ull;
    const uint64_t h = kind[i] == ITT_KIND_HTOD ? (1ull << 31) : 0ull;
    return m | h;
  }
  __device__ __forceinline__ void store(uint64_t k, uint64_t excl, uint64_t v) const {
    if (!v) return;
    const uint32_t i = row(k);
    const int64_t s = start[i];
    const int64_t e = s + dur[i];
    if (v & 1ull) {
      const uint32_t j = static_cast<uint32_t>(excl & 0x7FFFFFFFull);
      const uint32_t sl = slot[i];
      tok_slot[j] = sl;
      tok_start[j] = s;
      tok_end[j] = e;
      tok_kind[j] = kind[i];
      if (tok_record) tok_record[j] = k;
      if (__ldcg(&tfirst[sl]) > j) atomicMin(&tfirst[sl], j);
    }
    if (v >> 31) {
      const uint64_t h = excl >> 31;
      htod_start[h] = s;
      htod_end[h] = e;
      htod_size[h] = (rflags[i] & ITT_REC_HAS_SIZE) ? size[i] : 0;
      const unsigned long long fe = static_cast<unsigned long long>(e) ^ (1ull << 63);
      atomicMin(&htod_range[0], fe);
      atomicMax(&htod_range[1], fe);
    }
  }
};

// Compaction of rows already in (start, row) order by reduce-then-scan: (1) per-tile counts, (2) one
// block scans the tile counts, (3) every tile writes at its known offset.  No tile waits on a
// look-back chain (the single-pass kernel's CTAs sat at the barrier behind warp 0's look-back);
// the price is a second read of the 5-7 bytes per row that decide main-stream / HtoD.
constexpr int kRSItems = 8, kRSTile = 256 * kRSItems;
struct RowSel {  // the selection ballots of one warp's rows (warp-striped: row = wbase + q*32 + lane)
  unsigned mm[kRSItems], hm[kRSItems];
  uint8_t kd[kRSItems];
  __device__ __forceinline__ void load(const CompactF& f, uint64_t wbase) {
#pragma unroll
    for (int q = 0; q < kRSItems; ++q) {
      const uint64_t k = wbase + q * 32 + lane_id();
      bool m = false, h = false;
      kd[q] = 0;
      if (k < f.n) {
        const uint32_t sm = __ldcs(&f.stream[k]);
        kd[q] = __ldcs(&f.kind[k]);
        const bool keep = !(f.filter && __ldcs(&f.device[k]) != f.majority);
        m = keep && sm == f.main_stream;
        h = keep && kd[q] == ITT_KIND_HTOD;
      }
      mm[q] = __ballot_sync(0xffffffffu, m);
      hm[q] = __ballot_sync(0xffffffffu, h);
    }
  }
  __device__ __forceinline__ uint64_t packed() const {
    uint64_t m = 0, h = 0;
#pragma unroll
    for (int q = 0; q < kRSItems; ++q) m += __popc(mm[q]), h += __popc(hm[q]);
    return m | (h << 31);
  }
};
__global__ void __launch_bounds__(256) k_compact_count(CompactF f, uint64_t* __restrict__ tile_counts) {
  __shared__ uint64_t s_w[8];
  const unsigned warp = threadIdx.x >> 5;
  const uint64_t wbase = static_cast<uint64_t>(blockIdx.x) * kRSTile + warp * (32 * kRSItems);
  uint64_t packed;
  if (!f.filter && wbase + 32 * kRSItems <= f.n && kRSItems == 8 && (reinterpret_cast<uintptr_t>(f.stream) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(f.kind) & 7) == 0) {
    // only the totals matter here: 8 consecutive rows per lane, 16-byte stream / 8-byte kind loads
    const uint64_t r0 = wbase + lane_id() * 8;
    const uint4 s0 = __ldcs(reinterpret_cast<const uint4*>(f.stream + r0));
    const uint4 s1 = __ldcs(reinterpret_cast<const uint4*>(f.stream + r0 + 4));
    const uint2 k8 = __ldcs(reinterpret_cast<const uint2*>(f.kind + r0));
    const uint32_t sv[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
    uint32_t m = 0, h = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      m += sv[q] == f.main_stream;
      h += ((q < 4 ? k8.x >> (8 * q) : k8.y >> (8 * (q - 4))) & 0xFFu) == ITT_KIND_HTOD;
    }
    m = __reduce_add_sync(0xffffffffu, m);
    h = __reduce_add_sync(0xffffffffu, h);
    packed = static_cast<uint64_t>(m) | (static_cast<uint64_t>(h) << 31);
  } else {
    RowSel sel;
    sel.load(f, wbase);
    packed = sel.packed();
  }
  if (lane_id() == 0) s_w[warp] = packed;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
    for (int w = 0; w < 8; ++w) t += s_w[w];
    tile_counts[blockIdx.x] = t;
  }
}
// exclusive scan of the tile counts in place, one block walking chunks of 8K counts (8 consecutive
// per thread, coalesced) with a running carry (C3: 49K tiles, C5: 489K)
__global__ void __launch_bounds__(1024) k_scan_tile_counts(uint64_t* __restrict__ tc, uint64_t tiles) {
  __shared__ uint64_t s_warp[32];
  constexpr int kPer = 8;
  uint64_t carry = 0;
  for (uint64_t c0 = 0; c0 < tiles; c0 += 1024 * kPer) {
    const uint64_t b0 = c0 + static_cast<uint64_t>(threadIdx.x) * kPer;
    uint64_t v[kPer], run = 0;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      v[q] = b0 + q < tiles ? tc[b0 + q] : 0ull;
      run += v[q];
    }
    uint64_t total;
    uint64_t acc = carry + block_exclusive_scan<uint64_t, SumOp<uint64_t>, 1024>(run, SumOp<uint64_t>(), &total, s_warp);
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      if (b0 + q < tiles) tc[b0 + q] = acc;
      acc += v[q];
    }
    carry += total;
    __syncthreads();  // s_warp is reused by the next chunk
  }
}
#ifndef ITT_COMPACT_MINB
#define ITT_COMPACT_MINB 4  // 64 registers, 4 CTAs per SM (C3 A/B: 1.22 ms with the default cap, 1.17 at 4, 1.60 at 6)
#endif
__global__ void __launch_bounds__(256, ITT_COMPACT_MINB) k_compact_write(CompactF f, const uint64_t* __restrict__ tile_excl) {
  __shared__ uint64_t s_w[8];
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const uint64_t wbase = static_cast<uint64_t>(blockIdx.x) * kRSTile + warp * (32 * kRSItems);
  uint64_t excl = __ldg(&tile_excl[blockIdx.x]);  // ready before launch: no round trip after the barrier
  RowSel sel;
  sel.load(f, wbase);
  // the columns the outputs need (main-stream / HtoD rows only), in flight during the block scan
  int64_t st[kRSItems], du[kRSItems];
  uint32_t sl[kRSItems];
#pragma unroll
  for (int q = 0; q < kRSItems; ++q) {
    const uint64_t k = wbase + q * 32 + lane;
    st[q] = du[q] = 0, sl[q] = 0;
    if ((sel.mm[q] | sel.hm[q]) >> lane & 1u) {
      st[q] = __ldcs(&f.start[k]);
      du[q] = f.dur ? __ldcs(&f.dur[k]) : 0;  // null: late durations (the ends pass writes tok_end)
    }
    if (!f.ends_only && (sel.mm[q] >> lane & 1u)) sl[q] = __ldcs(&f.slot[k]);
  }
  // first-appearance filter values in flight across the barrier
  uint32_t tf[kRSItems];
#pragma unroll
  for (int q = 0; q < kRSItems; ++q) tf[q] = (!f.ends_only && (sel.mm[q] >> lane & 1u)) ? __ldcg(&f.tfirst[sl[q]]) : 0u;
  if (lane == 0) s_w[warp] = sel.packed();
  __syncthreads();
  for (unsigned w = 0; w < warp; ++w) excl += s_w[w];
  uint32_t jm = static_cast<uint32_t>(excl & 0x7FFFFFFFull);
  uint64_t jh = excl >> 31;
  const unsigned lt = lanemask_lt();
  unsigned long long emin = ~0ull, emax = 0;
#pragma unroll
  for (int q = 0; q < kRSItems; ++q) {
    const int64_t en = st[q] + du[q];
    if (sel.mm[q] >> lane & 1u) {
      const uint32_t j = jm + __popc(sel.mm[q] & lt);
      f.tok_end[j] = en;
      if (!f.ends_only) {
        f.tok_slot[j] = sl[q];
        f.tok_start[j] = st[q];
        f.tok_kind[j] = sel.kd[q];
        if (f.tok_record) f.tok_record[j] = wbase + q * 32 + lane;
        if (tf[q] > j) atomicMin(&f.tfirst[sl[q]], j);
      }
    }
    if (sel.hm[q] >> lane & 1u) {
      const uint64_t h = jh + __popc(sel.hm[q] & lt);
      const uint64_t i = wbase + q * 32 + lane;
      f.htod_end[h] = en;
      if (!f.ends_only) {
        f.htod_start[h] = st[q];
        f.htod_size[h] = (f.rflags[i] & ITT_REC_HAS_SIZE) ? f.size[i] : 0;
      }
      const unsigned long long fe = static_cast<unsigned long long>(en) ^ (1ull << 63);
      emin = fe < emin ? fe : emin;
      emax = fe > emax ? fe : emax;
    }
    jm += __popc(sel.mm[q]);
    jh += __popc(sel.hm[q]);
  }
  if (__any_sync(0xffffffffu, emax != 0)) {  // HtoD end range: one pair of atomics per warp
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long a = __shfl_xor_sync(0xffffffffu, emin, o), b = __shfl_xor_sync(0xffffffffu, emax, o);
      emin = a < emin ? a : emin;
      emax = b > emax ? b : emax;
    }
    if (lane == 0) {
      atomicMin(&f.htod_range[0], emin);
      atomicMax(&f.htod_range[1], emax);
    }
  }
}

// Compaction when the row order is block-local (rows already sorted, or the 256-row block sort
// was the whole order): a tile of 2048 sorted positions reads exactly the source rows of the same
// range, so the tile stages stream / device / kind / slot / start / dur in shared memory with
// coalesced loads and resolves the permutation there, instead of one scattered global gather
// per column per record.  Same outputs as CompactF (one packed look-back scan).
#ifndef ITT_COMPACT_ITEMS
#define ITT_COMPACT_ITEMS 4
#endif
constexpr int kCompactBlock = 256, kCompactItems = ITT_COMPACT_ITEMS, kCompactTile = kCompactBlock * kCompactItems;
static_assert(kCompactTile % 256 == 0, "tiles must be whole order blocks");
struct CompactLocalSmem {
  int64_t start[kCompactTile];
  int64_t dur[kCompactTile];
  uint32_t stream[kCompactTile];
  uint32_t slot[kCompactTile];
  uint16_t device[kCompactTile];
  uint8_t kind[kCompactTile];
};
__global__ void __launch_bounds__(kCompactBlock) k_compact_local(CompactF f, uint64_t* status, uint32_t* tile_counter) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CompactLocalSmem& S = *reinterpret_cast<CompactLocalSmem*>(smem_raw);
  __shared__ uint64_t s_warp[kCompactBlock / 32];
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t r0 = static_cast<uint64_t>(tile) * kCompactTile;
  const uint32_t len = static_cast<uint32_t>(umin64(kCompactTile, f.n - r0));
  {  // coalesced: the source rows of this tile, every load in flight before the first store
    int64_t st[kCompactItems], du[kCompactItems];
    uint32_t sm[kCompactItems], sl[kCompactItems];
    uint8_t kd[kCompactItems];
#pragma unroll
    for (int q = 0; q < kCompactItems; ++q) {
      const uint32_t i = threadIdx.x + q * kCompactBlock;
      if (i < len) {
        const uint64_t r = r0 + i;
        st[q] = __ldcs(&f.start[r]);
        du[q] = __ldcs(&f.dur[r]);
        sm[q] = __ldcs(&f.stream[r]);
        sl[q] = __ldcs(&f.slot[r]);
        kd[q] = f.kind[r];
      }
    }
#pragma unroll
    for (int q = 0; q < kCompactItems; ++q) {
      const uint32_t i = threadIdx.x + q * kCompactBlock;
      if (i < len) {
        S.start[i] = st[q];
        S.dur[i] = du[q];
        S.stream[i] = sm[q];
        S.slot[i] = sl[q];
        S.kind[i] = kd[q];
        if (f.filter) S.device[i] = f.device[r0 + i];
      }
    }
  }
  __syncthreads();
  // warp-striped positions (k = r0 + warp*256 + q*32 + lane): ballots give every prefix, and
  // consecutive lanes write consecutive outputs (coalesced token columns)
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const uint64_t wbase = r0 + static_cast<uint64_t>(warp) * (32 * kCompactItems);
  const unsigned lt = lanemask_lt();
  unsigned mm[kCompactItems], hm[kCompactItems];
  uint32_t loc[kCompactItems];
  uint32_t wm = 0, wh = 0;
#pragma unroll
  for (int q = 0; q < kCompactItems; ++q) {
    const uint64_t k = wbase + q * 32 + lane;
    bool is_main = false, is_htod = false;
    loc[q] = 0;
    if (k < f.n) {
      const uint32_t il = f.perm ? static_cast<uint32_t>(__ldcs(&f.perm[k]) - r0) : static_cast<uint32_t>(k - r0);
      loc[q] = il;
      if (!(f.filter && S.device[il] != f.majority)) {
        is_main = S.stream[il] == f.main_stream;
        is_htod = S.kind[il] == ITT_KIND_HTOD;
      }
    }
    mm[q] = __ballot_sync(0xffffffffu, is_main);
    hm[q] = __ballot_sync(0xffffffffu, is_htod);
    wm += __popc(mm[q]);
    wh += __popc(hm[q]);
  }
  const uint64_t wtot = static_cast<uint64_t>(wm) | (static_cast<uint64_t>(wh) << 31);
  // block scan over the warps' packed totals (one value per warp: lane 0 contributes)
  uint64_t total;
  const uint64_t wexcl =
      block_exclusive_scan<uint64_t, SumOp<uint64_t>, kCompactBlock>(lane == 0 ? wtot : 0ull, SumOp<uint64_t>(), &total, s_warp);
  if (threadIdx.x < 32) {
    const uint64_t p = tile_lookback<uint64_t, SumOp<uint64_t>>(status, tile, total, SumOp<uint64_t>());
    if (threadIdx.x == 0) s_prefix = p;
  }
  __syncthreads();
  const uint64_t start_acc = s_prefix + __shfl_sync(0xffffffffu, wexcl, 0);
  uint32_t jm = static_cast<uint32_t>(start_acc & 0x7FFFFFFFull);
  uint64_t jh = start_acc >> 31;
  // first-appearance candidates: all eight tfirst reads in flight before any compare
  uint32_t tf[kCompactItems];
#pragma unroll
  for (int q = 0; q < kCompactItems; ++q)
    tf[q] = (mm[q] >> lane & 1u) ? __ldcg(&f.tfirst[S.slot[loc[q]]]) : 0u;
#pragma unroll
  for (int q = 0; q < kCompactItems; ++q) {
    const uint32_t il = loc[q];
    if ((mm[q] | hm[q]) >> lane & 1u) {
      const int64_t st = S.start[il];
      const int64_t en = st + S.dur[il];
      if (mm[q] >> lane & 1u) {
        const uint32_t j = jm + __popc(mm[q] & lt);
        const uint32_t sl = S.slot[il];
        f.tok_slot[j] = sl;
        f.tok_start[j] = st;
        f.tok_end[j] = en;
        f.tok_kind[j] = S.kind[il];
        if (f.tok_record) f.tok_record[j] = wbase + q * 32 + lane;
        if (tf[q] > j) atomicMin(&f.tfirst[sl], j);
      }
      if (hm[q] >> lane & 1u) {
        const uint64_t h = jh + __popc(hm[q] & lt);
        const uint64_t i = r0 + il;
        f.htod_start[h] = st;
        f.htod_end[h] = en;
        f.htod_size[h] = (f.rflags[i] & ITT_REC_HAS_SIZE) ? f.size[i] : 0;
        const unsigned long long fe = static_cast<unsigned long long>(en) ^ (1ull << 63);
        atomicMin(&f.htod_range[0], fe);
        atomicMax(&f.htod_range[1], fe);
      }
    }
    jm += __popc(mm[q]);
    jh += __popc(hm[q]);
  }
}

// ------------------------------------------------------------------ renumber
// rank of each used slot among slots with a main-stream first position (first-appearance id)
__global__ void k_rank_slots(const uint32_t* __restrict__ used, uint32_t n_used, const uint32_t* __restrict__ tfirst,
                             uint32_t* __restrict__ id_of_slot, uint32_t* __restrict__ name_count) {
  __shared__ uint32_t s_first[1024];
  const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t my = u < n_used ? tfirst[used[u]] : kNone;
  uint32_t less = 0;
  for (uint32_t t0 = 0; t0 < n_used; t0 += 1024) {
    __syncthreads();
    for (uint32_t q = threadIdx.x; q < 1024; q += blockDim.x)
      s_first[q] = t0 + q < n_used ? tfirst[used[t0 + q]] : kNone;
    __syncthreads();
    const uint32_t lim = min(1024u, n_used - t0);
    if (my != kNone)
      for (uint32_t q = 0; q < lim; ++q) less += s_first[q] < my;
  }
  if (u < n_used) {
    id_of_slot[used[u]] = my == kNone ? kNone : less;
    if (my != kNone) atomicAdd(name_count, 1u);
  }
}

__global__ void k_slot_ids_from_sorted(const uint32_t* __restrict__ sorted_slots, uint32_t m,
                                       uint32_t* __restrict__ id_of_slot) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < m) id_of_slot[sorted_slots[r]] = r;
}

__global__ void k_first_pairs(const uint32_t* __restrict__ used, uint32_t n_used, const uint32_t* __restrict__ tfirst,
                              uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u < n_used) {
    keys[u] = tfirst[used[u]];
    vals[u] = used[u];
  }
}

// 4 tokens per thread (16-byte loads and stores; both arrays come from the pool, 16-byte aligned)
__global__ void k_map_tokens(const uint32_t* __restrict__ tok_slot, uint64_t n, const uint32_t* __restrict__ id_of_slot,
                             int32_t* __restrict__ tokens) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x * 4;
  for (uint64_t j = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4; j < n; j += stride) {
    if (j + 4 <= n) {
      const uint4 sl = __ldcs(reinterpret_cast<const uint4*>(tok_slot + j));
      __stcs(reinterpret_cast<int4*>(tokens + j),
             make_int4(static_cast<int32_t>(__ldg(&id_of_slot[sl.x])), static_cast<int32_t>(__ldg(&id_of_slot[sl.y])),
                       static_cast<int32_t>(__ldg(&id_of_slot[sl.z])), static_cast<int32_t>(__ldg(&id_of_slot[sl.w]))));
    } else {
      for (uint64_t q = j; q < n; ++q) tokens[q] = static_cast<int32_t>(id_of_slot[tok_slot[q]]);
    }
  }
}

__global__ void k_name_rows(const uint32_t* __restrict__ used, uint32_t n_used, const uint32_t* __restrict__ id_of_slot,
                            const uint32_t* __restrict__ trep, uint64_t* __restrict__ name_row) {
  const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u < n_used) {
    const uint32_t id = id_of_slot[used[u]];
    if (id != kNone) name_row[id] = trep[used[u]];
  }
}

__global__ void k_overlaps(const int64_t* __restrict__ ts, const int64_t* __restrict__ te, uint64_t n,
                           unsigned long long* out) {
  unsigned long long c = 0;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j + 1 < n; j += stride)
    c += te[j] > ts[j + 1];
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane_id() == 0 && c) atomicAdd(out, c);
}

}  // namespace

// ------------------------------------------------------------------ host side
void upload_records(Ctx* c, const itt_records* r, DevRecords& d, bool allow_late_dur) {
  d.n = r->n;
  d.order = r->order;
  const uint64_t n = r->n;
  if (r->mem < ITT_MEM_HOST || r->mem > ITT_MEM_DEVICE_HOST_NAMES)
    fail(ITT_E_INVALID_ARGUMENT, "ingest: unknown itt_records.mem");
  const bool streamed = r->mem == ITT_MEM_HOST_STREAM_NAMES || r->mem == ITT_MEM_DEVICE_HOST_NAMES;
  if (streamed) d.host_names = r->name_bytes;
  if (r->mem == ITT_MEM_DEVICE || r->mem == ITT_MEM_DEVICE_HOST_NAMES) {
    d.start = r->start_ns;
    d.dur = r->duration_ns;
    d.size = r->size_bytes;
    d.flags = r->flags;
    d.stream = r->stream;
    d.device = r->device;
    d.name_off = r->name_off;
    d.name_bytes = streamed ? nullptr : r->name_bytes;
    return;
  }
  uint64_t nb = 0;
  if (n) std::memcpy(&nb, &r->name_off[n], sizeof(nb));
  d.name_total = static_cast<int64_t>(nb);
  // Large host traces: only `start` goes first on the compute stream (the order stage needs nothing
  // else); the other columns follow on the copy stream while the order stage runs, and the names
  // are streamed in 64 MiB chunks behind them, each hashed as soon as it lands — the PCIe transfer
  // overlaps the first stages instead of preceding them.
  uint64_t overlap_min = 256ull << 20;
  if (const char* e = std::getenv("ITT_TEST_OVERLAP_MIN"); e && *e) overlap_min = std::strtoull(e, nullptr, 10);  // tests
  // (streamed names keep their own chunking; their columns take the same two-stream copy)
  const bool overlap = (r->mem == ITT_MEM_HOST || r->mem == ITT_MEM_HOST_STREAM_NAMES) && nb >= overlap_min;
  if (overlap && r->mem == ITT_MEM_HOST) {
    d.host_names = r->name_bytes;
    d.stream_chunk = 64ull << 20;
  }
  // sizes are read only for HtoD records (the compaction's htod_size): from pinned host memory the
  // kernels read them in place (zero-copy) instead of copying the whole column over PCIe (8 B/record)
  const int64_t* size_mapped = nullptr;
  if (n) {
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, r->size_bytes) == cudaSuccess) {
      if (pa.type == cudaMemoryTypeHost && pa.devicePointer) size_mapped = static_cast<const int64_t*>(pa.devicePointer);
    } else {
      cudaGetLastError();
    }
  }
  // late durations: a pinned duration column of an analyze goes last over PCIe (after the names),
  // overlapping the suffix array; only a census end and the token ends need it, later
  if (overlap && allow_late_dur && n) {
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, r->duration_ns) == cudaSuccess) {
      if (pa.type == cudaMemoryTypeHost) d.dur_host = r->duration_ns;
    } else {
      cudaGetLastError();
    }
  }
  d.o_start.alloc(c, n);
  d.o_dur.alloc(c, n);
  if (!size_mapped) d.o_size.alloc(c, n);
  d.o_flags.alloc(c, n);
  d.o_stream.alloc(c, n);
  d.o_off.alloc(c, n + 1);
  if (r->device) d.o_device.alloc(c, n);
  if (!streamed && !overlap) d.o_names.alloc(c, nb + 16);
  h2d_bulk(c, d.o_start.p, r->start_ns, n * 8);
  cudaStream_t cs = c->stream;
  if (overlap) {
    cs = c->copier();
    ITT_CUDA(cudaEventCreateWithFlags(&d.cols_ready, cudaEventDisableTiming));
    ITT_CUDA(cudaEventRecord(d.cols_ready, c->stream));  // the allocations above are stream-ordered
    ITT_CUDA(cudaStreamWaitEvent(cs, d.cols_ready, 0));
  }
  h2d_bulk(c, d.o_off.p, r->name_off, (n + 1) * 8, cs);
  if (!d.dur_host) h2d_bulk(c, d.o_dur.p, r->duration_ns, n * 8, cs);
  if (!size_mapped) h2d_bulk(c, d.o_size.p, r->size_bytes, n * 8, cs);
  h2d_bulk(c, d.o_flags.p, r->flags, n, cs);
  h2d_bulk(c, d.o_stream.p, r->stream, n * 4, cs);
  if (r->device) h2d_bulk(c, d.o_device.p, r->device, n * 2, cs);
  if (!streamed && !overlap) h2d_bulk(c, d.o_names.p, r->name_bytes, nb, cs);
  if (overlap) ITT_CUDA(cudaEventRecord(d.cols_ready, cs));  // the compute stream waits before the dictionary
  d.start = d.o_start.p;
  d.dur = d.o_dur.p;
  d.size = size_mapped ? size_mapped : d.o_size.p;
  d.flags = d.o_flags.p;
  d.stream = d.o_stream.p;
  d.name_off = d.o_off.p;
  d.name_bytes = (streamed || overlap) ? nullptr : d.o_names.p;
  d.device = r->device ? d.o_device.p : nullptr;
}

static std::vector<StreamEntry> census_pass(TraceState& t, const int64_t* dur);

void issue_late_durations(TraceState& t) {
  DevRecords& d = t.rec;
  if (!d.dur_host || d.dur_ready) return;
  Ctx* c = t.c;
  cudaStream_t cp = c->copier();  // after the columns and names queued on it (the buffer is allocated)
  ITT_CUDA(cudaEventCreateWithFlags(&d.dur_ready, cudaEventDisableTiming));
  ITT_CUDA(cudaMemcpyAsync(d.o_dur.p, d.dur_host, d.n * 8, cudaMemcpyHostToDevice, cp));
  ITT_CUDA(cudaEventRecord(d.dur_ready, cp));
}

void finish_late_durations(TraceState& t) {
  DevRecords& d = t.rec;
  if (!d.dur_host) return;
  Ctx* c = t.c;
  issue_late_durations(t);
  ITT_CUDA(cudaStreamWaitEvent(c->stream, d.dur_ready, 0));
  d.dur_host = nullptr;
  const uint64_t n = d.n;
  if (d.compact_ends_late) {  // the same selection and tile offsets; ends only
    d.compact_ends_late = false;
    Fills fz(c);
    fz.add(t.htod_range.p, 8, 0xFF);
    fz.add(t.htod_range.p + 1, 8, 0);
    fz.flush();
    CompactF f{n, nullptr, d.stream, d.device, t.filtering ? 1 : 0, t.majority, t.main_stream, t.kind.p, nullptr,
               d.start, d.dur, d.size, d.flags, nullptr, nullptr, t.tok_end.p, nullptr, nullptr, nullptr,
               nullptr, t.htod_end.p, nullptr, t.htod_range.p, 1};
    const uint64_t tiles = (n + kRSTile - 1) / kRSTile;
    launch(c, "compact_ends", n * (t.filtering ? 7.0 : 5.0) + t.n_tok * 24.0 + t.n_htod * 24.0, k_compact_write,
           dim3(static_cast<unsigned>(tiles)), dim3(256), 0, f, t.compact_tiles.p);
    t.compact_tiles.release();
  }
  if (d.census_ends_late) {  // a second census pass with durations: each stream's last end
    d.census_ends_late = false;
    const std::vector<StreamEntry> all = census_pass(t, d.dur);
    for (size_t u = 1; u < all.size(); ++u) {
      const uint32_t st = static_cast<uint32_t>(all[u].key - 1);
      for (auto& o : t.streams)
        if (o.stream == st) o.last_end = unord64(all[u].max_end);
    }
  }
}

void release_rows_but_late(TraceState& t) {  // all but what finish_late_durations reads
  t.perm.release();
  t.slot.release();
  t.tok_slot.release();
  t.tfirst.release();
  DevRecords& d = t.rec;
  d.o_size.release(), d.o_flags.release(), d.o_names.release(), d.o_off.release();
  d.size = nullptr, d.flags = nullptr, d.name_off = nullptr, d.name_bytes = nullptr;
}

void release_rows(TraceState& t) {
  t.perm.release();
  t.slot.release();
  t.kind.release();
  t.tok_slot.release();
  t.tfirst.release();
  DevRecords& d = t.rec;
  d.o_start.release(), d.o_dur.release(), d.o_size.release(), d.o_flags.release(), d.o_names.release();
  d.o_stream.release(), d.o_device.release(), d.o_off.release();
  d.start = d.dur = d.size = nullptr;
  d.flags = nullptr, d.stream = nullptr, d.device = nullptr, d.name_off = nullptr, d.name_bytes = nullptr;
}

// K1 in two halves around the dictionary (which does not depend on the order): the block sort and
// its check are launched first, their 32-byte verdict is copied to pinned memory, and the host
// reads it only after the dictionary's own readback — no round trip of its own.
void order_launch(TraceState& t) {
  Ctx* c = t.c;
  const uint64_t n = t.rec.n;
  t.sorted = true;
  t.order_pending = false;
  if (n <= 1 || t.rec.order == ITT_ORDER_SORTED) return;
  // fast path: sort 256-row blocks locally; if block ranges do not overlap the result is global
  const uint64_t nb = (n + kOrderBlock - 1) / kOrderBlock;
  t.order_stats.alloc(c, 4);  // min, max, descents, overlapping block boundaries
  unsigned long long init[4] = {static_cast<unsigned long long>(LLONG_MAX), static_cast<unsigned long long>(LLONG_MIN), 0, 0};
  h2d(c, t.order_stats.p, init, 4);
  t.perm.alloc(c, n);
  DBuf<int64_t> bmin(c, nb), bmax(c, nb);
  DBuf<uint8_t> bdesc(c, nb);
  DBuf<unsigned int> any(c, 1);
  any.zero();
  launch(c, "order_descent", n * 8.0, k_order_descent, dim3(grid_for((n + 7) / 8, 256, c->sm_count * 8)), dim3(256), 0,
         t.rec.start, n, any.p);
  launch(c, "order_blocks", n * 12.0, k_order_block_sort,
         dim3(static_cast<unsigned>(std::min<uint64_t>(nb, static_cast<uint64_t>(c->sm_count) * 32))), dim3(kOrderBlock), 0,
         t.rec.start, n, t.perm.p, bmin.p, bmax.p, bdesc.p, any.p);
  launch(c, "order_check", nb * 17.0, k_order_check, dim3(grid_for(nb, 256)), dim3(256), 0, bmin.p, bmax.p, bdesc.p, nb,
         t.order_stats.p, any.p);
  ITT_CUDA(cudaMemcpyAsync(c->deferred_block(), t.order_stats.p, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                           c->stream));
  ITT_CUDA(cudaEventRecord(c->deferred_ev, c->stream));
  t.order_pending = true;
}

void order_finish(TraceState& t) {
  if (!t.order_pending) return;
  Ctx* c = t.c;
  t.order_pending = false;
  ITT_CUDA(cudaEventSynchronize(c->deferred_ev));  // normally long complete: the dictionary synchronized
  unsigned long long h[4];
  std::memcpy(h, c->deferred, sizeof h);
  t.order_stats.release();
  const uint64_t n = t.rec.n;
  if (h[2] == 0) {  // already in (start,row) order
    t.perm.release();
    return;
  }
  t.sorted = false;
  if (h[3] == 0) {  // locally shuffled rows (the usual profiler export): the block sort is the order
    t.perm_local = true;
    return;
  }
  t.perm.release();
  const int64_t mn = static_cast<int64_t>(h[0]), mx = static_cast<int64_t>(h[1]);
  const int bits = bits_for(static_cast<uint64_t>(mx - mn));
  DBuf<uint64_t> k0(c, n), k1(c, n);
  DBuf<uint32_t> v0(c, n), v1(c, n);
  launch(c, "order_keys", n * 20.0, k_order_keys, dim3(grid_for(n, 256)), dim3(256), 0, t.rec.start, n, mn, k0.p, v0.p);
  // LSD radix sort is stable, so equal starts keep source-row order (ingest.hpp:396-400)
  const bool alt = radix_sort_pairs<uint64_t>(c, k0.p, v0.p, k1.p, v1.p, n, 0, bits, t.rs);
  t.perm = alt ? std::move(v1) : std::move(v0);
}

void order_records(TraceState& t) {
  order_launch(t);
  order_finish(t);
}

void build_dictionary(TraceState& t) {
  Ctx* c = t.c;
  const uint64_t n = t.rec.n;
  // the byte total is only needed on the host to plan streamed chunks (and for the profiler's
  // byte count); resident names let the hash kernel read name_off[n] itself
  const bool streamed = t.rec.host_names != nullptr;
  uint64_t total = ~0ull;
  if (n && t.rec.name_total >= 0) total = static_cast<uint64_t>(t.rec.name_total);
  else if (n && (streamed || c->profiling)) total = read1(c, t.rec.name_off + n);
  const double name_bytes = total == ~0ull ? 0.0 : static_cast<double>(total);
  t.slot.alloc(c, n);
  t.kind.alloc(c, n);
  DBuf<uint32_t> counters(c, 4);  // used count, overflow, collision, streamed-name arena overflow
  DBuf<unsigned long long> dev_counts;
  DBuf<uint32_t> dev_max(c, 1);
  if (t.rec.device) dev_counts.alloc(c, 65536);
  uint32_t bits = 14;
  uint64_t seed = 0x243F6A8885A308D3ull;
  // test hook: the first attempt puts every name into one slot, so the byte compare must catch the
  // collisions and the re-run with a real seed must recover
  if (const char* e = std::getenv("ITT_TEST_FORCE_COLLISION"); e && *e == '1') seed = 0;
  const unsigned groups = static_cast<unsigned>(std::min<uint64_t>((n + 31) / 32, 1ull << 30));
  constexpr unsigned kWarpsPerBlock = kHashBlock / 32;
  const unsigned grid =
      std::max(1u, std::min<unsigned>((groups + kWarpsPerBlock - 1) / kWarpsPerBlock, c->sm_count * 12));
  // streamed names: row chunks of ~kStreamChunk bytes through two device windows (copy stream),
  // overlapping the copy of chunk k+1 with the hash pass over chunk k
  std::vector<uint64_t> bounds;  // name_off at chunk boundaries
  uint64_t rows_per_chunk = n, chunks = 1, window = 0;
  uint8_t* win[2] = {nullptr, nullptr};
  uint8_t* bnc[2] = {nullptr, nullptr};
  DBuf<uint8_t> arena;
  DBuf<uint64_t> arena_off;
  DBuf<unsigned long long> arena_top;
  DBuf<uint32_t> snap;
  uint64_t arena_cap = 0;
  cudaEvent_t copied[2] = {nullptr, nullptr}, done[2] = {nullptr, nullptr};
  struct Events {
    cudaEvent_t* e[2];
    ~Events() {
      for (auto* p : e)
        for (int i = 0; i < 2; ++i)
          if (p[i]) cudaEventDestroy(p[i]);
    }
  } ev_guard{{copied, done}};
  if (t.rec.cols_ready) ITT_CUDA(cudaStreamWaitEvent(c->stream, t.rec.cols_ready, 0));  // host columns landed
  if (streamed && n) {
    uint64_t chunk_bytes = t.rec.stream_chunk ? t.rec.stream_chunk : (1ull << 30);
    if (const char* e = std::getenv("ITT_STREAM_CHUNK")) chunk_bytes = std::max<uint64_t>(64, std::strtoull(e, nullptr, 10));
    chunks = std::max<uint64_t>(1, (total + chunk_bytes - 1) / chunk_bytes);
    rows_per_chunk = ((n + chunks - 1) / chunks + 31) & ~31ull;
    chunks = (n + rows_per_chunk - 1) / rows_per_chunk;
    DBuf<uint64_t> db(c, chunks + 1);
    launch(c, "intern_name_bounds", 0.0, k_name_bounds, dim3(grid_for(chunks + 1, 128)), dim3(128), 0, t.rec.name_off, n,
           rows_per_chunk, chunks, db.p);
    bounds.resize(chunks + 1);
    readback(c, bounds.data(), db.p, chunks + 1);
    for (uint64_t k = 0; k < chunks; ++k) window = std::max<uint64_t>(window, bounds[k + 1] + 16 - (bounds[k] & ~15ull));
    win[0] = c->window(0, window);
    win[1] = c->window(1, window);
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, t.rec.host_names) != cudaSuccess) cudaGetLastError();
    if (pa.type != cudaMemoryTypeHost) {  // pageable: bounce through pinned buffers (parallel host memcpy)
      bnc[0] = c->bounce_buf(0, window);
      bnc[1] = c->bounce_buf(1, window);
    }
    arena_cap = std::min<uint64_t>(total + 16, 64ull << 20);
    snap.alloc(c, 1);
    arena_top.alloc(c, 1);
    for (int i = 0; i < 2; ++i) {
      ITT_CUDA(cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming));
      ITT_CUDA(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
    }
  }
  // 16-byte aligned copies of the slot representatives' names (the fast verify path); a slot
  // whose copy does not fit is verified against its representative row instead
  DBuf<uint64_t> tready;
  DBuf<uint8_t> copies;
  DBuf<unsigned long long> copies_top(c, 1);
  for (int attempt = 0;; ++attempt) {
    const uint32_t cap = 1u << bits;
    t.tkey.alloc(c, cap);
    t.trep.alloc(c, cap);
    t.tflags.alloc(c, cap);
    t.used.alloc(c, cap);
    tready.alloc(c, cap);
    const uint64_t copies_cap = std::min<uint64_t>(64ull << 20, std::max<uint64_t>(1ull << 20, static_cast<uint64_t>(cap) * 256));
    if (copies.n < copies_cap) copies.alloc(c, copies_cap);
    Fills fz(c);  // one launch for the table's and counters' initial values
    fz.add(t.tkey.p, cap * 8, 0);
    fz.add(tready.p, cap * 8, 0);
    fz.add(copies_top.p, 8, 0);
    fz.add(t.trep.p, cap * 4, 0xFF);
    fz.add(counters.p, 16, 0);
    fz.add(dev_max.p, 4, 0);
    if (t.rec.device) fz.add(dev_counts.p, 65536 * 8, 0);
    fz.flush();
    if (!streamed) {
      HashArgs ha{t.rec.name_off, t.rec.name_bytes, 0,         total,        0,          n,         nullptr,
                  nullptr,        t.rec.device,     t.tkey.p,  tready.p,     copies.p,   copies.n,  copies_top.p,
                  cap - 1,        seed,             t.slot.p,  t.used.p,     counters.p, dev_counts.p, dev_max.p};
      // algorithmic bytes (names once): name bytes + offset (8) + slot (4) + device id (2)
      launch(c, "intern_hash", static_cast<double>(name_bytes) + n * (t.rec.device ? 14.0 : 12.0), k_hash_insert, dim3(grid),
             dim3(kHashBlock), 0, ha);
    } else if (n) {
      if (arena.n < arena_cap) arena.alloc(c, arena_cap);
      arena_off.alloc(c, cap);
      arena_top.zero();
      cudaStream_t cp = c->copier();
      ITT_CUDA(cudaEventRecord(done[0], c->stream));  // windows free; the copy stream starts after prior work
      ITT_CUDA(cudaEventRecord(done[1], c->stream));
      for (uint64_t k = 0; k < chunks; ++k) {
        const int b = static_cast<int>(k & 1);
        const uint64_t r0 = k * rows_per_chunk, r1 = std::min(n, r0 + rows_per_chunk);
        // window [lo, hi): 16-byte aligned start, 16 bytes of slack past the chunk (zeros past the
        // last name, so the host buffer needs no slack)
        const uint64_t lo = bounds[k] & ~15ull, hi = bounds[k + 1] + 16, hc = std::min<uint64_t>(hi, total);
        ITT_CUDA(cudaStreamWaitEvent(cp, done[b], 0));
        const uint8_t* src = t.rec.host_names + lo;
        if (bnc[b]) {  // the DMA that last read this bounce buffer (chunk k-2) must be finished
          if (k >= 2) ITT_CUDA(cudaEventSynchronize(copied[b]));
          parallel_memcpy(bnc[b], src, hc - lo);
          src = bnc[b];
        }
        ITT_CUDA(cudaMemcpyAsync(win[b], src, hc - lo, cudaMemcpyHostToDevice, cp));
        if (hi > hc) ITT_CUDA(cudaMemsetAsync(win[b] + (hc - lo), 0, hi - hc, cp));
        ITT_CUDA(cudaEventRecord(copied[b], cp));
        if (k + 1 == chunks) issue_late_durations(t);  // behind the last names on the copy stream
        ITT_CUDA(cudaStreamWaitEvent(c->stream, copied[b], 0));
        ITT_CUDA(cudaMemcpyAsync(snap.p, counters.p, 4, cudaMemcpyDeviceToDevice, c->stream));
        const uint8_t* bytes = win[b] - lo;  // bytes[o] valid for o in [lo, hi)
        const uint64_t cgroups = (r1 - r0 + 31) / 32;
        const unsigned cgrid = static_cast<unsigned>(
            std::max<uint64_t>(1, std::min<uint64_t>((cgroups + kWarpsPerBlock - 1) / kWarpsPerBlock, c->sm_count * 12)));
        HashArgs ha{t.rec.name_off, bytes,        lo,       hi,       r0,         r1,       arena.p,
                    arena_off.p,    t.rec.device, t.tkey.p, tready.p, copies.p,   copies.n, copies_top.p,
                    cap - 1,        seed,         t.slot.p, t.used.p, counters.p, dev_counts.p, dev_max.p};
        launch(c, "intern_hash", static_cast<double>(bounds[k + 1] - bounds[k]) + (r1 - r0) * (t.rec.device ? 14.0 : 12.0), k_hash_insert,
               dim3(cgrid), dim3(kHashBlock), 0, ha);
        launch(c, "intern_save_reps", 0.0, k_save_reps, dim3(c->sm_count), dim3(128), 0, t.used.p, snap.p, counters.p,
               t.tkey.p, t.rec.name_off, bytes, arena.p, arena_cap, arena_off.p, arena_top.p, counters.p + 3);
        ITT_CUDA(cudaEventRecord(done[b], c->stream));
      }
    }
    uint32_t cnt[4];
    readback(c, cnt, counters.p, 4);
    if (cnt[1] || cnt[0] > cap / 2) {  // table too full: grow and redo
      if (bits >= 30) fail(ITT_E_INVALID_ARGUMENT, "stream-classify: name dictionary overflow");
      bits += 2;
      continue;
    }
    if (cnt[3]) {  // streamed names: the representatives' bytes outgrew the arena
      if (arena_cap >= total + 16) fail(ITT_E_CUDA, "internal: streamed-name arena overflow");
      arena_cap = std::min<uint64_t>(total + 16, arena_cap * 8);
      counters.zero();
      continue;
    }
    if (cnt[2]) {  // a true 64-bit collision between different names: new seed
      if (attempt >= 3) fail(ITT_E_INVALID_ARGUMENT, "stream-classify: unresolvable name hash collision");
      seed = seed * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
      if (seed == 0) seed = 1;
      continue;
    }
    t.n_used = cnt[0];
    t.table_bits = bits;
    break;
  }
  issue_late_durations(t);  // (a no-op when the last name chunk already queued it)
  if (t.n_used)
    launch(c, "intern_classify", t.n_used * 128.0, k_classify_slots, dim3(grid_for(static_cast<uint64_t>(t.n_used) * 32, 128)),
           dim3(128), 0, t.used.p,
           t.n_used, t.tkey.p, t.rec.name_off, t.rec.name_bytes, streamed ? arena.p : nullptr,
           streamed ? arena_off.p : nullptr, t.tflags.p);
  const uint32_t tcap = 1u << t.table_bits;
  if (n && tcap <= kKindsSmemCap && n >= (1ull << 20)) {
    const size_t smem = static_cast<size_t>(tcap) * 5;
    smem_optin(c, k_kinds_minrow_smem, smem);
    const unsigned g2 = std::min<unsigned>(grid_for((n + 3) / 4, 1024), c->sm_count * 2);
    launch(c, "intern_kinds", n * 6.0, k_kinds_minrow_smem, dim3(g2), dim3(1024), smem, t.slot.p, t.rec.flags, n, t.tflags.p,
           tcap, t.kind.p, t.trep.p);
  } else if (n) {
    const unsigned g2 = std::min<unsigned>(grid_for(n, 256), c->sm_count * 16);
    launch(c, "intern_kinds", n * 6.0, k_kinds_minrow, dim3(g2), dim3(256), 0, t.slot.p, t.rec.flags, n, t.tflags.p,
           t.kind.p, t.trep.p);
  }
  // device census -> majority (ties to the smallest label rank, streams.hpp:187-194)
  t.n_devices = 1;
  t.majority = 0;
  t.filtering = false;
  t.kept = n;
  if (t.rec.device && n) {
    // device max and the first 64 label counts in one round trip (traces carry a handful of devices)
    constexpr uint32_t kFewDev = 64;
    uint32_t mx = 0;
    t.dev_counts.assign(kFewDev, 0);
    readback2(c, &mx, dev_max.p, 1, reinterpret_cast<unsigned long long*>(t.dev_counts.data()), dev_counts.p, kFewDev);
    t.dev_counts.resize(mx + 1, 0);
    if (mx >= kFewDev) readback(c, reinterpret_cast<unsigned long long*>(t.dev_counts.data()), dev_counts.p, mx + 1);
    uint64_t best = 0;
    t.n_devices = 0;
    for (uint32_t d = 0; d <= mx; ++d) {
      if (t.dev_counts[d]) ++t.n_devices;
      if (t.dev_counts[d] > best) best = t.dev_counts[d], t.majority = static_cast<uint16_t>(d);
    }
    if (t.n_devices > 1) {
      t.filtering = true;
      t.kept = best;
    }
  }
}

// one census pass over the kept records: the packed used entries (dur null: ends = starts)
static std::vector<StreamEntry> census_pass(TraceState& t, const int64_t* dur) {
  Ctx* c = t.c;
  const uint64_t n = t.rec.n;
  DBuf<StreamEntry> table(c, kStreamTableCap);
  DBuf<uint32_t> list(c, kStreamTableCap + 1);
  launch(c, "census_init", 0.0, k_init_stream_table, dim3(kStreamTableCap / 256), dim3(256), 0, table.p, list.p,
         kStreamTableCap + 1);
  CensusArgs ca{n, t.rec.stream, t.rec.device, t.filtering ? 1 : 0, t.majority, t.kind.p, t.rec.start, dur,
                table.p, list.p + 1, list.p};
  if (n) {
    const unsigned grid = std::min<unsigned>(grid_for((n + 3) / 4, 256), c->sm_count * 8);
    launch(c, "census", n * 23.0, k_stream_census, dim3(grid), dim3(256), 0, ca);
  }
  // one round trip for the usual handful of streams: count + the first kFew packed entries
  constexpr uint32_t kFew = 63;
  DBuf<StreamEntry> packed(c, kStreamTableCap + 1);
  launch(c, "census_pack", 0.0, k_pack_streams, dim3(1), dim3(256), 0, table.p, list.p, packed.p);
  std::vector<StreamEntry> all(kFew + 1);
  readback(c, all.data(), packed.p, kFew + 1);
  const uint32_t ns = static_cast<uint32_t>(all[0].key);
  if (ns > kFew) {
    all.resize(ns + 1);
    readback(c, all.data(), packed.p, ns + 1);
  }
  all.resize(ns + 1);
  return all;
}

void stream_census(TraceState& t) {
  // late durations: the census counts and first starts now, the stream ends after the copy lands
  const bool late = t.rec.dur_host != nullptr;
  if (late) t.rec.census_ends_late = true;
  const std::vector<StreamEntry> all = census_pass(t, late ? nullptr : t.rec.dur);
  const uint32_t ns = static_cast<uint32_t>(all.size() - 1);
  t.streams.clear();
  for (uint32_t u = 0; u < ns; ++u) {
    const StreamEntry& e = all[1 + u];
    itt_stream_summary o{};
    o.stream = static_cast<uint32_t>(e.key - 1);
    for (int k = 0; k < 6; ++k) o.counts[k] = static_cast<int64_t>(e.counts[k]);
    o.first_start = unord64(e.min_start);
    o.last_end = unord64(e.max_end);
    // classify_streams (streams.hpp:85-103)
    const int64_t total = o.counts[0] + o.counts[1] + o.counts[2] + o.counts[3] + o.counts[4] + o.counts[5];
    const int64_t mem = o.counts[ITT_KIND_HTOD] + o.counts[ITT_KIND_DTOH] + o.counts[ITT_KIND_DTOD];
    o.cls = ITT_CLASS_ASSIST;
    if (o.counts[ITT_KIND_KERNEL] > 0) {
      o.cls = ITT_CLASS_MAIN;
    } else if (total > 0 && mem == total) {
      const bool h = o.counts[ITT_KIND_HTOD] > 0, d = o.counts[ITT_KIND_DTOH] > 0, dd = o.counts[ITT_KIND_DTOD] > 0;
      o.cls = (h && !d && !dd) ? ITT_CLASS_COPY_HTOD : (d && !h && !dd) ? ITT_CLASS_COPY_DTOH : ITT_CLASS_COPY_MIXED;
    }
    t.streams.push_back(o);
  }
  std::sort(t.streams.begin(), t.streams.end(),
            [](const itt_stream_summary& a, const itt_stream_summary& b) { return a.stream < b.stream; });
}

void compact_main(TraceState& t, uint32_t main_stream, bool want_record_index) {
  Ctx* c = t.c;
  const uint64_t n = t.rec.n;
  t.tfirst.alloc(c, t.tkey.n);
  Fills fz(c);  // first-appearance sentinels and the HtoD end range's initial (min, max) in one launch
  fz.add(t.tfirst.p, t.tfirst.n * 4, 0xFF);
  // capacities: count first (cheap readback of the census would do, but the scan itself is exact)
  uint64_t n_main = 0, n_htod = 0;
  for (const auto& s : t.streams) {
    if (s.stream == main_stream) n_main = s.counts[0] + s.counts[1] + s.counts[2] + s.counts[3] + s.counts[4] + s.counts[5];
    n_htod += s.counts[ITT_KIND_HTOD];
  }
  t.tok_slot.alloc(c, n_main + 1);
  t.tok_start.alloc(c, n_main + 1);
  t.tok_end.alloc(c, n_main + 1);
  t.tok_kind.alloc(c, n_main + 1);
  t.tokens.alloc(c, n_main + 1);
  if (want_record_index) t.tok_record.alloc(c, n_main + 1);
  t.htod_start.alloc(c, n_htod + 1);
  t.htod_end.alloc(c, n_htod + 1);
  t.htod_size.alloc(c, n_htod + 1);
  t.htod_range.alloc(c, 2);
  fz.add(t.htod_range.p, 8, 0xFF);
  fz.add(t.htod_range.p + 1, 8, 0);
  fz.flush();
  DBuf<uint64_t> tot(c, 1);
  CompactF f{n,
             t.sorted ? nullptr : t.perm.p,
             t.rec.stream,
             t.rec.device,
             t.filtering ? 1 : 0,
             t.majority,
             main_stream,
             t.kind.p,
             t.slot.p,
             t.rec.start,
             t.rec.dur,
             t.rec.size,
             t.rec.flags,
             t.tok_slot.p,
             t.tok_start.p,
             t.tok_end.p,
             t.tok_kind.p,
             want_record_index ? t.tok_record.p : nullptr,
             t.tfirst.p,
             t.htod_start.p,
             t.htod_end.p,
             t.htod_size.p,
             t.htod_range.p};
  static const bool two_pass = [] {  // ITT_COMPACT_RS=0: the single-pass look-back kernel for sorted rows too (A/B)
    const char* e = std::getenv("ITT_COMPACT_RS");
    return !(e && *e == '0');
  }();
  t.main_stream = main_stream;
  const bool rs_path = t.sorted && two_pass;
  if (t.rec.dur_host && !t.rec.compact_ends_late) {
    if (rs_path && n) {  // the ends pass (finish_late_durations) writes tok_end / htod_end later
      f.dur = nullptr;
      t.rec.compact_ends_late = true;
    } else {  // other compaction paths read durations now: wait for the late copy
      issue_late_durations(t);
      ITT_CUDA(cudaStreamWaitEvent(c->stream, t.rec.dur_ready, 0));
    }
  }
  if (rs_path) {  // rows in order: reduce-then-scan
    const uint64_t tiles = (n + kRSTile - 1) / kRSTile;
    if (n) {
      t.compact_tiles.alloc(c, tiles);
      uint64_t* tc = t.compact_tiles.p;
      launch(c, "compact_count", n * (t.filtering ? 7.0 : 5.0), k_compact_count, dim3(static_cast<unsigned>(tiles)), dim3(256), 0,
             f, tc);
      launch(c, "compact_scan", tiles * 16.0, k_scan_tile_counts, dim3(1), dim3(1024), 0, tc, tiles);
      launch(c, "compact", n * (t.filtering ? 7.0 : 5.0) + n_main * (f.dur ? 45.0 : 37.0) + n_htod * 48.0, k_compact_write,
             dim3(static_cast<unsigned>(tiles)), dim3(256), 0, f, tc);
      if (!t.rec.compact_ends_late) t.compact_tiles.release();
    }
  } else if (t.sorted || t.perm_local) {  // block-local order: stage each tile's rows in shared memory
    const uint64_t tiles = (n + kCompactTile - 1) / kCompactTile;
    t.scan.prepare(c, tiles);
    const size_t smem = sizeof(CompactLocalSmem);
    smem_optin(c, k_compact_local, smem);
    if (n)
      launch(c, "compact", n * (t.sorted ? 27.0 : 31.0) + n_main * 25.0 + n_htod * 24.0, k_compact_local,
             dim3(static_cast<unsigned>(tiles)), dim3(kCompactBlock), smem, f, t.scan.buf.p + 1,
             reinterpret_cast<uint32_t*>(t.scan.buf.p));
  } else {
    device_scan<uint64_t, SumOp<uint64_t>>(c, "compact", n * 18.0 + n_main * 28.0 + n_htod * 24.0, f, n, t.scan);
  }
  if (t.streams.empty()) fail(ITT_E_INVALID_ARGUMENT, "internal: compact_main needs the stream census");
  t.n_tok = n_main;
  t.n_htod = n_htod;
}

void renumber_tokens(TraceState& t) {
  Ctx* c = t.c;
  DBuf<uint32_t> id_of_slot(c, t.tkey.n);
  DBuf<uint32_t> cnt(c, 1);
  cnt.zero();
  const uint32_t nu = t.n_used;
  if (nu <= 16384) {
    launch(c, "intern_rank", nu * 4.0, k_rank_slots, dim3(grid_for(nu, 256)), dim3(256), 0, t.used.p, nu, t.tfirst.p,
           id_of_slot.p, cnt.p);
    t.n_names = read1(c, cnt.p);
  } else {
    DBuf<uint32_t> k0(c, nu), k1(c, nu), v0(c, nu), v1(c, nu);
    launch(c, "intern_pairs", nu * 16.0, k_first_pairs, dim3(grid_for(nu, 256)), dim3(256), 0, t.used.p, nu, t.tfirst.p,
           k0.p, v0.p);
    const bool alt = radix_sort_pairs<uint32_t>(c, k0.p, v0.p, k1.p, v1.p, nu, 0, 32, t.rs);
    std::vector<uint32_t> keys(nu);
    readback(c, keys.data(), alt ? k1.p : k0.p, nu);
    uint32_t m = 0;
    while (m < nu && keys[m] != kNone) ++m;
    id_of_slot.fill_bytes(0xFF);
    launch(c, "intern_ids", m * 8.0, k_slot_ids_from_sorted, dim3(grid_for(m, 256)), dim3(256), 0, alt ? v1.p : v0.p, m,
           id_of_slot.p);
    t.n_names = m;
  }
  if (t.n_tok)
    launch(c, "intern_map", t.n_tok * 8.0, k_map_tokens, dim3(grid_for((t.n_tok + 3) / 4, 256, c->sm_count * 16)), dim3(256), 0,
           t.tok_slot.p, t.n_tok,
           id_of_slot.p, t.tokens.p);
  DBuf<uint64_t> rows(c, t.n_names + 1);
  launch(c, "intern_names", nu * 8.0, k_name_rows, dim3(grid_for(nu, 256)), dim3(256), 0, t.used.p, nu, id_of_slot.p,
         t.trep.p, rows.p);
  t.name_row.resize(t.n_names);
  readback(c, t.name_row.data(), rows.p, t.n_names);
}

int64_t count_overlaps(TraceState& t) {
  Ctx* c = t.c;
  if (t.n_tok < 2) return 0;
  DBuf<unsigned long long> out(c, 1);
  out.zero();
  const unsigned grid = std::min<unsigned>(grid_for(t.n_tok, 256), c->sm_count * 8);
  launch(c, "overlaps", t.n_tok * 16.0, k_overlaps, dim3(grid), dim3(256), 0, t.tok_start.p, t.tok_end.p, t.n_tok, out.p);
  return static_cast<int64_t>(read1(c, out.p));
}

}  // namespace itt
