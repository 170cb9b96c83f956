// metrics.cu — per-iteration segmented reductions, sm_100a.
//
// partition_iterations + compute_iteration_metrics (metrics.hpp:44-164), integer core only:
// the two double divisions (overlap ratio, op-gap mean) and the ordered summary sums are
// left to the host in reference order so the doubles are bit-identical.
//
// The reference scans all H HtoD records for every iteration (O(I*H), metrics.hpp:132-143).
// Here HtoD records stay in (start,row) order, so per iteration k with lo = t_end(k-1):
//   * union of clip(HtoD, (lo, t_start(k))): carry-in [lo, min(prefmax_end(start < lo), hi))
//     then a running-max merge of the records with lo <= start < hi (metrics.hpp:76-100);
//   * HtoD bytes over start in (lo, t_end(k)] (first lo = -1, metrics.hpp:138-143);
//   * op gaps: one warp per span sums max(0, start[j+1] - end[j]) over j in [s, e) and
//     counts the clamped ones (metrics.hpp:145-157).
#include <algorithm>

#include "pipeline.cuh"

namespace itt {

namespace {

constexpr unsigned long long kFlip = 1ull << 63;  // int64 order -> uint64 order
__device__ __forceinline__ int64_t unflip(unsigned long long v) { return static_cast<int64_t>(v ^ kFlip); }

// inclusive prefix max of HtoD ends relative to their minimum (the look-back words carry 62-bit
// values); the minimum comes from compact_main's atomics, so no range pass or host sync is needed
struct PrefMaxF {
  const int64_t* end;
  const unsigned long long* range;
  int64_t* out;
  __device__ __forceinline__ uint64_t load(uint64_t i) const {
    return static_cast<uint64_t>(end[i] - unflip(__ldg(&range[0]))) & ((1ull << 62) - 1);
  }
  __device__ __forceinline__ void store(uint64_t i, uint64_t excl, uint64_t v) const {
    out[i] = static_cast<int64_t>(excl > v ? excl : v) + unflip(__ldg(&range[0]));
  }
};

struct AggArgs {
  const int64_t* ts;  // main-stream token start / end
  const int64_t* te;
  const int64_t* hs;  // HtoD start / end / size, (start,row) order
  const int64_t* he;
  const int64_t* hz;
  const int64_t* hpmax;  // inclusive prefix max of he
  uint64_t H;
  const uint32_t* sp_start;
  const uint32_t* sp_end;
  const uint32_t* sp_extra;
  uint64_t I;
  itt_iter_row* rows;
  const unsigned long long* htod_range;
  unsigned long long* clamps;  // [0] negative gaps, [1] negative intervals, [2] HtoD range overflow
};

__device__ __forceinline__ uint64_t lower_bound64(const int64_t* a, uint64_t n, int64_t x) {  // first a[i] >= x
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ uint64_t upper_bound64(const int64_t* a, uint64_t n, int64_t x) {  // first a[i] > x
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void k_span_aggregates(AggArgs a) {
  const uint64_t k = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (k == 0 && threadIdx.x == 0 && a.H &&
      static_cast<unsigned long long>(unflip(a.htod_range[1]) - unflip(a.htod_range[0])) >= (1ull << 62))
    a.clamps[2] = 1;
  if (k >= a.I) return;
  const unsigned lane = lane_id();
  const uint64_t s = a.sp_start[k], e = a.sp_end[k];
  // ---- op gaps inside the span
  long long gsum = 0;
  unsigned neg = 0;
  for (uint64_t j = s + lane; j < e; j += 32) {
    long long g = a.ts[j + 1] - a.te[j];
    if (g < 0) {
      g = 0;
      ++neg;
    }
    gsum += g;
  }
  for (int o = 16; o > 0; o >>= 1) {
    gsum += __shfl_xor_sync(0xffffffffu, gsum, o);
    neg += __shfl_xor_sync(0xffffffffu, neg, o);
  }
  if (lane != 0) return;
  itt_iter_row r;
  r.start_token = static_cast<int64_t>(s);
  r.end_token = static_cast<int64_t>(e);
  r.extra = a.sp_extra[k];
  r.t_start = a.ts[s];
  r.t_end = a.te[e];
  r.gap_sum = gsum;
  r.gap_count = static_cast<int64_t>(e - s);
  r.interval_ns = 0;
  r.copy_ns = 0;
  r.has_interval = 0;
  r.pad_ = 0;
  if (neg) atomicAdd(&a.clamps[0], static_cast<unsigned long long>(neg));
  int64_t lo_b = -1;
  if (k > 0) {
    const int64_t prev_end = a.te[a.sp_end[k - 1]];
    lo_b = prev_end;
    int64_t interval = r.t_start - prev_end;
    if (interval < 0) {
      interval = 0;
      atomicAdd(&a.clamps[1], 1ull);
    }
    r.has_interval = 1;
    r.interval_ns = interval;
    if (interval > 0) {
      const int64_t lo = prev_end, hi = r.t_start;
      const uint64_t i0 = lower_bound64(a.hs, a.H, lo);
      int64_t total = 0, cl = 0, ch = 0;
      bool open = false;
      if (i0 > 0) {
        const int64_t b = min(a.hpmax[i0 - 1], hi);
        if (b > lo) {
          cl = lo;
          ch = b;
          open = true;
        }
      }
      for (uint64_t i = i0; i < a.H && a.hs[i] < hi; ++i) {
        const int64_t x = a.hs[i];
        const int64_t y = min(a.he[i], hi);
        if (y <= x) continue;
        if (!open || x > ch) {
          if (open) total += ch - cl;
          cl = x;
          ch = y;
          open = true;
        } else if (y > ch) {
          ch = y;
        }
      }
      if (open) total += ch - cl;
      r.copy_ns = total;
    }
  }
  // ---- HtoD bytes with start in (lo_b, t_end]
  int64_t bytes = 0;
  for (uint64_t i = upper_bound64(a.hs, a.H, lo_b); i < a.H && a.hs[i] <= r.t_end; ++i) bytes += a.hz[i];
  r.htod_bytes = bytes;
  a.rows[k] = r;
}

}  // namespace

void iteration_aggregates(Ctx* c, const int64_t* tok_start, const int64_t* tok_end, uint64_t n_tok,
                          const int64_t* htod_start, const int64_t* htod_end, const int64_t* htod_size, uint64_t n_htod,
                          const unsigned long long* htod_range, const SpanState& spans, itt_iter_row* rows,
                          itt_clamps& clamps,
                          ScanScratch& scan) {
  (void)n_tok;
  clamps = itt_clamps{0, 0};
  if (spans.n == 0) return;
  DBuf<int64_t> pmax(c, n_htod + 1);
  if (n_htod)
    device_scan<uint64_t, MaxOp<uint64_t>>(c, "agg_htod_prefmax", n_htod * 16.0, PrefMaxF{htod_end, htod_range, pmax.p}, n_htod, scan);
  DBuf<itt_iter_row> drows(c, spans.n);
  DBuf<unsigned long long> dcl(c, 3);
  dcl.zero();
  AggArgs a{tok_start,     tok_end,     htod_start,    htod_end, htod_size, pmax.p,     n_htod,
            spans.start.p, spans.end.p, spans.extra.p, spans.n,  drows.p,   htod_range, dcl.p};
  const uint64_t threads = spans.n * 32;
  launch(c, "agg_spans", static_cast<double>(n_tok) * 16.0 + spans.n * 96.0, k_span_aggregates, dim3(grid_for(threads, 256)),
         dim3(256), 0, a);
  d2h(c, rows, drows.p, spans.n);  // straight into the caller's (pinned) buffer
  unsigned long long cl[3];
  readback(c, cl, dcl.p, 3);  // synchronizes
  if (cl[2]) fail(ITT_E_INVALID_ARGUMENT, "metrics: HtoD time range exceeds 2^62 ns");
  clamps.negative_gap_clamps = static_cast<int64_t>(cl[0]);
  clamps.negative_interval_clamps = static_cast<int64_t>(cl[1]);
}

}  // namespace itt
