// report.cu — the host finish at scale: compute_summary (metrics.hpp:166-202)
// and details_to_csv (report.hpp:191-220) over the integer per-iteration rows the device
// produced, natively and in parallel.  Host code only; exactness rules:
//   * overlap_ratio = (double)copy_ns / (double)interval_ns when the interval exists and is > 0,
//     op_gap_mean = (double)gap_sum / (double)gap_count (0.0 when gap_count == 0): the two
//     divisions of compute_iteration_metrics (metrics.hpp:131-135, 145-160), done here as there;
//   * summary sums are accumulated row by row in index order (the reference's loop), so the
//     doubles are bit-identical; integers use the reference's int64 accumulators;
//   * CSV cells: std::to_string for integers, "%.6f" (detail::format_double, report.hpp:49-53),
//     std::llround for the gap mean; rows are formatted in independent blocks by host threads
//     and concatenated in order.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "itertrace_cuda.h"

namespace {

constexpr const char* kDetailsHeader =
    "iteration,token_start,token_end,t_start_ns,t_end_ns,interval_ns,overlap_ratio,htod_bytes,op_gap_mean_ns,extra_ops\n";

inline bool has_interval(const itt_iter_row& r) { return r.has_interval != 0; }
inline bool has_overlap(const itt_iter_row& r) { return r.has_interval != 0 && r.interval_ns > 0; }
inline double overlap(const itt_iter_row& r) { return static_cast<double>(r.copy_ns) / static_cast<double>(r.interval_ns); }
inline double gap_mean(const itt_iter_row& r) {
  return r.gap_count > 0 ? static_cast<double>(r.gap_sum) / static_cast<double>(r.gap_count) : 0.0;
}

inline void put_i64(std::string& s, long long v) {
  char b[24];
  const int k = std::snprintf(b, sizeof b, "%lld", v);
  s.append(b, static_cast<size_t>(k));
}

void render_rows(const itt_iter_row* rows, uint64_t a, uint64_t b, std::string& s) {
  s.reserve((b - a) * 80);
  char buf[64];
  for (uint64_t k = a; k < b; ++k) {
    const itt_iter_row& r = rows[k];
    put_i64(s, static_cast<long long>(k + 1));
    s += ',';
    put_i64(s, r.start_token);
    s += ',';
    put_i64(s, r.end_token);
    s += ',';
    put_i64(s, r.t_start);
    s += ',';
    put_i64(s, r.t_end);
    s += ',';
    if (has_interval(r)) put_i64(s, r.interval_ns);
    s += ',';
    if (has_overlap(r)) {
      const int n = std::snprintf(buf, sizeof buf, "%.*f", 6, overlap(r));
      s.append(buf, static_cast<size_t>(n));
    }
    s += ',';
    put_i64(s, r.htod_bytes);
    s += ',';
    put_i64(s, std::llround(gap_mean(r)));
    s += ',';
    put_i64(s, r.extra);
    s += '\n';
  }
}

}  // namespace

extern "C" __attribute__((visibility("hidden"))) int itt_ctx_set_error_(itt_ctx* ctx, const char* msg);  // capi.cu (not exported)

int itt_compute_summary(itt_ctx* ctx, const itt_iter_row* rows, uint64_t n, int64_t iterations_declared, itt_summary* out) {
  if (!out || (n && !rows)) return ITT_E_INVALID_ARGUMENT;
  std::memset(out, 0, sizeof *out);
  if (n == 0) {
    itt_ctx_set_error_(ctx, "metrics: no iterations to summarize");
    return ITT_E_NO_ITERATIONS;
  }
  out->iterations_found = static_cast<int64_t>(n);
  out->iterations_declared = iterations_declared;
  int64_t isum = 0, icnt = 0, ocnt = 0, btot = 0, imax = 0;
  double osum = 0.0, gsum = 0.0;
  for (uint64_t k = 0; k < n; ++k) {
    const itt_iter_row& r = rows[k];
    if (has_interval(r)) {
      isum += r.interval_ns;
      ++icnt;
      if (r.interval_ns > imax) imax = r.interval_ns;
    }
    if (has_overlap(r)) {
      osum += overlap(r);
      ++ocnt;
    }
    gsum += gap_mean(r);
    btot += r.htod_bytes;
  }
  out->max_interval_ns = imax;
  if (icnt > 0) out->avg_interval_ns = static_cast<double>(isum) / static_cast<double>(icnt);
  else out->insufficient_intervals = 1;
  if (ocnt > 0) out->avg_overlap = osum / static_cast<double>(ocnt);
  out->avg_operation_ns = gsum / static_cast<double>(n);
  out->avg_size_bytes = static_cast<double>(btot) / static_cast<double>(n);
  itt_ctx_set_error_(ctx, "");
  return ITT_OK;
}

int itt_render_details_csv(itt_ctx* ctx, const itt_iter_row* rows, uint64_t n, char** out, uint64_t* len) {
  if (!out || !len || (n && !rows)) return ITT_E_INVALID_ARGUMENT;
  *out = nullptr;
  *len = 0;
  try {
    constexpr uint64_t kRowsPerBlock = 16384;
    const uint64_t blocks = (n + kRowsPerBlock - 1) / kRowsPerBlock;
    std::vector<std::string> parts(blocks);
    const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    const unsigned nt = static_cast<unsigned>(std::min<uint64_t>(hw, blocks));
    auto work = [&](unsigned t) {
      for (uint64_t b = t; b < blocks; b += nt) render_rows(rows, b * kRowsPerBlock, std::min(n, (b + 1) * kRowsPerBlock), parts[b]);
    };
    if (nt <= 1) {
      if (blocks) work(0);
    } else {
      std::vector<std::thread> th;
      for (unsigned t = 0; t < nt; ++t) th.emplace_back(work, t);
      for (auto& x : th) x.join();
    }
    uint64_t total = std::strlen(kDetailsHeader);
    for (const auto& p : parts) total += p.size();
    char* buf = static_cast<char*>(std::malloc(total + 1));
    if (!buf) return ITT_E_CUDA;
    uint64_t at = std::strlen(kDetailsHeader);
    std::memcpy(buf, kDetailsHeader, at);
    for (const auto& p : parts) {
      std::memcpy(buf + at, p.data(), p.size());
      at += p.size();
    }
    buf[total] = '\0';
    *out = buf;
    *len = total;
    itt_ctx_set_error_(ctx, "");
    return ITT_OK;
  } catch (const std::exception& e) {
    itt_ctx_set_error_(ctx, e.what());
    return ITT_E_CUDA;
  }
}
