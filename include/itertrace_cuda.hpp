// itertrace_cuda.hpp — C++ drop-in for the reference's hot-path functions, over the C-ABI of
// libitertrace_cuda.so (include/itertrace_cuda.h).
//
// Include AFTER the reference's own headers (it uses their types, unchanged):
//
//     #include "itertrace/itertrace.hpp"   // reference, /root/reference/proj/include
//     #include "itertrace_cuda.hpp"        // this file
//
// Every function in itertrace::cuda has the signature and the error behaviour (itertrace::Error
// with the same ErrorKind and stage-prefixed message) of the reference function it replaces;
// only the device-side stages move — compute_summary, diagnose, render_report and the CLI stay
// the reference's code.  Replaced functions (paths under proj/include/itertrace/):
//   build_token_sequence      streams.hpp:147-169
//   count_interval_overlaps   streams.hpp:212-221
//   mine_pattern              mine.hpp:119-122
//   mine_patterns_multi       mine.hpp:132-165
//   approx_match              match.hpp:41-85, :87-91
//   partition_iterations      metrics.hpp:44-55
//   compute_iteration_metrics metrics.hpp:109-164 (both the reference's 4-parameter form and a
//                             3-parameter form whose HtoD list is collect_htod_records(trace))
//   analyze_trace             pipeline.hpp:34-134
//   parse_trace + analyze_trace, parse_trace + summarize_streams (the CLI's analyze / inspect
//                             bodies, itertrace_main.cpp:121-149) with the CSV parsed on the GPU:
//                             analyze_csv_file, inspect_csv_file
// Device failures (no sm_100 GPU, CUDA errors) throw CudaError, a std::runtime_error — the
// reference CLI maps those to exit code 1 (itertrace_main.cpp:294-296).  No CPU fallback.
#pragma once

#include <algorithm>
#include <cstdlib>
#include <fstream>
#include <iterator>
#include <map>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "itertrace_cuda.h"

namespace itertrace::cuda {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

class Context {
 public:
  explicit Context(int device = 0) {
    if (itt_ctx_create(device, &c_) != 0) throw CudaError("itertrace-cuda: no usable sm_100 device");
  }
  ~Context() { itt_ctx_destroy(c_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  itt_ctx* get() const { return c_; }
  // one context per host thread (the C-ABI contract)
  static Context& thread_default() {
    thread_local std::unique_ptr<Context> ctx;
    if (!ctx) {
      const char* d = std::getenv("ITT_DEVICE");
      ctx = std::make_unique<Context>(d ? std::atoi(d) : 0);
    }
    return *ctx;
  }
  void check(int rc) const {
    if (rc == 0) return;
    const std::string msg = itt_last_error(c_);
    if (rc >= 1 && rc <= 12) throw Error(static_cast<ErrorKind>(rc - 1), msg);
    throw CudaError(msg);
  }

 private:
  itt_ctx* c_ = nullptr;
};

namespace detail {

// TraceRecord AoS -> itt_records SoA.  Device labels are interned in byte-lexicographic order
// so "ties to the lexicographically smallest label" (streams.hpp:187-194) is "smallest id".
struct Columns {
  std::vector<int64_t> start, dur, size;
  std::vector<uint8_t> flags;
  std::vector<uint32_t> stream;
  std::vector<uint16_t> device;
  std::vector<uint64_t> off;
  std::string names;
  std::vector<std::string> labels;

  explicit Columns(const NormalizedTrace& t) {
    const size_t n = t.records.size();
    start.resize(n), dur.resize(n), size.resize(n), flags.resize(n), stream.resize(n), device.resize(n);
    off.resize(n + 1);
    for (const auto& r : t.records) labels.push_back(r.device);
    std::sort(labels.begin(), labels.end());
    labels.erase(std::unique(labels.begin(), labels.end()), labels.end());
    std::map<std::string, uint16_t> id;
    for (size_t i = 0; i < labels.size(); ++i) id[labels[i]] = static_cast<uint16_t>(i);
    for (size_t i = 0; i < n; ++i) {
      const TraceRecord& r = t.records[i];
      start[i] = r.start_ns;
      dur[i] = r.duration_ns;
      size[i] = r.size_bytes.value_or(0);
      flags[i] = static_cast<uint8_t>((r.size_bytes ? ITT_REC_HAS_SIZE : 0u) | (r.throughput_bps ? ITT_REC_HAS_THROUGHPUT : 0u));
      stream[i] = r.stream;
      device[i] = id[r.device];
      off[i] = names.size();
      names += r.name;
    }
    off[n] = names.size();
  }
  itt_records view() const {
    itt_records v{};
    v.n = start.size();
    v.start_ns = start.data();
    v.duration_ns = dur.data();
    v.size_bytes = size.data();
    v.flags = flags.data();
    v.stream = stream.data();
    v.device = device.data();
    v.name_off = off.data();
    v.name_bytes = reinterpret_cast<const uint8_t*>(names.data());
    v.mem = ITT_MEM_HOST;
    v.order = ITT_ORDER_SORTED;  // a NormalizedTrace is already in (start,row) order
    return v;
  }
};

inline IterationMetrics to_metrics(const itt_iter_row& r, int64_t index) {
  IterationMetrics m;  // the reference's own divisions (metrics.hpp:131-135, 158-160)
  m.index = index;
  m.span = MatchSpan{r.start_token, r.end_token, r.extra};
  m.t_start = r.t_start;
  m.t_end = r.t_end;
  m.extra_ops = r.extra;
  if (r.has_interval) {
    m.interval_ns = r.interval_ns;
    if (r.interval_ns > 0) m.overlap_ratio = static_cast<double>(r.copy_ns) / static_cast<double>(r.interval_ns);
  }
  m.htod_bytes = r.htod_bytes;
  m.op_gap_mean_ns = r.gap_count > 0 ? static_cast<double>(r.gap_sum) / static_cast<double>(r.gap_count) : 0.0;
  return m;
}

}  // namespace detail

inline TokenSequence build_token_sequence(const NormalizedTrace& trace, std::uint32_t main_stream) {
  Context& ctx = Context::thread_default();
  const detail::Columns cols(trace);
  const itt_records rv = cols.view();
  itt_tokens* t = nullptr;
  ctx.check(itt_build_token_sequence(ctx.get(), &rv, main_stream, &t));
  TokenSequence seq;
  seq.tokens.assign(t->tokens, t->tokens + t->n);
  seq.record_index.assign(t->record_index, t->record_index + t->n);
  for (uint32_t v = 0; v < t->n_names; ++v) {
    seq.names.push_back(trace.records[t->name_row[v]].name);
    seq.ids.emplace(seq.names.back(), static_cast<int32_t>(v));
  }
  itt_free(ctx.get(), t->tokens);
  itt_free(ctx.get(), t->record_index);
  itt_free(ctx.get(), t->name_row);
  itt_free(ctx.get(), t);
  return seq;
}

inline std::int64_t count_interval_overlaps(const NormalizedTrace& trace, std::uint32_t stream) {
  Context& ctx = Context::thread_default();
  const detail::Columns cols(trace);
  const itt_records rv = cols.view();
  int64_t out = 0;
  ctx.check(itt_count_interval_overlaps(ctx.get(), &rv, stream, &out));
  return out;
}

inline std::vector<PatternCandidate> mine_patterns_impl(const TokenSequence& seq, const std::vector<MiningConfig>& loops,
                                                        bool multi) {
  Context& ctx = Context::thread_default();
  std::vector<itt_mining_cfg> cfg;
  for (const auto& l : loops) cfg.push_back(itt_mining_cfg{l.iterations, l.epsilon0, l.epsilon_cap.value_or(0)});
  itt_pattern* p = nullptr;
  ctx.check(itt_mine_patterns(ctx.get(), seq.tokens.data(), seq.tokens.size(), seq.terminator(), cfg.data(),
                              static_cast<uint32_t>(cfg.size()), multi ? 1 : 0, &p));
  std::vector<PatternCandidate> out;
  const size_t k = multi ? cfg.size() : 1;
  for (size_t i = 0; i < k; ++i) {
    PatternCandidate c;
    c.tokens.assign(p[i].tokens, p[i].tokens + p[i].length);
    c.count = p[i].count;
    c.first_token = p[i].first_token;
    c.epsilon_used = p[i].epsilon_used;
    out.push_back(std::move(c));
  }
  itt_free_patterns(ctx.get(), p, static_cast<uint32_t>(k));
  return out;
}

inline PatternCandidate mine_pattern(const TokenSequence& seq, const MiningConfig& cfg) {
  return mine_patterns_impl(seq, {cfg}, false).front();
}

inline std::vector<PatternCandidate> mine_patterns_multi(const TokenSequence& seq, const std::vector<MiningConfig>& loops) {
  return mine_patterns_impl(seq, loops, true);
}

inline std::vector<MatchSpan> approx_match(std::span<const std::int32_t> tokens, std::span<const std::int32_t> pattern,
                                           const MatchConfig& cfg) {
  Context& ctx = Context::thread_default();
  itt_span* s = nullptr;
  uint64_t n = 0;
  ctx.check(itt_approx_match(ctx.get(), tokens.data(), tokens.size(), pattern.data(), pattern.size(), cfg.k0, &s, &n));
  std::vector<MatchSpan> out(n);
  for (uint64_t i = 0; i < n; ++i) out[i] = MatchSpan{s[i].start_token, s[i].end_token, s[i].extra};
  itt_free(ctx.get(), s);
  return out;
}

inline std::vector<MatchSpan> approx_match(const TokenSequence& seq, std::span<const std::int32_t> pattern,
                                           const MatchConfig& cfg) {
  return itertrace::cuda::approx_match(std::span<const std::int32_t>(seq.tokens), pattern, cfg);
}

// windows: partition_iterations(trace, seq, spans); the HtoD list is every MemcpyHtoD record of
// `trace`, i.e. what the pipeline passes (collect_htod_records, pipeline.hpp:93).
inline IterationAnalysis compute_iteration_metrics(const NormalizedTrace& trace, const TokenSequence& seq,
                                                   const std::vector<IterationWindow>& windows) {
  Context& ctx = Context::thread_default();
  const detail::Columns cols(trace);
  const itt_records rv = cols.view();
  std::vector<itt_span> spans;
  for (const auto& w : windows) spans.push_back(itt_span{w.span.start_token, w.span.end_token, w.span.extra});
  std::vector<uint64_t> ri(seq.record_index.begin(), seq.record_index.end());
  itt_iter_row* rows = nullptr;
  itt_clamps cl{};
  ctx.check(itt_iteration_metrics(ctx.get(), &rv, ri.data(), ri.size(), spans.data(), spans.size(), &rows, &cl));
  IterationAnalysis out;
  for (size_t k = 0; k < spans.size(); ++k) out.iterations.push_back(detail::to_metrics(rows[k], static_cast<int64_t>(k + 1)));
  out.negative_gap_clamps = cl.negative_gap_clamps;
  out.negative_interval_clamps = cl.negative_interval_clamps;
  itt_free(ctx.get(), rows);
  return out;
}

// partition_iterations (metrics.hpp:44-55): the windows' times come from the device aggregate pass
// (t_start / t_end of every span), so a caller swapping namespaces gets the same vector.
inline std::vector<IterationWindow> partition_iterations(const NormalizedTrace& trace, const TokenSequence& seq,
                                                         const std::vector<MatchSpan>& spans) {
  std::vector<IterationWindow> windows;
  windows.reserve(spans.size());
  for (const auto& sp : spans) windows.push_back(IterationWindow{sp, 0, 0});
  const IterationAnalysis a = itertrace::cuda::compute_iteration_metrics(trace, seq, windows);
  for (size_t k = 0; k < windows.size(); ++k) {
    windows[k].t_start = a.iterations[k].t_start;
    windows[k].t_end = a.iterations[k].t_end;
  }
  return windows;
}

// The reference's 4-parameter form (metrics.hpp:109-112): the HtoD list is the caller's.  When
// it is collect_htod_records(trace) (what the pipeline passes, pipeline.hpp:93) the trace goes to
// the device as is; otherwise the device sees the trace with the records' kinds adjusted so that
// exactly the listed records are MemcpyHtoD (names of unlisted HtoD records neutralised, listed
// records given an HtoD name) — the token columns are untouched, so the windows are too.
inline IterationAnalysis compute_iteration_metrics(const NormalizedTrace& trace, const TokenSequence& seq,
                                                   const std::vector<IterationWindow>& windows,
                                                   const std::vector<const TraceRecord*>& htod_records) {
  const size_t n = trace.records.size();
  std::vector<uint8_t> listed(n, 0);
  bool same = true;
  size_t j = 0;
  for (const TraceRecord* r : htod_records) {
    if (r < trace.records.data() || r >= trace.records.data() + n)
      throw Error(ErrorKind::InvalidConfig, "metrics: HtoD record outside the trace");
    const size_t i = static_cast<size_t>(r - trace.records.data());
    if (listed[i]) throw Error(ErrorKind::InvalidConfig, "metrics: HtoD record listed twice");
    listed[i] = 1;
    while (j < n && kind_of(trace.records[j]) != OpKind::MemcpyHtoD) ++j;
    same = same && j < n && j == i;
    ++j;
  }
  while (same && j < n && kind_of(trace.records[j]) != OpKind::MemcpyHtoD) ++j;
  if (same && j >= n) return itertrace::cuda::compute_iteration_metrics(trace, seq, windows);
  NormalizedTrace adj = trace;
  for (size_t i = 0; i < n; ++i) {
    const bool htod = kind_of(adj.records[i]) == OpKind::MemcpyHtoD;
    if (listed[i] && !htod) adj.records[i].name = "[CUDA memcpy HtoD]";
    if (!listed[i] && htod) adj.records[i].name = "unlisted-copy";
  }
  return itertrace::cuda::compute_iteration_metrics(adj, seq, windows);
}

// a12, the north star's per-op x per-iteration profile (no reference counterpart; definition
// in itertrace_cuda.h, itt_op_cell): over the reference's own token sequence and windows.
struct OpProfile {
  std::vector<itt_op_total> per_op;             // [seq.names.size()], by token id
  std::vector<itt_iter_op_total> per_iteration;  // [windows.size()]
  std::vector<itt_op_cell> cells;               // (iteration, op) order; empty unless requested
};
inline OpProfile op_profile(const NormalizedTrace& trace, const TokenSequence& seq,
                            const std::vector<IterationWindow>& windows, bool with_cells = false) {
  Context& ctx = Context::thread_default();
  const size_t n = seq.tokens.size();
  std::vector<int64_t> ts(n), te(n);
  std::vector<uint8_t> kind(n);
  for (size_t j = 0; j < n; ++j) {
    const TraceRecord& r = trace.records[seq.record_index[j]];
    ts[j] = r.start_ns;
    te[j] = r.end_ns();
    kind[j] = static_cast<uint8_t>(kind_of(r));  // OpKind order == ITT_KIND_* order
  }
  std::vector<itt_span> spans;
  for (const auto& w : windows) spans.push_back(itt_span{w.span.start_token, w.span.end_token, w.span.extra});
  OpProfile out;
  out.per_op.resize(seq.names.size());
  out.per_iteration.resize(spans.size());
  itt_op_cell* cells = nullptr;
  uint64_t n_cells = 0;
  ctx.check(itt_op_profile(ctx.get(), seq.tokens.data(), ts.data(), te.data(), kind.data(), n,
                           static_cast<uint32_t>(seq.names.size()), spans.data(), spans.size(), ITT_OP_PROFILE_AUTO,
                           out.per_op.data(), out.per_iteration.data(), with_cells ? &cells : nullptr, &n_cells));
  if (cells) {
    out.cells.assign(cells, cells + n_cells);
    itt_free(ctx.get(), cells);
  }
  return out;
}

namespace detail {

struct AnalysisHold {
  itt_ctx* c;
  void operator()(itt_analysis* x) const { itt_free_analysis(c, x); }  // rows return to the context's pool
};
using AnalysisPtr = std::unique_ptr<itt_analysis, AnalysisHold>;

inline AnalysisPtr run_analyze(Context& ctx, const itt_records& rv, const AnalyzeOptions& opt) {
  if (opt.loops.empty()) throw Error(ErrorKind::InvalidConfig, "analyze: at least one iteration count is required");
  itt_analyze_opts o{};
  o.loops = opt.loops.data();
  o.n_loops = static_cast<uint32_t>(opt.loops.size());
  o.epsilon0 = opt.epsilon0;
  o.k0 = opt.k0 ? *opt.k0 : -1;
  o.main_stream = opt.main_stream ? static_cast<int64_t>(*opt.main_stream) : -1;
  itt_analysis* a = nullptr;
  ctx.check(itt_analyze(ctx.get(), &rv, &o, &a));
  return AnalysisPtr(a, AnalysisHold{ctx.get()});
}

inline void fill_streams(const itt_census& c, std::vector<StreamSummary>& streams, std::map<std::uint32_t, StreamClass>& cls) {
  for (uint32_t i = 0; i < c.n_streams; ++i) {
    const itt_stream_summary& s = c.streams[i];
    StreamSummary ss;
    ss.stream = s.stream;
    for (int k = 0; k < 6; ++k) ss.counts[static_cast<size_t>(k)] = s.counts[k];
    ss.first_start = s.first_start;
    ss.last_end = s.last_end;
    streams.push_back(ss);
    cls[s.stream] = static_cast<StreamClass>(s.cls);
  }
}

// The host part of analyze_trace (pipeline.hpp:34-134) after the device pipeline: Report fields,
// the warnings in the reference's order, the reference's own compute_summary / diagnose.
// label_of(device rank) -> device label; name_of(row) -> name of the record at `row` of the
// record set itt_analyze ran on.
template <typename LabelOf, typename NameOf>
AnalysisResult assemble(const itt_analysis* a, const AnalyzeOptions& opt, const std::string& trace_label,
                        std::vector<std::string> warnings, LabelOf label_of, NameOf name_of) {
  AnalysisResult result;
  Report& report = result.report;
  report.trace_path = trace_label;
  report.epsilon0 = opt.epsilon0;
  report.theta_copy = opt.theta_copy;
  report.theta_cpu = opt.theta_cpu;
  report.k0_override = opt.k0;
  report.main_stream_override = opt.main_stream;
  report.warnings = std::move(warnings);
  if (a->census.n_devices > 1)  // streams.hpp:198-203
    report.warnings.push_back("MultiDeviceTrace: kept majority device '" + label_of(a->census.majority_device) +
                              "', dropped " + std::to_string(a->census.dropped_records) + " records from other devices");
  fill_streams(a->census, report.streams, report.classes);
  report.main_stream = a->main_stream;
  if (opt.main_stream) {
    if (a->main_stream_override_non_main)
      report.warnings.push_back("MainStreamOverride: stream " + std::to_string(*opt.main_stream) +
                                " carries no kernels but was selected by override");
  } else if (a->n_main_streams > 1) {  // streams.hpp:130-143
    std::string others;
    for (const auto& s : report.streams) {
      if (report.classes[s.stream] != StreamClass::Main || s.stream == a->main_stream) continue;
      if (!others.empty()) others += ", ";
      others += std::to_string(s.stream);
    }
    report.warnings.push_back("MultipleMainStreams: analyzing stream " + std::to_string(a->main_stream) +
                              " (most kernels); other kernel-bearing streams: " + others);
  }
  if (a->overlapping_kernels > 0)
    report.warnings.push_back("OverlappingKernels: " + std::to_string(a->overlapping_kernels) +
                              " consecutive main-stream records report overlapping intervals (timer granularity)");
  const DiagnosisThresholds thresholds{opt.theta_copy, opt.theta_cpu};
  for (uint32_t k = 0; k < a->n_loops; ++k) {
    const itt_loop_result& L = a->loops[k];
    LoopReport loop;
    loop.iterations_declared = L.iterations_declared;
    loop.pattern_length = L.pattern_length;
    loop.pattern_count = L.pattern_count;
    loop.epsilon_used = L.epsilon_used;
    loop.first_occurrence_token = L.first_token;
    loop.k0_used = L.k0_used;
    for (int64_t j = 0; j < L.pattern_length; ++j) loop.pattern_names.push_back(name_of(a->name_row[L.pattern_tokens[j]]));
    std::vector<IterationMetrics> items;
    items.reserve(L.n_iterations);
    for (uint64_t i = 0; i < L.n_iterations; ++i) items.push_back(to_metrics(L.rows[i], static_cast<int64_t>(i + 1)));
    if (L.clamps.negative_gap_clamps > 0)
      report.warnings.push_back("NegativeGaps: " + std::to_string(L.clamps.negative_gap_clamps) +
                                " negative dispatch gaps clamped to zero");
    if (L.clamps.negative_interval_clamps > 0)
      report.warnings.push_back("NegativeIntervals: " + std::to_string(L.clamps.negative_interval_clamps) +
                                " negative iteration intervals clamped to zero");
    loop.iterations_found = static_cast<int64_t>(items.size());
    loop.summary = itertrace::compute_summary(items, opt.loops[k]);
    loop.diagnosis = itertrace::diagnose(loop.summary, thresholds);
    report.loops.push_back(std::move(loop));
    result.details.push_back(std::move(items));
  }
  return result;
}

// itt_parse_csv result, released with the context's allocator
struct ParsedHold {
  itt_ctx* c;
  void operator()(itt_parsed_trace* p) const { itt_free_parsed(c, p); }
};
using ParsedPtr = std::unique_ptr<itt_parsed_trace, ParsedHold>;

// parse_trace (ingest.hpp:408-417) with parse_trace_text on the GPU: the file's text crosses to
// HBM once and the records stay there
inline ParsedPtr parse_file(Context& ctx, const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw Error(ErrorKind::UnreadableFile, "ingest: cannot open trace file '" + path + "'");
  const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  itt_parsed_trace* p = nullptr;
  ctx.check(itt_parse_csv(ctx.get(), text.data(), text.size(), path.c_str(), &p));
  return ParsedPtr(p, ParsedHold{ctx.get()});
}

inline IngestReport ingest_report(const itt_parsed_trace& p) {
  static const char* const kCols[7] = {"Start", "Duration", "Size", "Throughput", "Device", "Stream", "Name"};
  IngestReport r;
  r.rows_total = p.rows_total;
  r.rows_parsed = p.rows_parsed;
  r.rows_skipped = p.rows_skipped;
  for (uint64_t i = 0; i < p.n_skips; ++i) r.skip_reasons.emplace_back(p.skip_line[i], p.skip_reason[i]);
  for (int c = 0; c < 7; ++c)
    if (p.column[c] >= 0) r.column_map[kCols[c]] = static_cast<size_t>(p.column[c]);
  return r;
}

}  // namespace detail

// analyze_trace (pipeline.hpp:34-134): the device runs filter -> census -> tokens -> SA/LCP ->
// mining -> matching -> integer aggregates in one call; the host finishes with the reference's
// own compute_summary / diagnose and assembles warnings in the reference's order.
inline AnalysisResult analyze_trace(NormalizedTrace trace, const std::string& trace_label, const AnalyzeOptions& opt) {
  if (opt.loops.empty()) throw Error(ErrorKind::InvalidConfig, "analyze: at least one iteration count is required");
  Context& ctx = Context::thread_default();
  const detail::Columns cols(trace);
  const itt_records rv = cols.view();
  const detail::AnalysisPtr a = detail::run_analyze(ctx, rv, opt);
  return detail::assemble(
      a.get(), opt, trace_label, trace.warnings, [&](uint16_t d) { return cols.labels[d]; },
      [&](uint64_t row) { return trace.records[row].name; });
}

// The CLI's analyze body (itertrace_main.cpp:121-139, parse_trace + analyze_trace) with the CSV
// parsed on the GPU (itt_parse_csv) and analyzed where it lies.  Same Report, details, ingest
// counts, warnings and errors as the reference.
inline std::pair<AnalysisResult, IngestReport> analyze_csv_file(const std::string& path, const AnalyzeOptions& opt) {
  if (opt.loops.empty()) throw Error(ErrorKind::InvalidConfig, "analyze: at least one iteration count is required");
  Context& ctx = Context::thread_default();
  const detail::ParsedPtr p = detail::parse_file(ctx, path);
  const detail::AnalysisPtr a = detail::run_analyze(ctx, p->records, opt);
  // names of the pattern tokens: (offset, bytes) of their rows from the device columns
  auto name_of = [&](uint64_t row) {
    uint64_t off[2];
    ctx.check(itt_memcpy_d2h(ctx.get(), off, p->records.name_off + row, sizeof(off)));
    std::string name(off[1] - off[0], '\0');
    if (!name.empty()) ctx.check(itt_memcpy_d2h(ctx.get(), name.data(), p->records.name_bytes + off[0], name.size()));
    return name;
  };
  std::vector<std::string> warnings(p->warnings, p->warnings + p->n_warnings);
  AnalysisResult r = detail::assemble(
      a.get(), opt, path, std::move(warnings), [&](uint16_t d) { return std::string(p->device_labels[d]); }, name_of);
  return {std::move(r), detail::ingest_report(*p)};
}

// The CLI's inspect body (itertrace_main.cpp:141-149): parse_trace + summarize_streams +
// classify_streams (no device filter), the parse and the census on the GPU.
struct InspectResult {
  std::vector<StreamSummary> streams;
  std::map<std::uint32_t, StreamClass> classes;
  IngestReport ingest;
};
inline InspectResult inspect_csv_file(const std::string& path) {
  Context& ctx = Context::thread_default();
  const detail::ParsedPtr p = detail::parse_file(ctx, path);
  InspectResult out;
  out.ingest = detail::ingest_report(*p);
  if (p->records.n == 0) return out;
  itt_census c{};
  ctx.check(itt_summarize_streams(ctx.get(), &p->records, 0, &c));
  detail::fill_streams(c, out.streams, out.classes);
  itt_free(ctx.get(), c.streams);
  return out;
}

}  // namespace itertrace::cuda
