// oracle/ref_wrapper.cpp — C wrapper around the UNMODIFIED reference headers.
// TEST INFRASTRUCTURE ONLY (see ref_api.h).  Compiled by oracle/Makefile with
// -I/root/reference/proj/include into oracle/_ref/libitertrace_ref.so; nothing here
// re-implements reference logic, it only marshals columns into the reference's own
// types and calls its functions.
#include "ref_api.h"

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "itertrace/itertrace.hpp"

using namespace itertrace;

namespace {

char* dup_str(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.data(), s.size());
  p[s.size()] = 0;
  return p;
}

std::string device_label(uint16_t id) {
  char buf[16];
  std::snprintf(buf, sizeof(buf), "dev%05u", static_cast<unsigned>(id));  // lexicographic == numeric
  return buf;
}

// columns -> NormalizedTrace exactly as parse_trace_text leaves it: rows numbered from 1 in
// source order, then stable-sorted by (start, row) (ingest.hpp:396-400).
NormalizedTrace to_trace(const itt_records* r, double* order_ms = nullptr) {
  NormalizedTrace t;
  t.records.resize(r->n);
  for (uint64_t i = 0; i < r->n; ++i) {
    TraceRecord& x = t.records[i];
    x.start_ns = r->start_ns[i];
    x.duration_ns = r->duration_ns[i];
    if (r->flags[i] & ITT_REC_HAS_SIZE) x.size_bytes = r->size_bytes[i];
    if (r->flags[i] & ITT_REC_HAS_THROUGHPUT) x.throughput_bps = 1e9;
    x.device = device_label(r->device ? r->device[i] : 0);
    x.stream = r->stream[i];
    x.name.assign(reinterpret_cast<const char*>(r->name_bytes + r->name_off[i]), r->name_off[i + 1] - r->name_off[i]);
    x.row = static_cast<size_t>(i + 1);
  }
  const auto t0 = std::chrono::steady_clock::now();
  std::stable_sort(t.records.begin(), t.records.end(), [](const TraceRecord& a, const TraceRecord& b) {
    if (a.start_ns != b.start_ns) return a.start_ns < b.start_ns;
    return a.row < b.row;
  });
  if (order_ms) order_ms[0] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return t;
}

double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

int status_of(const Error& e) { return 1 + static_cast<int>(e.kind()); }

void fill_summaries(const std::vector<StreamSummary>& ss, const std::map<uint32_t, StreamClass>& cls,
                    itt_stream_summary* out) {
  for (size_t i = 0; i < ss.size(); ++i) {
    out[i].stream = ss[i].stream;
    auto it = cls.find(ss[i].stream);
    out[i].cls = it == cls.end() ? ITT_CLASS_ASSIST : static_cast<int32_t>(it->second);
    for (int k = 0; k < 6; ++k) out[i].counts[k] = ss[i].counts[static_cast<size_t>(k)];
    out[i].first_start = ss[i].first_start;
    out[i].last_end = ss[i].last_end;
  }
}

void fill_iter(const IterationMetrics& m, ref_iter* o) {
  o->index = m.index;
  o->start_token = m.span.start_token;
  o->end_token = m.span.end_token;
  o->extra = m.extra_ops;
  o->t_start = m.t_start;
  o->t_end = m.t_end;
  o->has_interval = m.interval_ns.has_value();
  o->interval_ns = m.interval_ns.value_or(0);
  o->has_overlap = m.overlap_ratio.has_value();
  o->overlap_ratio = m.overlap_ratio.value_or(0.0);
  o->htod_bytes = m.htod_bytes;
  o->op_gap_mean_ns = m.op_gap_mean_ns;
}

// analyze_trace (pipeline.hpp:34-134) with the same calls in the same order, timed per stage.
AnalysisResult staged_analyze(NormalizedTrace trace, const std::string& label, const AnalyzeOptions& opt,
                              ref_stage_times* tm) {
  using clk = std::chrono::steady_clock;
  if (opt.loops.empty()) throw Error(ErrorKind::InvalidConfig, "analyze: at least one iteration count is required");
  AnalysisResult result;
  Report& report = result.report;
  report.trace_path = label;
  report.epsilon0 = opt.epsilon0;
  report.theta_copy = opt.theta_copy;
  report.theta_cpu = opt.theta_cpu;
  report.k0_override = opt.k0;
  report.main_stream_override = opt.main_stream;
  auto t0 = clk::now();
  auto filtered = filter_majority_device(std::move(trace));
  const NormalizedTrace& working = filtered.trace;
  report.warnings = working.warnings;
  for (auto& w : filtered.warnings) report.warnings.push_back(w);
  report.streams = summarize_streams(working);
  report.classes = classify_streams(report.streams);
  if (opt.main_stream) {
    report.main_stream = *opt.main_stream;
    const auto it = report.classes.find(*opt.main_stream);
    if (it == report.classes.end())
      throw Error(ErrorKind::EmptyMainStream, "stream-classify: override stream " + std::to_string(*opt.main_stream) +
                                                  " does not appear in the trace");
    if (it->second != StreamClass::Main)
      report.warnings.push_back("MainStreamOverride: stream " + std::to_string(*opt.main_stream) +
                                " carries no kernels but was selected by override");
  } else {
    auto choice = select_main_stream(report.classes, report.streams);
    report.main_stream = choice.stream;
    for (auto& w : choice.warnings) report.warnings.push_back(w);
  }
  tm->filter_census_ms = ms_since(t0);
  t0 = clk::now();
  const auto seq = build_token_sequence(working, report.main_stream);
  const auto overlaps = count_interval_overlaps(working, report.main_stream);
  tm->intern_ms = ms_since(t0);
  if (overlaps > 0)
    report.warnings.push_back("OverlappingKernels: " + std::to_string(overlaps) +
                              " consecutive main-stream records report overlapping intervals (timer granularity)");
  t0 = clk::now();
  std::vector<MiningConfig> configs;
  for (const auto iters : opt.loops) configs.push_back({iters, opt.epsilon0, std::nullopt});
  std::vector<PatternCandidate> patterns;
  if (configs.size() == 1) patterns.push_back(mine_pattern(seq, configs.front()));
  else patterns = mine_patterns_multi(seq, configs);
  tm->mine_ms = ms_since(t0);
  t0 = clk::now();
  const auto htod = collect_htod_records(working);
  const DiagnosisThresholds thresholds{opt.theta_copy, opt.theta_cpu};
  tm->metrics_ms = ms_since(t0);
  tm->match_ms = 0;
  for (size_t k = 0; k < patterns.size(); ++k) {
    const auto& pattern = patterns[k];
    LoopReport loop;
    loop.iterations_declared = opt.loops[k];
    loop.pattern_length = pattern.length();
    loop.pattern_count = pattern.count;
    loop.epsilon_used = pattern.epsilon_used;
    loop.first_occurrence_token = pattern.first_token;
    for (const auto tok : pattern.tokens) loop.pattern_names.push_back(seq.name_of(tok));
    t0 = clk::now();
    const MatchConfig match_cfg{opt.k0.value_or(default_k0(pattern.length()))};
    loop.k0_used = match_cfg.k0;
    const auto spans = approx_match(seq, pattern.tokens, match_cfg);
    if (const auto v = validate_spans(spans, seq.tokens, pattern.tokens, match_cfg); !v.empty())
      throw Error(ErrorKind::InvalidConfig, "matching: internal span contract violated: " + v.front().message);
    tm->match_ms += ms_since(t0);
    t0 = clk::now();
    const auto windows = partition_iterations(working, seq, spans);
    auto analysis = compute_iteration_metrics(working, seq, windows, htod);
    if (analysis.negative_gap_clamps > 0)
      report.warnings.push_back("NegativeGaps: " + std::to_string(analysis.negative_gap_clamps) +
                                " negative dispatch gaps clamped to zero");
    if (analysis.negative_interval_clamps > 0)
      report.warnings.push_back("NegativeIntervals: " + std::to_string(analysis.negative_interval_clamps) +
                                " negative iteration intervals clamped to zero");
    loop.iterations_found = static_cast<int64_t>(analysis.iterations.size());
    loop.summary = compute_summary(analysis.iterations, opt.loops[k]);
    loop.diagnosis = diagnose(loop.summary, thresholds);
    tm->metrics_ms += ms_since(t0);
    report.loops.push_back(std::move(loop));
    result.details.push_back(std::move(analysis.iterations));
  }
  return result;
}

}  // namespace

extern "C" int ref_analyze(const itt_records* recs, const itt_analyze_opts* opts, int staged, ref_analysis* out) {
  std::memset(out, 0, sizeof(*out));
  const auto t_all = std::chrono::steady_clock::now();
  try {
    AnalyzeOptions opt;
    for (uint32_t i = 0; i < opts->n_loops; ++i) opt.loops.push_back(opts->loops[i]);
    opt.epsilon0 = opts->epsilon0;
    if (opts->k0 >= 0) opt.k0 = opts->k0;
    if (opts->main_stream >= 0) opt.main_stream = static_cast<uint32_t>(opts->main_stream);
    NormalizedTrace trace = to_trace(recs, &out->times.order_ms);
    AnalysisResult res;
    const auto t_an = std::chrono::steady_clock::now();
    if (staged) res = staged_analyze(std::move(trace), "trace.csv", opt, &out->times);
    else res = analyze_trace(std::move(trace), "trace.csv", opt);
    out->times.analyze_ms = ms_since(t_an);
    const Report& rep = res.report;
    out->n_streams = static_cast<uint32_t>(rep.streams.size());
    out->streams = static_cast<itt_stream_summary*>(std::calloc(rep.streams.size() + 1, sizeof(itt_stream_summary)));
    fill_summaries(rep.streams, rep.classes, out->streams);
    out->main_stream = rep.main_stream;
    out->n_loops = static_cast<uint32_t>(rep.loops.size());
    out->loops = static_cast<ref_loop*>(std::calloc(rep.loops.size() + 1, sizeof(ref_loop)));
    for (size_t k = 0; k < rep.loops.size(); ++k) {
      const LoopReport& l = rep.loops[k];
      ref_loop& o = out->loops[k];
      o.iterations_declared = l.iterations_declared;
      o.pattern_length = l.pattern_length;
      o.pattern_count = l.pattern_count;
      o.epsilon_used = l.epsilon_used;
      o.first_token = l.first_occurrence_token;
      o.k0_used = l.k0_used;
      o.pattern_tokens = nullptr;  // names only at this level; token ids via ref_mine_patterns
      o.n_iterations = res.details[k].size();
      o.iters = static_cast<ref_iter*>(std::calloc(res.details[k].size() + 1, sizeof(ref_iter)));
      for (size_t i = 0; i < res.details[k].size(); ++i) fill_iter(res.details[k][i], &o.iters[i]);
      o.avg_interval_ns = l.summary.avg_interval_ns;
      o.avg_overlap = l.summary.avg_overlap;
      o.avg_operation_ns = l.summary.avg_operation_ns;
      o.avg_size_bytes = l.summary.avg_size_bytes;
      o.max_interval_ns = l.summary.max_interval_ns;
      o.insufficient_intervals = l.summary.insufficient_intervals;
      o.diagnosis = static_cast<int32_t>(l.diagnosis.code);
    }
    std::string w;
    for (size_t i = 0; i < rep.warnings.size(); ++i) {
      if (i) w += '\n';
      w += rep.warnings[i];
    }
    out->warnings = dup_str(w);
    out->summary_json = dup_str(summary_to_json(rep).dump(2) + "\n");
    out->details_csv = dup_str(res.details.empty() ? std::string() : details_to_csv(res.details[0]));
  } catch (const Error& e) {
    out->status = status_of(e);
    out->error = dup_str(e.what());
  } catch (const std::exception& e) {
    out->status = 1000;
    out->error = dup_str(e.what());
  }
  out->times.total_ms = ms_since(t_all);
  return out->status;
}

extern "C" void ref_free_analysis(ref_analysis* a) {
  if (!a) return;
  for (uint32_t k = 0; k < a->n_loops; ++k) {
    std::free(a->loops[k].iters);
    std::free(a->loops[k].pattern_tokens);
  }
  std::free(a->loops);
  std::free(a->streams);
  std::free(a->error);
  std::free(a->warnings);
  std::free(a->summary_json);
  std::free(a->details_csv);
  std::memset(a, 0, sizeof(*a));
}

extern "C" int ref_suffix_array(const int32_t* tokens, uint64_t n, int32_t term, uint32_t* sa, uint32_t* lcp) {
  try {
    const SuffixTree tree(std::span<const int32_t>(tokens, n), term);
    const auto& nodes = tree.nodes();
    const int64_t np = static_cast<int64_t>(n) + 1;
    // iterative DFS, children visited in ascending key order (std::map order)
    std::vector<int32_t> stack{0};
    uint64_t k = 0;
    while (!stack.empty()) {
      const int32_t v = stack.back();
      stack.pop_back();
      const auto& node = nodes[static_cast<size_t>(v)];
      if (node.is_leaf()) {
        sa[k++] = static_cast<uint32_t>(np - node.depth);
        continue;
      }
      for (auto it = node.children.rbegin(); it != node.children.rend(); ++it) stack.push_back(it->second);
    }
    if (k != static_cast<uint64_t>(np)) return 1000;
    if (lcp) {  // Kasai over tokens+[term]
      std::vector<int32_t> text(tokens, tokens + n);
      text.push_back(term);
      std::vector<uint32_t> rank(static_cast<size_t>(np));
      for (int64_t j = 0; j < np; ++j) rank[sa[j]] = static_cast<uint32_t>(j);
      int64_t h = 0;
      lcp[0] = 0;
      for (int64_t i = 0; i < np; ++i) {
        if (rank[static_cast<size_t>(i)] > 0) {
          const int64_t j = sa[rank[static_cast<size_t>(i)] - 1];
          while (i + h < np && j + h < np && text[static_cast<size_t>(i + h)] == text[static_cast<size_t>(j + h)]) ++h;
          lcp[rank[static_cast<size_t>(i)]] = static_cast<uint32_t>(h);
          if (h > 0) --h;
        } else {
          h = 0;
        }
      }
    }
  } catch (const Error& e) {
    return status_of(e);
  }
  return 0;
}

extern "C" int ref_enumerate_repeats(const int32_t* tokens, uint64_t n, int32_t term, int64_t min_count, int64_t max_len,
                                     itt_repeat** out, uint64_t* n_out) {
  const SuffixTree tree(std::span<const int32_t>(tokens, n), term);
  const auto reps = enumerate_repeats(tree, min_count, max_len);
  *out = static_cast<itt_repeat*>(std::malloc((reps.size() + 1) * sizeof(itt_repeat)));
  for (size_t i = 0; i < reps.size(); ++i) (*out)[i] = itt_repeat{reps[i].start, reps[i].length, reps[i].count};
  *n_out = reps.size();
  return 0;
}

extern "C" int ref_mine_patterns(const int32_t* tokens, uint64_t n, uint32_t n_names, const itt_mining_cfg* loops,
                                 uint32_t n_loops, int multi, itt_pattern* out, char* err, uint64_t err_cap) {
  try {
    TokenSequence seq;
    seq.tokens.assign(tokens, tokens + n);
    for (uint32_t v = 0; v < n_names; ++v) seq.names.push_back("t" + std::to_string(v));
    std::vector<MiningConfig> cfgs;
    for (uint32_t i = 0; i < n_loops; ++i) {
      MiningConfig c{loops[i].iterations, loops[i].epsilon0, std::nullopt};
      if (loops[i].epsilon_cap > 0) c.epsilon_cap = loops[i].epsilon_cap;
      cfgs.push_back(c);
    }
    std::vector<PatternCandidate> res;
    if (multi) res = mine_patterns_multi(seq, cfgs);
    else res.push_back(mine_pattern(seq, cfgs.front()));
    for (size_t i = 0; i < res.size(); ++i) {
      out[i].length = res[i].length();
      out[i].tokens = static_cast<int32_t*>(std::malloc((res[i].tokens.size() + 1) * 4));
      std::memcpy(out[i].tokens, res[i].tokens.data(), res[i].tokens.size() * 4);
      out[i].count = res[i].count;
      out[i].first_token = res[i].first_token;
      out[i].epsilon_used = res[i].epsilon_used;
    }
  } catch (const Error& e) {
    if (err && err_cap) std::snprintf(err, err_cap, "%s", e.what());
    return status_of(e);
  }
  return 0;
}

extern "C" int ref_approx_match(const int32_t* tokens, uint64_t n, const int32_t* pattern, uint64_t m, int64_t k0,
                                itt_span** out, uint64_t* n_out) {
  const auto spans = approx_match(std::span<const int32_t>(tokens, n), std::span<const int32_t>(pattern, m), MatchConfig{k0});
  *out = static_cast<itt_span*>(std::malloc((spans.size() + 1) * sizeof(itt_span)));
  for (size_t i = 0; i < spans.size(); ++i) (*out)[i] = itt_span{spans[i].start_token, spans[i].end_token, spans[i].extra};
  *n_out = spans.size();
  return 0;
}

extern "C" int ref_build_token_sequence(const itt_records* recs, uint32_t main_stream, int32_t* tokens,
                                        uint64_t* record_index, uint64_t* n_out, uint32_t* n_names, uint64_t* name_row) {
  try {
    const NormalizedTrace t = to_trace(recs);
    const auto seq = build_token_sequence(t, main_stream);
    for (size_t i = 0; i < seq.tokens.size(); ++i) {
      tokens[i] = seq.tokens[i];
      record_index[i] = seq.record_index[i];
    }
    *n_out = seq.tokens.size();
    *n_names = static_cast<uint32_t>(seq.names.size());
    if (name_row) {  // first record (source row) carrying each name
      std::vector<int> seen(seq.names.size(), 0);
      for (size_t i = 0; i < seq.tokens.size(); ++i) {
        const auto v = static_cast<size_t>(seq.tokens[i]);
        if (!seen[v]) {
          seen[v] = 1;
          name_row[v] = t.records[seq.record_index[i]].row - 1;
        }
      }
    }
  } catch (const Error& e) {
    return status_of(e);
  }
  return 0;
}

extern "C" int ref_iteration_metrics(const itt_records* recs, uint32_t main_stream, const itt_span* spans, uint64_t n_spans,
                                     ref_iter* rows, itt_clamps* clamps) {
  try {
    const NormalizedTrace t = to_trace(recs);
    const auto seq = build_token_sequence(t, main_stream);
    std::vector<MatchSpan> sp;
    for (uint64_t i = 0; i < n_spans; ++i) sp.push_back(MatchSpan{spans[i].start_token, spans[i].end_token, spans[i].extra});
    const auto windows = partition_iterations(t, seq, sp);
    const auto a = compute_iteration_metrics(t, seq, windows, collect_htod_records(t));
    for (size_t i = 0; i < a.iterations.size(); ++i) fill_iter(a.iterations[i], &rows[i]);
    clamps->negative_gap_clamps = a.negative_gap_clamps;
    clamps->negative_interval_clamps = a.negative_interval_clamps;
  } catch (const Error& e) {
    return status_of(e);
  }
  return 0;
}

extern "C" int ref_summarize_streams(const itt_records* recs, int filter_device, itt_stream_summary* out, uint32_t cap,
                                     uint32_t* n_out, uint64_t* dropped) {
  try {
    NormalizedTrace t = to_trace(recs);
    const uint64_t before = t.records.size();
    if (filter_device) t = filter_majority_device(std::move(t)).trace;
    *dropped = before - t.records.size();
    const auto ss = summarize_streams(t);
    const auto cls = classify_streams(ss);
    *n_out = static_cast<uint32_t>(ss.size());
    if (ss.size() > cap) return 1000;
    fill_summaries(ss, cls, out);
  } catch (const Error& e) {
    return status_of(e);
  }
  return 0;
}

extern "C" void ref_free(void* p) { std::free(p); }

// ---- CSV ingest through the reference (test infrastructure)
extern "C" int ref_parse_csv(const char* text, uint64_t len, const char* label, ref_parsed* out) {
  std::memset(out, 0, sizeof(*out));
  try {
    auto [trace, rep] = parse_trace_text(std::string_view(text, len), label);
    const size_t n = trace.records.size();
    out->n = n;
    out->start_ns = static_cast<int64_t*>(std::calloc(n + 1, 8));
    out->duration_ns = static_cast<int64_t*>(std::calloc(n + 1, 8));
    out->size_bytes = static_cast<int64_t*>(std::calloc(n + 1, 8));
    out->flags = static_cast<uint8_t*>(std::calloc(n + 1, 1));
    out->stream = static_cast<uint32_t*>(std::calloc(n + 1, 4));
    out->row = static_cast<uint64_t*>(std::calloc(n + 1, 8));
    out->name_off = static_cast<uint64_t*>(std::calloc(n + 1, 8));
    out->device_off = static_cast<uint64_t*>(std::calloc(n + 1, 8));
    std::string names, devs;
    for (size_t i = 0; i < n; ++i) {
      const TraceRecord& r = trace.records[i];
      out->start_ns[i] = r.start_ns;
      out->duration_ns[i] = r.duration_ns;
      if (r.size_bytes) out->size_bytes[i] = *r.size_bytes, out->flags[i] |= ITT_REC_HAS_SIZE;
      if (r.throughput_bps) out->flags[i] |= ITT_REC_HAS_THROUGHPUT;
      out->stream[i] = r.stream;
      out->row[i] = r.row;
      out->name_off[i] = names.size();
      names += r.name;
      out->device_off[i] = devs.size();
      devs += r.device;
    }
    out->name_off[n] = names.size();
    out->device_off[n] = devs.size();
    out->name_bytes = static_cast<uint8_t*>(std::malloc(names.size() + 1));
    std::memcpy(out->name_bytes, names.data(), names.size());
    out->device_bytes = static_cast<uint8_t*>(std::malloc(devs.size() + 1));
    std::memcpy(out->device_bytes, devs.data(), devs.size());
    out->rows_total = rep.rows_total;
    out->rows_parsed = rep.rows_parsed;
    out->rows_skipped = rep.rows_skipped;
    out->n_skips = rep.skip_reasons.size();
    out->skip_line = static_cast<uint64_t*>(std::calloc(rep.skip_reasons.size() + 1, 8));
    std::string why;
    for (size_t i = 0; i < rep.skip_reasons.size(); ++i) {
      out->skip_line[i] = rep.skip_reasons[i].first;
      if (i) why += '\n';
      why += rep.skip_reasons[i].second;
    }
    out->skip_reasons = dup_str(why);
    const char* cols[7] = {"Start", "Duration", "Size", "Throughput", "Device", "Stream", "Name"};
    for (int q = 0; q < 7; ++q) {
      auto it = rep.column_map.find(cols[q]);
      out->column[q] = it == rep.column_map.end() ? -1 : static_cast<int32_t>(it->second);
    }
    std::string w;
    for (size_t i = 0; i < trace.warnings.size(); ++i) {
      if (i) w += '\n';
      w += trace.warnings[i];
    }
    out->warnings = dup_str(w);
  } catch (const Error& e) {
    out->status = status_of(e);
    out->error = dup_str(e.what());
  } catch (const std::exception& e) {
    out->status = 1000;
    out->error = dup_str(e.what());
  }
  return out->status;
}

extern "C" void ref_free_parsed(ref_parsed* p) {
  if (!p) return;
  for (void* x : {static_cast<void*>(p->start_ns), static_cast<void*>(p->duration_ns), static_cast<void*>(p->size_bytes),
                  static_cast<void*>(p->flags), static_cast<void*>(p->stream), static_cast<void*>(p->row),
                  static_cast<void*>(p->name_off), static_cast<void*>(p->name_bytes), static_cast<void*>(p->device_off),
                  static_cast<void*>(p->device_bytes), static_cast<void*>(p->skip_line), static_cast<void*>(p->skip_reasons),
                  static_cast<void*>(p->error), static_cast<void*>(p->warnings)})
    std::free(x);
  std::memset(p, 0, sizeof(*p));
}

extern "C" char* ref_synth_csv(uint64_t seed, int64_t pattern_len, int64_t iterations, int64_t vocab_size, double insert_prob,
                               int64_t max_inserts, int32_t inside_pattern, int32_t pathology, uint64_t* len) {
  SynthConfig cfg;
  cfg.seed = seed;
  cfg.pattern_len = pattern_len;
  cfg.iterations = iterations;
  cfg.vocab_size = vocab_size;
  cfg.insert_prob = insert_prob;
  cfg.max_inserts = max_inserts;
  cfg.insert_placement = inside_pattern ? InsertPlacement::inside_pattern : InsertPlacement::after_pattern;
  cfg.pathology = static_cast<Pathology>(pathology);
  try {
    const std::string csv = generate(cfg).trace_csv;
    *len = csv.size();
    return dup_str(csv);
  } catch (const std::exception&) {  // invalid generator config
    *len = 0;
    return nullptr;
  }
}

extern "C" int ref_analyze_csv(const char* text, uint64_t len, const char* label, const itt_analyze_opts* opts,
                               ref_analysis* out) {
  std::memset(out, 0, sizeof(*out));
  try {
    AnalyzeOptions opt;
    for (uint32_t i = 0; i < opts->n_loops; ++i) opt.loops.push_back(opts->loops[i]);
    opt.epsilon0 = opts->epsilon0;
    if (opts->k0 >= 0) opt.k0 = opts->k0;
    if (opts->main_stream >= 0) opt.main_stream = static_cast<uint32_t>(opts->main_stream);
    auto [trace, rep] = parse_trace_text(std::string_view(text, len), label);
    (void)rep;
    const AnalysisResult res = analyze_trace(std::move(trace), label, opt);
    std::string w;
    for (size_t i = 0; i < res.report.warnings.size(); ++i) {
      if (i) w += '\n';
      w += res.report.warnings[i];
    }
    out->warnings = dup_str(w);
    out->summary_json = dup_str(summary_to_json(res.report).dump(2) + "\n");
    out->details_csv = dup_str(res.details.empty() ? std::string() : details_to_csv(res.details[0]));
  } catch (const Error& e) {
    out->status = status_of(e);
    out->error = dup_str(e.what());
  } catch (const std::exception& e) {
    out->status = 1000;
    out->error = dup_str(e.what());
  }
  return out->status;
}

// nlohmann::json(v).dump() of one double (pins the Python Grisu2 restatement, jsonfloat.py)
extern "C" int ref_json_double(double v, char* out, int cap) {
  const std::string s = nlohmann::json(v).dump();
  if (static_cast<int>(s.size()) + 1 > cap) return -1;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return static_cast<int>(s.size());
}
