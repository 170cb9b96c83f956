// dropin_test.cpp — the C++ drop-in (include/itertrace_cuda.hpp) against the reference, in C++.
//
// TEST INFRASTRUCTURE: compiled by oracle/Makefile against the reference headers (only where
// /root/reference exists) into oracle/_ref/dropin_test; run on the GPU box by
// tests/test_gpu_dropin.py.  For each trace — produced by the REFERENCE's own generator
// (synth.hpp:187-372), rendered to CSV and parsed by the reference's ingest
// (ingest.hpp:154-402) — it runs itertrace::analyze_trace and itertrace::cuda::analyze_trace
// and requires byte-identical summary JSON and details CSV (or the same error kind and
// message), plus the stage functions one by one.  The configs follow the reference's
// acceptance criterion 4 (acceptance.cpp:65-85,164-184) and its pathologies (:215-254).
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "itertrace/itertrace.hpp"
#include "itertrace_cuda.hpp"

using namespace itertrace;

namespace {

int failures = 0, checks = 0;

void expect(bool ok, const std::string& what) {
  ++checks;
  if (!ok) {
    ++failures;
    std::fprintf(stderr, "MISMATCH: %s\n", what.c_str());
  }
}

SynthConfig random_recovery_config(std::mt19937_64& rng, int index) {  // acceptance.cpp:65-85
  SynthConfig cfg;
  cfg.seed = 77'000 + static_cast<std::uint64_t>(index);
  cfg.pattern_len = 5 + static_cast<std::int64_t>(rng() % 46);
  cfg.iterations = 50 + static_cast<std::int64_t>(rng() % 951);
  cfg.insert_prob = static_cast<double>(rng() % 31) / 100.0;
  cfg.max_inserts = static_cast<std::int64_t>(rng() % 3);
  cfg.init_ops = 1 + static_cast<std::int64_t>(rng() % 10);
  cfg.vocab_size = cfg.pattern_len + 1 + static_cast<std::int64_t>(rng() % 8);
  cfg.kernel_duration_ns = 2000 + static_cast<std::int64_t>(rng() % 2000);
  cfg.kernel_jitter_ns = static_cast<std::int64_t>(rng() % static_cast<std::uint64_t>(cfg.kernel_duration_ns / 4));
  cfg.intra_gap_ns = 500 + static_cast<std::int64_t>(rng() % 1000);
  cfg.interval_gap_ns = 4000 + static_cast<std::int64_t>(rng() % 8000);
  cfg.interval_jitter_ns = static_cast<std::int64_t>(rng() % static_cast<std::uint64_t>(cfg.interval_gap_ns / 4));
  cfg.htod_bytes_per_iter = 1024 + static_cast<std::int64_t>(rng() % 8192);
  return cfg;
}

struct Outcome {
  std::string summary, details, error;
};

template <typename F>
Outcome run(F&& f) {
  Outcome o;
  try {
    AnalysisResult r = f();
    o.summary = summary_to_json(r.report).dump(2) + "\n";
    for (const auto& d : r.details) o.details += details_to_csv(d) + "\x1e";
  } catch (const Error& e) {
    o.error = std::to_string(static_cast<int>(e.kind())) + ": " + e.what();
  }
  return o;
}

void compare_trace(const std::string& tag, const NormalizedTrace& trace, const AnalyzeOptions& opt) {
  const Outcome want = run([&] { return itertrace::analyze_trace(trace, "t.csv", opt); });
  const Outcome got = run([&] { return itertrace::cuda::analyze_trace(trace, "t.csv", opt); });
  expect(want.error == got.error, tag + " error: [" + want.error + "] vs [" + got.error + "]");
  expect(want.summary == got.summary, tag + " summary json");
  expect(want.details == got.details, tag + " details csv");
  if (!want.error.empty() || opt.loops.size() != 1) return;
  // stage functions one by one on the filtered trace
  const auto filtered = filter_majority_device(trace).trace;
  const auto classes = classify_streams(summarize_streams(filtered));
  const auto main = select_main_stream(classes, summarize_streams(filtered)).stream;
  const auto seq = itertrace::build_token_sequence(filtered, main);
  const auto gseq = itertrace::cuda::build_token_sequence(filtered, main);
  expect(seq.tokens == gseq.tokens && seq.record_index == gseq.record_index && seq.names == gseq.names, tag + " tokens");
  expect(count_interval_overlaps(filtered, main) == itertrace::cuda::count_interval_overlaps(filtered, main),
         tag + " overlaps");
  const MiningConfig mc{opt.loops[0], opt.epsilon0, std::nullopt};
  const auto p = itertrace::mine_pattern(seq, mc);
  const auto gp = itertrace::cuda::mine_pattern(seq, mc);
  expect(p.tokens == gp.tokens && p.count == gp.count && p.first_token == gp.first_token &&
             p.epsilon_used == gp.epsilon_used,
         tag + " mine_pattern");
  const MatchConfig k{opt.k0.value_or(default_k0(p.length()))};
  const auto spans = itertrace::approx_match(seq, p.tokens, k);
  expect(spans == itertrace::cuda::approx_match(seq, p.tokens, k), tag + " approx_match");
  const auto windows = partition_iterations(filtered, seq, spans);
  const auto ma = compute_iteration_metrics(filtered, seq, windows, collect_htod_records(filtered));
  const auto ga = itertrace::cuda::compute_iteration_metrics(filtered, seq, windows);
  bool same = ma.iterations.size() == ga.iterations.size() && ma.negative_gap_clamps == ga.negative_gap_clamps &&
              ma.negative_interval_clamps == ga.negative_interval_clamps;
  for (size_t i = 0; same && i < ma.iterations.size(); ++i) {
    const auto &a = ma.iterations[i], &b = ga.iterations[i];
    same = a.t_start == b.t_start && a.t_end == b.t_end && a.interval_ns == b.interval_ns &&
           a.overlap_ratio == b.overlap_ratio && a.htod_bytes == b.htod_bytes && a.op_gap_mean_ns == b.op_gap_mean_ns &&
           a.extra_ops == b.extra_ops && a.span == b.span;
  }
  expect(same, tag + " compute_iteration_metrics");
  // a12 (no reference function): its idle column must reproduce the reference's op-gap means
  // and its counts the span lengths; cells and totals must agree with each other
  const auto op = itertrace::cuda::op_profile(filtered, seq, windows, true);
  bool a12 = op.per_iteration.size() == ma.iterations.size();
  for (size_t i = 0; a12 && i < ma.iterations.size(); ++i) {
    const auto& m = ma.iterations[i];
    const int64_t gc = m.span.end_token - m.span.start_token;
    const double mean = gc > 0 ? static_cast<double>(op.per_iteration[i].idle_ns) / static_cast<double>(gc) : 0.0;
    a12 = mean == m.op_gap_mean_ns;
  }
  std::vector<int64_t> cnt(op.per_iteration.size(), 0), idle(op.per_op.size(), 0);
  for (const auto& c : op.cells) cnt[c.iteration] += c.count, idle[c.op] += c.idle_ns;
  for (size_t i = 0; a12 && i < cnt.size(); ++i)
    a12 = cnt[i] == ma.iterations[i].span.end_token - ma.iterations[i].span.start_token + 1;
  for (size_t v = 0; a12 && v < idle.size(); ++v) a12 = idle[v] == op.per_op[v].idle_ns;
  expect(a12, tag + " op_profile (a12) vs reference gap means");
}

NormalizedTrace trace_of(const SynthConfig& cfg) {
  return parse_trace_text(generate(cfg).trace_csv, "synth").first;
}

}  // namespace

int main() {
  std::mt19937_64 rng(1003);
  int n = 0;
  for (int index = 0; index < 100; ++index, ++n) {  // acceptance criterion 4 configs
    const auto cfg = random_recovery_config(rng, index);
    AnalyzeOptions opt;
    opt.loops = {cfg.iterations};
    opt.k0 = cfg.max_inserts;
    compare_trace("recovery_" + std::to_string(index), trace_of(cfg), opt);
  }
  for (int index = 0; index < 20; ++index, ++n) {  // inside-pattern inserts, default k0
    auto cfg = random_recovery_config(rng, 500 + index);
    cfg.insert_placement = InsertPlacement::inside_pattern;
    cfg.max_inserts = 1 + index % 3;
    cfg.insert_prob = 0.3;
    AnalyzeOptions opt;
    opt.loops = {cfg.iterations};
    compare_trace("inside_" + std::to_string(index), trace_of(cfg), opt);
  }
  {  // pathologies (acceptance.cpp:215-254) and option variants
    SynthConfig cfg;
    cfg.iterations = 200;
    cfg.pattern_len = 12;
    cfg.vocab_size = 20;
    for (auto [p, f] : {std::pair{Pathology::graph_growth, 8.0}, std::pair{Pathology::oversize_copy, 64.0}}) {
      cfg.pathology = p;
      cfg.pathology_factor = f;
      AnalyzeOptions opt;
      opt.loops = {200};
      compare_trace(std::string("pathology_") + to_string(p), trace_of(cfg), opt), ++n;
    }
    cfg.pathology = Pathology::none;
    const auto t = trace_of(cfg);
    for (const auto& loops : std::vector<std::vector<std::int64_t>>{{200}, {150}, {400}, {1}, {200, 100}, {200, 200}}) {
      AnalyzeOptions opt;
      opt.loops = loops;
      compare_trace("loops_" + std::to_string(loops.size()) + "_" + std::to_string(loops[0]), t, opt), ++n;
    }
    for (std::int64_t eps0 : {2, 16}) {
      AnalyzeOptions opt;
      opt.loops = {210};
      opt.epsilon0 = eps0;
      compare_trace("eps0_" + std::to_string(eps0), t, opt), ++n;
    }
    for (std::uint32_t ms : {13u, 14u, 99u}) {
      AnalyzeOptions opt;
      opt.loops = {200};
      opt.main_stream = ms;
      compare_trace("main_override_" + std::to_string(ms), t, opt), ++n;
    }
  }
  std::printf("dropin: %d traces, %d checks, %d mismatches\n", n, checks, failures);
  return failures == 0 ? 0 : 1;
}
