// oracle/ref_digest.cpp — reference outputs at BASELINE scale (TEST INFRASTRUCTURE ONLY).
//
// Runs the UNMODIFIED reference (headers under /root/reference/proj/include, compiled in place
// by oracle/Makefile) on a BASELINE-shaped trace from the repo's generator (include/itt_synth.h)
// and writes its outputs as files, so tests/golden/make_baseline_digests.py can commit their
// SHA-256 digests.  It exists because the Python route (ctypes columns + the reference's AoS
// NormalizedTrace + the suffix tree) does not fit C3 (100M events) into this container's 62 GB:
// here the generator's columns are released as soon as the AoS trace exists.
//
//   ref_digest analyze <outdir> <seed> <iterations> <body_len> <vocab> <noise> <shuffle>
//       stock analyze_trace (pipeline.hpp:34-134) -> summary.json (summary_to_json(report).dump(2)
//       + "\n", report.hpp:304), details.csv (details_to_csv, report.hpp:191-220), pattern.txt
//   ref_digest sa <outdir> <seed> <iterations> <body_len> <vocab> <noise> <shuffle>
//       device filter + stream selection + build_token_sequence (pipeline.hpp:49-75,
//       streams.hpp:147-169) -> tokens.u32; SuffixTree(tokens, V) leaf order -> sa.u32; Kasai
//       over it -> lcp.u32 (ref_suffix_array, SURVEY §8c's extraction)
#include "ref_wrapper.cpp"  // one translation unit: reuse to_trace() and ref_suffix_array()

#include <fstream>

#include "itt_synth.h"

namespace {

void write_file(const std::string& path, const void* p, size_t n) {
  std::ofstream f(path, std::ios::binary);
  f.write(static_cast<const char*>(p), static_cast<std::streamsize>(n));
  if (!f) throw std::runtime_error("cannot write " + path);
}

itt_records records_of(const itt_synth_trace& t) {
  itt_records r{};
  r.n = t.n;
  r.start_ns = t.start_ns;
  r.duration_ns = t.duration_ns;
  r.size_bytes = t.size_bytes;
  r.flags = t.flags;
  r.stream = t.stream;
  r.device = t.device;
  r.name_off = t.name_off;
  r.name_bytes = t.name_bytes;
  r.mem = ITT_MEM_HOST;
  r.order = ITT_ORDER_UNKNOWN;
  return r;
}

double secs(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

int main(int argc, char** argv) {
  if (argc != 9) {
    std::fprintf(stderr, "usage: %s analyze|sa <outdir> <seed> <iterations> <body_len> <vocab> <noise> <shuffle>\n",
                 argv[0]);
    return 2;
  }
  const std::string mode = argv[1], out = argv[2];
  itt_synth_cfg cfg;
  itt_synth_default(&cfg);
  cfg.seed = std::strtoull(argv[3], nullptr, 10);
  cfg.iterations = std::strtoll(argv[4], nullptr, 10);
  cfg.body_len = std::strtoll(argv[5], nullptr, 10);
  cfg.vocab = std::strtoll(argv[6], nullptr, 10);
  cfg.noise_frac = std::strtod(argv[7], nullptr);
  cfg.shuffle_window = std::strtoll(argv[8], nullptr, 10);
  const auto t0 = std::chrono::steady_clock::now();
  itt_synth_trace st;
  if (itt_synth_generate(&cfg, &st) != 0) {
    std::fprintf(stderr, "generator failed\n");
    return 1;
  }
  const itt_records recs = records_of(st);
  NormalizedTrace trace = to_trace(&recs);
  const uint64_t n_events = st.n;
  itt_synth_free(&st);  // the AoS trace is all the reference needs from here on
  std::fprintf(stderr, "[ref_digest] %llu events as NormalizedTrace in %.1f s\n",
               static_cast<unsigned long long>(n_events), secs(t0));
  try {
    if (mode == "analyze") {
      AnalyzeOptions opt;
      opt.loops.push_back(cfg.iterations);
      const auto t1 = std::chrono::steady_clock::now();
      const AnalysisResult res = analyze_trace(std::move(trace), "trace.csv", opt);
      const double dt = secs(t1);
      const std::string js = summary_to_json(res.report).dump(2) + "\n";
      const std::string csv = details_to_csv(res.details.at(0));
      write_file(out + "/summary.json", js.data(), js.size());
      write_file(out + "/details.csv", csv.data(), csv.size());
      const LoopReport& L = res.report.loops.at(0);
      std::ofstream p(out + "/pattern.txt");
      p << "events " << n_events << "\nanalyze_s " << dt << "\npattern_length " << L.pattern_length
        << "\npattern_count " << L.pattern_count << "\nepsilon_used " << L.epsilon_used << "\nfirst_token "
        << L.first_occurrence_token << "\nk0_used " << L.k0_used << "\niterations_found " << L.iterations_found
        << "\nmain_stream " << res.report.main_stream << "\n";
      std::fprintf(stderr, "[ref_digest] analyze_trace %.1f s: pattern %lld x %lld\n", dt,
                   static_cast<long long>(L.pattern_length), static_cast<long long>(L.pattern_count));
    } else if (mode == "sa") {
      auto filtered = filter_majority_device(std::move(trace));
      const NormalizedTrace& working = filtered.trace;
      const auto streams = summarize_streams(working);
      const auto classes = classify_streams(streams);
      const uint32_t main = select_main_stream(classes, streams).stream;
      std::vector<int32_t> tokens;
      int32_t term = 0;
      {
        const auto seq = build_token_sequence(working, main);
        tokens = seq.tokens;
        term = static_cast<int32_t>(seq.names.size());  // TokenSequence::terminator() (streams.hpp:56)
      }
      filtered = {};  // release the records before the tree
      const uint64_t n = tokens.size();
      write_file(out + "/tokens.i32", tokens.data(), n * 4);
      std::vector<uint32_t> sa(n + 1), lcp(n + 1);
      const auto t1 = std::chrono::steady_clock::now();
      const int rc = ref_suffix_array(tokens.data(), n, term, sa.data(), lcp.data());
      if (rc) {
        std::fprintf(stderr, "ref_suffix_array failed (%d)\n", rc);
        return 1;
      }
      write_file(out + "/sa.u32", sa.data(), sa.size() * 4);
      write_file(out + "/lcp.u32", lcp.data(), lcp.size() * 4);
      std::ofstream p(out + "/sa.txt");
      p << "tokens " << n << "\nterminator " << term << "\nmain_stream " << main << "\ntree_s " << secs(t1) << "\n";
      std::fprintf(stderr, "[ref_digest] suffix tree + SA + LCP over %llu tokens in %.1f s\n",
                   static_cast<unsigned long long>(n), secs(t1));
    } else {
      std::fprintf(stderr, "unknown mode %s\n", mode.c_str());
      return 2;
    }
  } catch (const Error& e) {
    std::fprintf(stderr, "reference error: %s\n", e.what());
    return 3;
  }
  return 0;
}
