// itertrace_cli.cpp — the reference tool's command line (tools/itertrace_main.cpp) on the B200 path.
//
// Same subcommands, options, defaults, console text, output files and exit codes as the
// reference CLI (itertrace_main.cpp:23-299), with its CLI11 front end replaced by a small parser
// of our own (CLI11 is not vendored by the reference) and the work moved to the GPU:
//   analyze  parse_trace + analyze_trace       -> itertrace::cuda::analyze_csv_file (itt_parse_csv +
//            itt_analyze); report rendering is the reference's own render_report
//   inspect  parse_trace + summarize_streams   -> itertrace::cuda::inspect_csv_file
//   synth    the reference's generator (synth.hpp, host only; not on the mining path)
// Exit codes: 0 ok; 2 NoPatternFound / AmbiguousLoops / NoIterations; 3 unreadable or malformed
// input and I/O errors; 4 usage errors and InvalidIterationCount / InvalidConfig; 1 anything else
// (device errors included).  `--config FILE` (analyze, synth) reads `name = value` lines (TOML
// style: '#' comments, quoted strings, [a, b] lists, an optional [analyze] / [synth] section);
// options given on the command line win over the file.
//
// Built against the reference headers (they define the types the drop-in keeps), so it is
// compiled where /root/reference exists and the binary travels prebuilt (build.py).
#include <cerrno>
#include <cstdarg>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <limits>
#include <iostream>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include <unistd.h>

#include "itertrace/itertrace.hpp"
#include "itertrace_cuda.hpp"

namespace {

using namespace itertrace;

// ---------------------------------------------------------------- exit codes (itertrace_main.cpp:23-42)
int code_of(ErrorKind k) {
  switch (k) {
    case ErrorKind::NoPatternFound:
    case ErrorKind::AmbiguousLoops:
    case ErrorKind::NoIterations:
      return 2;
    case ErrorKind::InvalidIterationCount:
    case ErrorKind::InvalidConfig:
      return 4;
    case ErrorKind::UnreadableFile:
    case ErrorKind::MissingColumn:
    case ErrorKind::TooManyBadRows:
    case ErrorKind::EmptyTrace:
    case ErrorKind::NoMainStream:
    case ErrorKind::EmptyMainStream:
    case ErrorKind::IoError:
      return 3;
  }
  return 1;
}

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------- option table
struct Opt {
  std::string name;  // long name without dashes
  std::string help;
  std::string def;   // default shown in --help ("" = none)
  bool required = false;
  bool list = false;  // comma-delimited / repeated values
  std::function<void(const std::string&)> set;
  bool seen = false;
};

bool parse_i64(const std::string& s, int64_t& v) {
  if (s.empty()) return false;
  errno = 0;
  char* end = nullptr;
  const long long x = std::strtoll(s.c_str(), &end, 10);
  if (errno || *end) return false;
  v = x;
  return true;
}

bool parse_f64(const std::string& s, double& v) {
  if (s.empty()) return false;
  errno = 0;
  char* end = nullptr;
  const double x = std::strtod(s.c_str(), &end);
  if (errno || *end) return false;
  v = x;
  return true;
}

std::string lower(std::string s) {
  for (auto& ch : s) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
  return s;
}

template <typename T>
std::function<void(const std::string&)> int_into(T& dst, const std::string& name) {
  return [&dst, name](const std::string& s) {
    int64_t v = 0;
    if (!parse_i64(s, v) || v < static_cast<int64_t>(std::numeric_limits<T>::min()) ||
        static_cast<uint64_t>(v) > static_cast<uint64_t>(std::numeric_limits<T>::max()))
      throw UsageError("--" + name + ": " + s + " is not a valid integer");
    dst = static_cast<T>(v);
  };
}
template <typename T>
std::function<void(const std::string&)> opt_int_into(std::optional<T>& dst, const std::string& name) {
  return [&dst, name](const std::string& s) {
    T v{};
    int_into(v, name)(s);
    dst = v;
  };
}
std::function<void(const std::string&)> f64_into(double& dst, const std::string& name) {
  return [&dst, name](const std::string& s) {
    if (!parse_f64(s, dst)) throw UsageError("--" + name + ": " + s + " is not a valid number");
  };
}
std::function<void(const std::string&)> str_into(std::string& dst) {
  return [&dst](const std::string& s) { dst = s; };
}

class Command {
 public:
  Command(std::string name, std::string about) : name_(std::move(name)), about_(std::move(about)) {}
  Opt& add(const std::string& name, const std::string& help, std::function<void(const std::string&)> set,
           const std::string& def = "") {
    opts_.push_back(Opt{name, help, def, false, false, std::move(set)});
    return opts_.back();
  }
  void allow_config() { config_ = true; }
  const std::string& name() const { return name_; }
  const std::string& about() const { return about_; }

  // argv after the subcommand name; returns false when --help was printed
  bool parse(const std::vector<std::string>& args) {
    std::string config_path;
    for (size_t i = 0; i < args.size(); ++i) {
      const std::string& a = args[i];
      if (a == "--help" || a == "-h") {
        print_help(std::cout);
        return false;
      }
      if (a.rfind("--", 0) != 0) throw UsageError("The following argument was not expected: " + a);
      std::string key = a.substr(2), val;
      bool inline_val = false;
      if (const auto eq = key.find('='); eq != std::string::npos) {
        val = key.substr(eq + 1);
        key = key.substr(0, eq);
        inline_val = true;
      }
      if (config_ && key == "config") {
        if (!inline_val) {
          if (i + 1 >= args.size()) throw UsageError("--config: 1 required argument missing");
          val = args[++i];
        }
        config_path = val;
        continue;
      }
      Opt* o = find(key);
      if (!o) throw UsageError("The following argument was not expected: " + a);
      std::vector<std::string> vals;
      if (inline_val) {
        vals.push_back(val);
      } else {
        if (i + 1 >= args.size() || is_flag(args[i + 1])) throw UsageError("--" + key + ": 1 required argument missing");
        vals.push_back(args[++i]);
        while (o->list && i + 1 < args.size() && !is_flag(args[i + 1])) vals.push_back(args[++i]);  // --loops 10 20
      }
      if (o->seen && !o->list) throw UsageError("--" + key + ": option given more than once");
      apply(*o, vals);
    }
    if (!config_path.empty()) read_config(config_path);
    for (const Opt& o : opts_)
      if (o.required && !o.seen) throw UsageError("--" + o.name + " is required");
    return true;
  }

  void print_help(std::ostream& os) const {
    os << about_ << "\nUsage: itertrace " << name_ << " [OPTIONS]\n\nOptions:\n";
    os << "  -h,--help                   print this help message and exit\n";
    if (config_) os << "  --config FILE               read options from a TOML-style file\n";
    for (const Opt& o : opts_) {
      std::string lhs = "  --" + o.name + (o.list ? " INT,..." : " VALUE");
      if (lhs.size() < 30) lhs.resize(30, ' ');
      os << lhs << o.help;
      if (!o.def.empty()) os << " [" << o.def << "]";
      if (o.required) os << " REQUIRED";
      os << "\n";
    }
  }

 private:
  static bool is_flag(const std::string& s) { return s.size() > 1 && s[0] == '-' && !std::isdigit(static_cast<unsigned char>(s[1])); }
  Opt* find(const std::string& key) {
    std::string k = key;
    for (auto& ch : k)
      if (ch == '_') ch = '-';
    for (Opt& o : opts_)
      if (o.name == k) return &o;
    return nullptr;
  }
  static void apply(Opt& o, const std::vector<std::string>& vals) {
    for (const std::string& v : vals) {
      if (o.list) {
        size_t p = 0;
        while (p <= v.size()) {
          const size_t q = v.find(',', p);
          const std::string part = v.substr(p, q == std::string::npos ? std::string::npos : q - p);
          if (!part.empty()) o.set(part);
          if (q == std::string::npos) break;
          p = q + 1;
        }
      } else {
        o.set(v);
      }
    }
    o.seen = true;
  }
  static std::string trim(const std::string& s) {
    const auto b = s.find_first_not_of(" \t\r");
    if (b == std::string::npos) return "";
    return s.substr(b, s.find_last_not_of(" \t\r") - b + 1);
  }
  static std::string unquote(const std::string& s) {
    if (s.size() >= 2 && ((s.front() == '"' && s.back() == '"') || (s.front() == '\'' && s.back() == '\'')))
      return s.substr(1, s.size() - 2);
    return s;
  }
  void read_config(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw UsageError("--config: file not found: " + path);
    std::string line, section;
    while (std::getline(in, line)) {
      line = trim(line);
      if (line.empty() || line[0] == '#' || line[0] == ';') continue;
      if (line.front() == '[' && line.back() == ']') {
        section = trim(line.substr(1, line.size() - 2));
        continue;
      }
      const auto eq = line.find('=');
      if (eq == std::string::npos) throw UsageError("--config: cannot parse line: " + line);
      std::string key = trim(line.substr(0, eq)), val = trim(line.substr(eq + 1));
      if (const auto dot = key.find('.'); dot != std::string::npos) {  // analyze.iterations = ...
        section = key.substr(0, dot);
        key = key.substr(dot + 1);
      }
      if (!section.empty() && section != name_) continue;
      Opt* o = find(key);
      if (!o) throw UsageError("--config: the option " + key + " is not known to " + name_);
      if (o->seen) continue;  // the command line wins
      std::vector<std::string> vals;
      if (val.size() >= 2 && val.front() == '[' && val.back() == ']') {
        std::stringstream ss(val.substr(1, val.size() - 2));
        std::string item;
        while (std::getline(ss, item, ',')) vals.push_back(unquote(trim(item)));
      } else {
        vals.push_back(unquote(val));
      }
      apply(*o, vals);
    }
  }

  std::string name_, about_;
  std::vector<Opt> opts_;
  bool config_ = false;
};

// ---------------------------------------------------------------- console text (itertrace_main.cpp:61-117)
std::string fmt(const char* f, ...) __attribute__((format(printf, 1, 2)));
std::string fmt(const char* f, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, f);
  std::vsnprintf(buf, sizeof(buf), f, ap);
  va_end(ap);
  return buf;
}

void stream_table(std::ostream& os, const std::vector<StreamSummary>& streams,
                  const std::map<std::uint32_t, StreamClass>& classes) {
  os << fmt("  %7s%11s%9s%7s%7s%7s%8s%7s%15s%15s\n", "stream", "class", "kernel", "htod", "dtoh", "dtod", "memset",
            "other", "first_ns", "last_ns");
  for (const StreamSummary& s : streams) {
    const auto c = classes.find(s.stream);
    const std::string cls = c == classes.end() ? "Assist" : to_string(c->second);
    os << fmt("  %7u%11s%9lld%7lld%7lld%7lld%8lld%7lld%15lld%15lld\n", s.stream, cls.c_str(),
              static_cast<long long>(s.count(OpKind::Kernel)), static_cast<long long>(s.count(OpKind::MemcpyHtoD)),
              static_cast<long long>(s.count(OpKind::MemcpyDtoH)), static_cast<long long>(s.count(OpKind::MemcpyDtoD)),
              static_cast<long long>(s.count(OpKind::Memset)), static_cast<long long>(s.count(OpKind::Other)),
              static_cast<long long>(s.first_start), static_cast<long long>(s.last_end));
  }
}

const char* color_of(DiagnosisCode c) {
  if (c == DiagnosisCode::NONE) return "\x1b[32m";
  if (c == DiagnosisCode::INSUFFICIENT_DATA) return "\x1b[33m";
  return "\x1b[31m";  // COPY_BOUND, CPU_BOUND
}

void console_summary(std::ostream& os, const Report& r, const IngestReport& ing) {
  const bool color = ::isatty(::fileno(stdout)) != 0 && std::getenv("NO_COLOR") == nullptr;
  os << r.tool << " " << r.version << " — " << r.trace_path << "\n";
  os << "rows: " << ing.rows_parsed << " parsed, " << ing.rows_skipped << " skipped of " << ing.rows_total << "\n";
  os << "streams:\n";
  stream_table(os, r.streams, r.classes);
  os << "main stream: " << r.main_stream << "\n";
  int k = 0;
  for (const LoopReport& L : r.loops) {
    os << "loop " << ++k << ": declared " << L.iterations_declared << " iterations, found " << L.iterations_found << "\n";
    os << "  pattern: length " << L.pattern_length << ", repeats " << L.pattern_count << ", epsilon " << L.epsilon_used
       << ", k0 " << L.k0_used << "\n   ";
    const size_t shown = std::min<size_t>(8, L.pattern_names.size());
    for (size_t j = 0; j < shown; ++j) os << " " << L.pattern_names[j];
    if (L.pattern_names.size() > shown) os << " ... (+" << L.pattern_names.size() - shown << " more)";
    os << "\n";
    const SummaryMetrics& m = L.summary;
    os << "  avg interval " << std::llround(m.avg_interval_ns) << " ns, max " << m.max_interval_ns << " ns, avg overlap "
       << fmt("%.4f", m.avg_overlap) << ", avg op gap " << std::llround(m.avg_operation_ns) << " ns, avg htod "
       << std::llround(m.avg_size_bytes) << " B/iter\n";
    os << "  diagnosis: " << (color ? color_of(L.diagnosis.code) : "") << to_string(L.diagnosis.code)
       << (color ? "\x1b[0m" : "") << " — " << L.diagnosis.message << "\n";
    for (const std::string& e : L.diagnosis.evidence) os << "    " << e << "\n";
  }
  if (r.warnings.empty()) {
    os << "warnings: none\n";
  } else {
    os << "warnings:\n";
    for (const std::string& w : r.warnings) os << "  - " << w << "\n";
  }
}

// ---------------------------------------------------------------- subcommands
struct AnalyzeArgs {
  std::string trace;
  std::optional<int64_t> iterations;
  std::vector<int64_t> loops;
  int64_t epsilon0 = 1;
  std::optional<int64_t> k0;
  double theta_copy = 0.10, theta_cpu = 10.0;
  std::string out_summary = "summary.json", out_details = "details.csv";
  std::optional<uint32_t> main_stream;
};

int do_analyze(const AnalyzeArgs& a) {
  if (!a.iterations && a.loops.empty()) {
    std::cerr << "error: analyze needs --iterations or --loops\n";
    return 4;
  }
  if (a.iterations && !a.loops.empty()) {
    std::cerr << "error: give either --iterations or --loops, not both\n";
    return 4;
  }
  if (a.out_summary == a.out_details) {
    std::cerr << "error: --out-summary and --out-details must differ\n";
    return 4;
  }
  AnalyzeOptions opt;
  if (a.iterations) opt.loops.push_back(*a.iterations);
  opt.loops.insert(opt.loops.end(), a.loops.begin(), a.loops.end());
  opt.epsilon0 = a.epsilon0;
  opt.k0 = a.k0;
  opt.theta_copy = a.theta_copy;
  opt.theta_cpu = a.theta_cpu;
  opt.main_stream = a.main_stream;
  auto [result, ingest] = itertrace::cuda::analyze_csv_file(a.trace, opt);
  render_report(result.report, result.details, a.out_summary, a.out_details);
  console_summary(std::cout, result.report, ingest);
  std::cout << "summary written: " << a.out_summary << "\ndetails written: " << a.out_details << "\n";
  return 0;
}

int do_inspect(const std::string& trace) {
  const auto r = itertrace::cuda::inspect_csv_file(trace);
  std::cout << "trace: " << trace << "\nrows: " << r.ingest.rows_parsed << " parsed, " << r.ingest.rows_skipped
            << " skipped of " << r.ingest.rows_total << "\n";
  stream_table(std::cout, r.streams, r.classes);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  std::vector<std::string> args(argv + 1, argv + argc);
  const std::string about = std::string(kToolName) +
                            " — iteration-level GPU trace analysis (B200 path)\n"
                            "exit codes: 0 success, 2 no pattern found, 3 unreadable or malformed trace, 4 invalid arguments";

  AnalyzeArgs an;
  Command analyze("analyze", "recover iterations and metrics from a trace");
  analyze.allow_config();
  analyze.add("trace", "GPU trace CSV", str_into(an.trace)).required = true;
  analyze.add("iterations", "declared iteration count of the training loop", opt_int_into(an.iterations, "iterations"));
  analyze.add("loops", "comma-separated iteration counts for multi-loop applications",
              [&an](const std::string& s) {
                int64_t v = 0;
                if (!parse_i64(s, v)) throw UsageError("--loops: " + s + " is not a valid integer");
                an.loops.push_back(v);
              }).list = true;
  analyze.add("epsilon0", "starting repetition slack (doubles on failed searches)", int_into(an.epsilon0, "epsilon0"), "1");
  analyze.add("k0", "unmatched-token budget per occurrence (default: pattern length / 4, rounded up)",
              opt_int_into(an.k0, "k0"));
  analyze.add("theta-copy", "avg-overlap threshold for the copy-bound diagnosis", f64_into(an.theta_copy, "theta-copy"),
              "0.1");
  analyze.add("theta-cpu", "interval/op-gap ratio threshold for the cpu-bound diagnosis",
              f64_into(an.theta_cpu, "theta-cpu"), "10");
  analyze.add("out-summary", "summary JSON path", str_into(an.out_summary), "summary.json");
  analyze.add("out-details", "per-iteration CSV path", str_into(an.out_details), "details.csv");
  analyze.add("main-stream", "analyze this stream id instead of auto-selecting", opt_int_into(an.main_stream, "main-stream"));

  std::string inspect_trace;
  Command inspect("inspect", "print the per-stream operation census");
  inspect.add("trace", "GPU trace CSV", str_into(inspect_trace)).required = true;

  SynthConfig sc;
  std::string out_trace = "synthetic_trace.csv", out_truth = "synthetic_truth.json";
  Command synth("synth", "generate a labeled synthetic trace (the reference's generator, synth.hpp)");
  synth.allow_config();
  synth.add("out-trace", "output trace CSV", str_into(out_trace), out_trace);
  synth.add("out-truth", "output ground-truth JSON", str_into(out_truth), out_truth);
  synth.add("seed", "RNG seed", int_into(sc.seed, "seed"), std::to_string(sc.seed));
  synth.add("init-ops", "operations before the first iteration", int_into(sc.init_ops, "init-ops"), std::to_string(sc.init_ops));
  synth.add("pattern-len", "operations per iteration body", int_into(sc.pattern_len, "pattern-len"),
            std::to_string(sc.pattern_len));
  synth.add("iterations", "planted iteration count", int_into(sc.iterations, "iterations"), std::to_string(sc.iterations));
  synth.add("vocab-size", "distinct operation names", int_into(sc.vocab_size, "vocab-size"), std::to_string(sc.vocab_size));
  synth.add("insert-prob", "per-iteration probability of extra ops", f64_into(sc.insert_prob, "insert-prob"),
            fmt("%g", sc.insert_prob));
  synth.add("max-inserts", "max extra ops per iteration", int_into(sc.max_inserts, "max-inserts"),
            std::to_string(sc.max_inserts));
  synth.add("insert-placement", "where extra ops go: after_pattern or inside_pattern", [&sc](const std::string& s) {
    const std::string v = lower(s);
    if (v == "after_pattern") sc.insert_placement = InsertPlacement::after_pattern;
    else if (v == "inside_pattern") sc.insert_placement = InsertPlacement::inside_pattern;
    else throw UsageError("--insert-placement: " + s + " not in {after_pattern, inside_pattern}");
  });
  synth.add("kernel-duration-ns", "base kernel duration", int_into(sc.kernel_duration_ns, "kernel-duration-ns"),
            std::to_string(sc.kernel_duration_ns));
  synth.add("kernel-jitter-ns", "kernel duration jitter", int_into(sc.kernel_jitter_ns, "kernel-jitter-ns"),
            std::to_string(sc.kernel_jitter_ns));
  synth.add("intra-gap-ns", "gap between ops inside an iteration", int_into(sc.intra_gap_ns, "intra-gap-ns"),
            std::to_string(sc.intra_gap_ns));
  synth.add("interval-gap-ns", "gap between iterations", int_into(sc.interval_gap_ns, "interval-gap-ns"),
            std::to_string(sc.interval_gap_ns));
  synth.add("interval-jitter-ns", "iteration gap jitter", int_into(sc.interval_jitter_ns, "interval-jitter-ns"),
            std::to_string(sc.interval_jitter_ns));
  synth.add("htod-bytes", "copied bytes per iteration", int_into(sc.htod_bytes_per_iter, "htod-bytes"),
            std::to_string(sc.htod_bytes_per_iter));
  synth.add("htod-bandwidth", "copy bandwidth, bytes/s", int_into(sc.htod_bandwidth_bps, "htod-bandwidth"),
            std::to_string(sc.htod_bandwidth_bps));
  synth.add("pathology", "planted bottleneck: none, graph_growth or oversize_copy", [&sc](const std::string& s) {
    const std::string v = lower(s);
    if (v == "none") sc.pathology = Pathology::none;
    else if (v == "graph_growth") sc.pathology = Pathology::graph_growth;
    else if (v == "oversize_copy") sc.pathology = Pathology::oversize_copy;
    else throw UsageError("--pathology: " + s + " not in {none, graph_growth, oversize_copy}");
  });
  synth.add("pathology-factor", "pathology scale factor", f64_into(sc.pathology_factor, "pathology-factor"),
            fmt("%g", sc.pathology_factor));

  Command* cmds[] = {&analyze, &inspect, &synth};
  auto top_help = [&](std::ostream& os) {
    os << about << "\nUsage: itertrace [OPTIONS] SUBCOMMAND\n\nOptions:\n  -h,--help    print this help message and exit\n"
       << "  --version    display program version information and exit\n\nSubcommands:\n";
    for (const Command* c : cmds) os << "  " << c->name() << std::string(10 - c->name().size(), ' ') << c->about() << "\n";
  };
  Command* cmd = nullptr;
  try {  // usage errors exit 4, help 0 (itertrace_main.cpp:266-271)
    if (args.empty()) throw UsageError("A subcommand is required");
    if (args[0] == "--version") {
      std::cout << kToolVersion << "\n";
      return 0;
    }
    if (args[0] == "--help" || args[0] == "-h") {
      top_help(std::cout);
      return 0;
    }
    for (Command* c : cmds)
      if (args[0] == c->name()) cmd = c;
    if (!cmd) throw UsageError("The following argument was not expected: " + args[0]);
    if (!cmd->parse(std::vector<std::string>(args.begin() + 1, args.end()))) return 0;
  } catch (const UsageError& e) {
    std::cerr << e.what() << "\nRun with --help for more information.\n";
    return 4;
  }
  try {
    if (cmd == &analyze) return do_analyze(an);
    if (cmd == &inspect) return do_inspect(inspect_trace);
    generate_trace(sc, out_trace, out_truth);
    std::cout << "trace written: " << out_trace << "\ntruth written: " << out_truth << "\n";
    return 0;
  } catch (const Error& e) {
    std::cerr << "error: " << e.what() << "\n";
    return code_of(e.kind());
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
