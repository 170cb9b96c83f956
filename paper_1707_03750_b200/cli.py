"""itertrace CLI mirror on the B200 path: `analyze` and `inspect` with the reference tool's options,
console text, output files and exit codes (tools/itertrace_main.cpp), the work on the GPU
(itt_parse_csv + itt_analyze).

    python -m paper_1707_03750_b200.cli analyze --trace t.csv --iterations 100 [--loops a,b]
        [--epsilon0 1] [--k0 K] [--theta-copy 0.1] [--theta-cpu 10] [--out-summary summary.json]
        [--out-details details.csv] [--main-stream S]
    python -m paper_1707_03750_b200.cli inspect --trace t.csv
    python -m paper_1707_03750_b200.cli --version

Exit codes (itertrace_main.cpp:23-42, 266-296): 0 ok; 2 NoPatternFound / AmbiguousLoops /
NoIterations; 3 unreadable or malformed trace; 4 invalid arguments / iteration count / config;
1 anything else (device errors included).  `synth` (the reference's generator, synth.hpp) is not
part of the mining path and is not mirrored.
"""
from __future__ import annotations

import argparse
import math
import os
import sys

from . import itertrace

EXIT_2 = {"NoPatternFound", "AmbiguousLoops", "NoIterations"}
EXIT_3 = {"UnreadableFile", "MissingColumn", "TooManyBadRows", "EmptyTrace", "NoMainStream", "EmptyMainStream", "IoError"}
EXIT_4 = {"InvalidIterationCount", "InvalidConfig"}


def exit_code_for(kind: str) -> int:  # itertrace_main.cpp:23-42
    if kind in EXIT_2:
        return 2
    if kind in EXIT_3:
        return 3
    if kind in EXIT_4:
        return 4
    return 1


def _llround(x: float) -> int:
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


def _use_color(out) -> bool:  # itertrace_main.cpp:44-46
    return out.isatty() and os.environ.get("NO_COLOR") is None


_DIAG_COLOR = {"COPY_BOUND": "\x1b[31m", "CPU_BOUND": "\x1b[31m", "NONE": "\x1b[32m", "INSUFFICIENT_DATA": "\x1b[33m"}


def console_summary(r: itertrace.AnalysisResult, rows: tuple, color: bool = False) -> str:
    """print_console_summary (itertrace_main.cpp:79-117); rows = (parsed, skipped, total)."""
    out = [f"{itertrace.TOOL} {itertrace.VERSION} — {r.trace_path}",
           "rows: %d parsed, %d skipped of %d" % rows, "streams:"]
    text = "\n".join(out) + "\n" + itertrace.stream_table(r.streams) + f"main stream: {r.main_stream}\n"
    for k, L in enumerate(r.loops):
        text += f"loop {k + 1}: declared {L.iterations_declared} iterations, found {L.iterations_found}\n"
        text += (f"  pattern: length {L.pattern_length}, repeats {L.pattern_count}, epsilon {L.epsilon_used}, "
                 f"k0 {L.k0_used}\n   ")
        show = L.pattern_names[:8]
        text += "".join(" " + n for n in show)
        if len(L.pattern_names) > len(show):
            text += f" ... (+{len(L.pattern_names) - len(show)} more)"
        text += "\n"
        m = L.summary
        text += (f"  avg interval {_llround(m.avg_interval_ns)} ns, max {m.max_interval_ns} ns, avg overlap "
                 f"{m.avg_overlap:.4f}, avg op gap {_llround(m.avg_operation_ns)} ns, avg htod "
                 f"{_llround(m.avg_size_bytes)} B/iter\n")
        code = L.diagnosis.code
        text += (f"  diagnosis: {_DIAG_COLOR.get(code, '') if color else ''}{code}{chr(27) + '[0m' if color else ''}"
                 f" — {L.diagnosis.message}\n")
        for line in L.diagnosis.evidence:
            text += f"    {line}\n"
    if not r.warnings:
        text += "warnings: none\n"
    else:
        text += "warnings:\n" + "".join(f"  - {w}\n" for w in r.warnings)
    return text


def loop_details_path(base: str, k: int) -> str:  # report.hpp:288-294
    if k == 0:
        return base
    d, name = os.path.split(base)
    stem, ext = os.path.splitext(name)
    if name.startswith(".") and ext == "":
        stem, ext = name, ""
    return os.path.join(d, f"{stem}.loop{k + 1}{ext}")


def _write(path: str, text: str):
    try:
        with open(path, "wb") as f:
            f.write(text.encode("utf-8", "surrogateescape"))
    except OSError:
        raise itertrace.AnalyzeError("IoError", f"report: cannot open '{path}' for writing")


def _read_trace(path: str) -> bytes:
    try:
        with open(path, "rb") as f:
            return f.read()
    except OSError:
        raise itertrace.AnalyzeError("UnreadableFile", f"ingest: cannot open trace file '{path}'")


def run_analyze(ctx, a) -> int:
    loops = ([a.iterations] if a.iterations is not None else []) + list(a.loops or [])
    text = _read_trace(a.trace)
    parsed = ctx.parse_csv(text, a.trace)
    try:
        cols = parsed.columns()
        off, nb = cols["name_off"], cols["name_bytes"].tobytes()
        names = itertrace._LazyNames(lambda r: nb[int(off[r]):int(off[r + 1])].decode("utf-8", "surrogateescape"))
        r = itertrace.analyze_trace(ctx, parsed, loops, epsilon0=a.epsilon0, k0=a.k0, theta_copy=a.theta_copy,
                                    theta_cpu=a.theta_cpu, main_stream=a.main_stream, trace_label=a.trace,
                                    device_labels=parsed.device_labels, names=names, trace_warnings=parsed.warnings)
        rows = (parsed.rows_parsed, parsed.rows_skipped, parsed.rows_total)
    finally:
        parsed.free()
    _write(a.out_summary, r.summary_json())
    for k in range(len(r.loops)):
        _write(loop_details_path(a.out_details, k), r.details_csv(k))
    sys.stdout.write(console_summary(r, rows, _use_color(sys.stdout)))
    sys.stdout.write(f"summary written: {a.out_summary}\ndetails written: {a.out_details}\n")
    sys.stdout.flush()
    return 0


def run_inspect(ctx, trace: str) -> int:
    sys.stdout.write(itertrace.inspect_csv(ctx, _read_trace(trace), trace))
    sys.stdout.flush()
    return 0


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # CLI11 parse errors exit 4 (itertrace_main.cpp:266-271)
        self.print_usage(sys.stderr)
        sys.stderr.write(f"error: {message}\n")
        raise SystemExit(4)


def _int_list(s: str) -> list:
    try:
        return [int(x) for x in s.split(",") if x != ""]
    except ValueError:
        raise argparse.ArgumentTypeError(f"invalid loop list '{s}'")


def main(argv=None) -> int:
    p = _Parser(prog=itertrace.TOOL, description="iteration-level GPU trace analysis (B200 path)")
    p.add_argument("--version", action="version", version=itertrace.VERSION)
    sub = p.add_subparsers(dest="cmd", parser_class=_Parser)
    an = sub.add_parser("analyze", help="recover iterations and metrics from a trace")
    an.add_argument("--trace", required=True)
    an.add_argument("--iterations", type=int)
    an.add_argument("--loops", type=_int_list)
    an.add_argument("--epsilon0", type=int, default=1)
    an.add_argument("--k0", type=int)
    an.add_argument("--theta-copy", type=float, default=0.10)
    an.add_argument("--theta-cpu", type=float, default=10.0)
    an.add_argument("--out-summary", default="summary.json")
    an.add_argument("--out-details", default="details.csv")
    an.add_argument("--main-stream", type=int)
    ins = sub.add_parser("inspect", help="print the per-stream operation census")
    ins.add_argument("--trace", required=True)
    a = p.parse_args(argv)
    if a.cmd is None:  # require_subcommand(1)
        p.error("a subcommand is required")
    if a.cmd == "analyze":
        if a.iterations is None and not a.loops:
            sys.stderr.write("error: analyze needs --iterations or --loops\n")
            return 4
        if a.iterations is not None and a.loops:
            sys.stderr.write("error: give either --iterations or --loops, not both\n")
            return 4
        if a.out_summary == a.out_details:
            sys.stderr.write("error: --out-summary and --out-details must differ\n")
            return 4
    from .cuda import Context, IttError
    try:
        ctx = Context(0)
        try:
            return run_analyze(ctx, a) if a.cmd == "analyze" else run_inspect(ctx, a.trace)
        finally:
            ctx.close()
    except itertrace.AnalyzeError as e:
        sys.stderr.write(f"error: {e}\n")
        return exit_code_for(e.kind)
    except IttError as e:
        sys.stderr.write(f"error: {e}\n")
        return exit_code_for(e.kind)
    except Exception as e:  # noqa: BLE001 (itertrace_main.cpp:294-296)
        sys.stderr.write(f"error: {e}\n")
        return 1


if __name__ == "__main__":
    sys.exit(main())
