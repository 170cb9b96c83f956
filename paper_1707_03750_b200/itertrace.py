"""Host-side mirror of the reference's analyze_trace (pipeline.hpp:34-134) over the C-ABI.

The device (``itt_analyze``) does every O(n) stage and returns integer per-iteration rows;
this module finishes what the reference does on the host, in the reference's order, so the
doubles are bit-identical:
  * IterationMetrics doubles: overlap = copy / interval (metrics.hpp:131-135),
    op_gap_mean = gap_sum / gap_count (metrics.hpp:158-160);
  * compute_summary ordered sums (metrics.hpp:166-202), diagnose (report.hpp:61-90);
  * warnings text and order (pipeline.hpp:51-52, 62-67, 72, 76-79, 117-125);
  * rendering: summary_to_json(...).dump(2) (report.hpp:121-185, 304) and details_to_csv
    (report.hpp:191-220), byte for byte.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

from . import abi
from .jsonfloat import dump_float
from .cuda import Context, IttError

TOOL = "itertrace"
VERSION = "0.1.0"  # version.hpp:5-6
DIAG = ["COPY_BOUND", "CPU_BOUND", "NONE", "INSUFFICIENT_DATA"]  # report.hpp:24
DETAILS_HEADER = ("iteration,token_start,token_end,t_start_ns,t_end_ns,interval_ns,overlap_ratio,"
                  "htod_bytes,op_gap_mean_ns,extra_ops")


@dataclass
class IterationMetrics:  # metrics.hpp:21-31
    index: int
    start_token: int
    end_token: int
    t_start: int
    t_end: int
    interval_ns: Optional[int]
    overlap_ratio: Optional[float]
    htod_bytes: int
    op_gap_mean_ns: float
    extra_ops: int


@dataclass
class SummaryMetrics:  # metrics.hpp:33-42
    avg_interval_ns: float = 0.0
    max_interval_ns: int = 0
    avg_overlap: float = 0.0
    avg_operation_ns: float = 0.0
    avg_size_bytes: float = 0.0
    iterations_found: int = 0
    iterations_declared: int = 0
    insufficient_intervals: bool = False


@dataclass
class Diagnosis:  # report.hpp:36-40
    code: str = "NONE"
    evidence: list = field(default_factory=list)
    message: str = ""


@dataclass
class LoopReport:  # report.hpp:92-103
    iterations_declared: int
    pattern_names: list
    pattern_tokens: list
    pattern_length: int
    pattern_count: int
    epsilon_used: int
    first_occurrence_token: int
    k0_used: int
    iterations_found: int
    summary: SummaryMetrics
    diagnosis: Diagnosis


@dataclass
class AnalysisResult:  # pipeline.hpp:27-30 (+ the rendered outputs)
    trace_path: str
    epsilon0: int
    theta_copy: float
    theta_cpu: float
    k0_override: Optional[int]
    main_stream_override: Optional[int]
    streams: list
    main_stream: int
    loops: list
    details: list
    warnings: list
    op_profiles: list = field(default_factory=list)  # a12, one OpProfile per loop when requested

    def summary_json(self) -> str:
        return render_summary(self)

    def details_csv(self, k: int = 0) -> str:
        if isinstance(self.details, LazyDetails):
            return self.details.csv(k)
        return details_to_csv(self.details[k])


class LazyDetails:
    """Per-loop IterationMetrics over the device's integer rows, built only when indexed; the CSV
    is rendered natively from the rows (itt_render_details_csv) — at C5's 500K iterations an
    interpreted finish would cost seconds."""

    def __init__(self, ctx: Context, rows: list):
        self._ctx = ctx
        self._rows = rows
        self._items = [None] * len(rows)

    def __len__(self):
        return len(self._rows)

    def __getitem__(self, k):
        if self._items[k] is None:
            self._items[k] = rows_to_metrics(self._rows[k])
        return self._items[k]

    def __iter__(self):
        return (self[k] for k in range(len(self)))

    def rows(self, k):
        return self._rows[k]

    def csv(self, k):
        return self._ctx.render_details_csv(self._rows[k])


class AnalyzeError(Exception):
    def __init__(self, kind: str, message: str):
        super().__init__(message)
        self.kind = kind


def fmt6(v: float) -> str:  # detail::format_double, report.hpp:49-53
    return "%.6f" % v


def compute_summary(items: list, iterations_declared: int) -> SummaryMetrics:
    """compute_summary, metrics.hpp:166-202 (same accumulation order)."""
    if not items:
        raise AnalyzeError("NoIterations", "metrics: no iterations to summarize")
    s = SummaryMetrics(iterations_found=len(items), iterations_declared=iterations_declared)
    isum = icnt = ocnt = btot = 0
    osum = 0.0
    gsum = 0.0
    for m in items:
        if m.interval_ns is not None:
            isum += m.interval_ns
            icnt += 1
            s.max_interval_ns = max(s.max_interval_ns, m.interval_ns)
        if m.overlap_ratio is not None:
            osum += m.overlap_ratio
            ocnt += 1
        gsum += m.op_gap_mean_ns
        btot += m.htod_bytes
    if icnt > 0:
        s.avg_interval_ns = float(isum) / float(icnt)
    else:
        s.insufficient_intervals = True
    if ocnt > 0:
        s.avg_overlap = osum / float(ocnt)
    s.avg_operation_ns = gsum / float(len(items))
    s.avg_size_bytes = float(btot) / float(len(items))
    return s


def diagnose(s: SummaryMetrics, theta_copy: float = 0.10, theta_cpu: float = 10.0) -> Diagnosis:
    """diagnose, report.hpp:61-90."""
    d = Diagnosis()
    if s.iterations_found < 2 or s.insufficient_intervals:
        d.code = "INSUFFICIENT_DATA"
        d.message = ("fewer than two recovered iterations; interval metrics are undefined, rerun with a longer trace "
                     "or check the declared iteration count")
        return d
    if s.avg_overlap >= theta_copy:
        d.code = "COPY_BOUND"
        d.evidence = ["avg_overlap=" + fmt6(s.avg_overlap) + " >= theta_copy=" + fmt6(theta_copy),
                      "avg_interval_ns=" + fmt6(s.avg_interval_ns)]
        d.message = ("host-to-device copies occupy a large share of the gap between iterations; data transfer is the "
                     "likely bottleneck. A smaller batch reduces per-step copy volume, at the cost of more steps; weigh "
                     "that against what the algorithm needs per batch.")
        return d
    if s.avg_interval_ns > 0 and s.avg_interval_ns >= theta_cpu * s.avg_operation_ns:
        d.code = "CPU_BOUND"
        d.evidence = ["avg_interval_ns=" + fmt6(s.avg_interval_ns) + " >= theta_cpu=" + fmt6(theta_cpu) +
                      " * avg_operation_ns=" + fmt6(s.avg_operation_ns),
                      "avg_overlap=" + fmt6(s.avg_overlap) + " below theta_copy=" + fmt6(theta_copy)]
        d.message = ("iteration gaps dwarf the in-iteration dispatch cadence while copy activity is low; host-side "
                     "work between steps is the likely bottleneck. Inspect the training loop for per-step work such as "
                     "operations that keep growing or re-initializing the computation graph.")
        return d
    d.code = "NONE"
    d.message = "no bottleneck indicated by the interval and copy-overlap heuristics"
    return d


def rows_to_metrics(rows) -> list:
    """itt_iter_row integers -> IterationMetrics with the reference's two divisions."""
    out = []
    for k, r in enumerate(rows):
        start, end, extra, t0, t1, interval, copy, htod, gsum, gcnt, has_int = (int(x) for x in r[:11])
        has_int = has_int & 0xFFFFFFFF
        iv = interval if has_int else None
        ov = (float(copy) / float(interval)) if (has_int and interval > 0) else None
        gap = float(gsum) / float(gcnt) if gcnt > 0 else 0.0
        out.append(IterationMetrics(k + 1, start, end, t0, t1, iv, ov, htod, gap, extra))
    return out


def analyze_trace(ctx: Context, recs, loops: list, epsilon0: int = 1, k0: Optional[int] = None,
                  theta_copy: float = 0.10, theta_cpu: float = 10.0, main_stream: Optional[int] = None,
                  trace_label: str = "trace.csv", device_labels=None, names=None,
                  op_profile=False, trace_warnings=(), sa_provider=None) -> AnalysisResult:
    """analyze_trace (pipeline.hpp:34-134): device pipeline + host finish in reference order.
    op_profile=True adds the a12 second-level per-op profile of every loop ("cells": with the
    (iteration, op) grid); no reference counterpart, and the reference's own outputs are unchanged.
    sa_provider: build the suffix array elsewhere (dist_sa.DistributedSAProvider: over G GPUs)."""
    try:
        raw = ctx.analyze_raw(recs, list(loops), epsilon0, -1 if k0 is None else k0,
                              -1 if main_stream is None else main_stream, op_profile=op_profile,
                              sa_provider=sa_provider)
    except IttError as e:
        raise AnalyzeError(e.kind, str(e)) from e
    label = (lambda d: device_labels[d]) if device_labels is not None else (lambda d: "dev%05u" % d)
    warnings = list(trace_warnings)  # the trace's own (ingest) warnings come first (pipeline.hpp:51)
    if raw["n_devices"] > 1:  # streams.hpp:198-203
        warnings.append("MultiDeviceTrace: kept majority device '%s', dropped %d records from other devices"
                        % (label(raw["majority_device"]), raw["dropped"]))
    if main_stream is not None:
        if raw["override_non_main"]:
            warnings.append("MainStreamOverride: stream %d carries no kernels but was selected by override" % main_stream)
    elif raw["n_main_streams"] > 1:  # streams.hpp:130-143
        others = ", ".join(str(s[0]) for s in raw["streams"] if s[1] == 0 and s[0] != raw["main_stream"])
        warnings.append("MultipleMainStreams: analyzing stream %d (most kernels); other kernel-bearing streams: %s"
                        % (raw["main_stream"], others))
    if raw["overlapping_kernels"] > 0:
        warnings.append("OverlappingKernels: %d consecutive main-stream records report overlapping intervals "
                        "(timer granularity)" % raw["overlapping_kernels"])
    name_of = None
    if isinstance(names, _LazyNames):
        name_of = names.bind(raw["name_row"])
    elif names is not None:
        name_of = names
    elif hasattr(recs, "name"):
        name_of = [recs.name(r).decode("utf-8", "surrogateescape") for r in raw["name_row"]]
    loop_reports, rows = [], []
    for k, L in enumerate(raw["loops"]):
        ng, ni = L["clamps"]
        if ng > 0:
            warnings.append("NegativeGaps: %d negative dispatch gaps clamped to zero" % ng)
        if ni > 0:
            warnings.append("NegativeIntervals: %d negative iteration intervals clamped to zero" % ni)
        try:  # compute_summary natively, same accumulation order (report.cu)
            n = ctx.compute_summary(L["rows"], loops[k])
        except IttError as e:
            raise AnalyzeError(e.kind, str(e)) from e
        summ = SummaryMetrics(n.avg_interval_ns, n.max_interval_ns, n.avg_overlap, n.avg_operation_ns,
                              n.avg_size_bytes, n.iterations_found, n.iterations_declared,
                              bool(n.insufficient_intervals))
        pnames = [name_of[t] for t in L["pattern_tokens"]] if name_of is not None else [str(t) for t in L["pattern_tokens"]]
        loop_reports.append(LoopReport(loops[k], pnames, L["pattern_tokens"], L["pattern_length"], L["pattern_count"],
                                       L["epsilon_used"], L["first_token"], L["k0_used"], len(L["rows"]), summ,
                                       diagnose(summ, theta_copy, theta_cpu)))
        rows.append(L["rows"])
    details = LazyDetails(ctx, rows)
    profiles = [OpProfile(L["op_cells"], L["op_totals"], L["iter_op_totals"], name_of) for L in raw["loops"]] \
        if op_profile else []
    return AnalysisResult(trace_label, epsilon0, theta_copy, theta_cpu, k0, main_stream, raw["streams"],
                          raw["main_stream"], loop_reports, details, warnings, profiles)


def analyze_csv(ctx: Context, text: bytes, loops: list, trace_label: str = "trace.csv", **kw) -> AnalysisResult:
    """parse_trace_text + analyze_trace (what the reference CLI's `analyze` runs, itertrace_main.cpp:143),
    both on the GPU: the CSV is parsed by itt_parse_csv and stays in HBM for itt_analyze."""
    try:
        parsed = ctx.parse_csv(text, trace_label)
    except IttError as e:
        raise AnalyzeError(e.kind, str(e)) from e
    names = None
    if kw.get("names") is None:
        cols = parsed.columns()
        off, nb = cols["name_off"], cols["name_bytes"].tobytes()
        names_all = lambda r: nb[int(off[r]):int(off[r + 1])].decode("utf-8", "surrogateescape")  # noqa: E731
        names = _LazyNames(names_all)
    try:
        return analyze_trace(ctx, parsed, loops, trace_label=trace_label, device_labels=parsed.device_labels,
                             trace_warnings=parsed.warnings, names=names, **kw)
    finally:
        parsed.free()


class _LazyNames:
    """token id -> name, resolved through name_row on first use (analyze_trace indexes by token id)."""

    def __init__(self, by_row):
        self.by_row = by_row
        self.rows = None

    def bind(self, name_row):
        self.rows = name_row
        return self

    def __getitem__(self, t):
        return self.by_row(self.rows[t])


# ---------------------------------------------------------------- a12 second-level profile
@dataclass
class OpProfile:
    """Per-op x per-iteration profile (definition in itertrace_cuda.h).
    per_op: abi.OP_TOTAL_DTYPE indexed by op id; per_iteration: abi.ITER_OP_TOTAL_DTYPE;
    cells: abi.OP_CELL_DTYPE (empty unless the cell grid was requested)."""
    cells: object
    per_op: object
    per_iteration: object
    names: Optional[list] = None

    def per_op_csv(self) -> str:
        return op_profile_csv(self)


def reduce_cells(cells, n_ops: int, n_iterations: int):
    """The two reductions of a cell grid (exact int64 sums) -> (per_op, per_iteration)."""
    import numpy as np
    per_op = np.zeros(n_ops, abi.OP_TOTAL_DTYPE)
    per_it = np.zeros(n_iterations, abi.ITER_OP_TOTAL_DTYPE)
    if len(cells):
        op = cells["op"].astype(np.int64)
        it = cells["iteration"].astype(np.int64)
        per_op["iterations"] = np.bincount(op, minlength=n_ops)
        per_it["distinct_ops"] = np.bincount(it, minlength=n_iterations)
        for col in ("count", "kernel_ns", "memcpy_ns", "idle_ns"):
            a = np.zeros(n_ops, np.int64)
            np.add.at(a, op, cells[col].astype(np.int64))
            per_op[col] = a
            if col != "count":
                b = np.zeros(n_iterations, np.int64)
                np.add.at(b, it, cells[col].astype(np.int64))
                per_it[col] = b
    return per_op, per_it


def op_profile_csv(p: OpProfile) -> str:
    """Per-op table of the second-level profile: ops occurring in some iteration, by op id."""
    lines = ["op,name,iterations,count,kernel_ns,memcpy_ns,idle_ns,mean_kernel_ns,mean_memcpy_ns,mean_idle_ns"]
    for v, r in enumerate(p.per_op):
        c = int(r["count"])
        if c == 0:
            continue
        nm = p.names[v] if p.names is not None else str(v)
        if any(ch in nm for ch in ',"\n'):
            nm = '"' + nm.replace('"', '""') + '"'
        lines.append("%d,%s,%d,%d,%d,%d,%d,%s,%s,%s" % (
            v, nm, int(r["iterations"]), c, int(r["kernel_ns"]), int(r["memcpy_ns"]), int(r["idle_ns"]),
            fmt6(int(r["kernel_ns"]) / c), fmt6(int(r["memcpy_ns"]) / c), fmt6(int(r["idle_ns"]) / c)))
    return "\n".join(lines) + "\n"


# ---------------------------------------------------------------- rendering (report.hpp)
def _json_str(s: str) -> str:
    out = ['"']
    for ch in s:
        o = ord(ch)
        if ch == '"':
            out.append('\\"')
        elif ch == "\\":
            out.append("\\\\")
        elif ch == "\b":
            out.append("\\b")
        elif ch == "\f":
            out.append("\\f")
        elif ch == "\n":
            out.append("\\n")
        elif ch == "\r":
            out.append("\\r")
        elif ch == "\t":
            out.append("\\t")
        elif o < 0x20:
            out.append("\\u%04x" % o)
        else:
            out.append(ch)
    out.append('"')
    return "".join(out)


def _json_float(v: float) -> str:
    """nlohmann::json number_float dump (Grisu2 digits + %g-like layout): jsonfloat.dump_float."""
    return dump_float(v)


def _dump(v, indent: int, level: int) -> str:
    pad = " " * (indent * (level + 1))
    end = " " * (indent * level)
    if v is None:
        return "null"
    if v is True:
        return "true"
    if v is False:
        return "false"
    if isinstance(v, int):
        return str(v)
    if isinstance(v, float):
        return _json_float(v)
    if isinstance(v, str):
        return _json_str(v)
    if isinstance(v, list):
        if not v:
            return "[]"
        return "[\n" + ",\n".join(pad + _dump(x, indent, level + 1) for x in v) + "\n" + end + "]"
    if isinstance(v, dict):
        if not v:
            return "{}"
        return "{\n" + ",\n".join(pad + _json_str(k) + ": " + _dump(x, indent, level + 1) for k, x in v.items()) + \
            "\n" + end + "}"
    raise TypeError(type(v))


def summary_object(r: AnalysisResult) -> dict:
    """summary_to_json, report.hpp:121-185 (key order preserved)."""
    streams = []
    for (sid, cls, counts, first, last) in r.streams:
        streams.append({"stream": sid, "class": abi.CLASS_NAMES[cls], "kernel": counts[0], "memcpy_htod": counts[1],
                        "memcpy_dtoh": counts[2], "memcpy_dtod": counts[3], "memset": counts[4], "other": counts[5],
                        "first_start_ns": first, "last_end_ns": last})
    loops = []
    for L in r.loops:
        s = L.summary
        loops.append({
            "iterations_declared": L.iterations_declared, "pattern": list(L.pattern_names),
            "pattern_length": L.pattern_length, "pattern_count": L.pattern_count, "epsilon_used": L.epsilon_used,
            "first_occurrence_token": L.first_occurrence_token, "k0": L.k0_used, "iterations_found": L.iterations_found,
            "metrics": {"avg_interval_ns": float(s.avg_interval_ns), "max_interval_ns": s.max_interval_ns,
                        "avg_overlap": float(s.avg_overlap), "avg_operation_ns": float(s.avg_operation_ns),
                        "avg_size_bytes": float(s.avg_size_bytes), "insufficient_intervals": s.insufficient_intervals},
            "diagnosis": {"code": L.diagnosis.code, "evidence": list(L.diagnosis.evidence),
                          "message": L.diagnosis.message}})
    return {"tool": TOOL, "version": VERSION, "trace": r.trace_path,
            "config": {"epsilon0": r.epsilon0, "theta_copy": float(r.theta_copy), "theta_cpu": float(r.theta_cpu),
                       "k0_override": r.k0_override, "main_stream_override": r.main_stream_override},
            "streams": streams, "main_stream": r.main_stream, "loops": loops, "warnings": list(r.warnings)}


def render_summary(r: AnalysisResult) -> str:
    return _dump(summary_object(r), 2, 0) + "\n"


def details_to_csv(items: list) -> str:
    """details_to_csv, report.hpp:191-220."""
    out = [DETAILS_HEADER]
    for m in items:
        cells = [str(m.index), str(m.start_token), str(m.end_token), str(m.t_start), str(m.t_end),
                 "" if m.interval_ns is None else str(m.interval_ns),
                 "" if m.overlap_ratio is None else fmt6(m.overlap_ratio), str(m.htod_bytes),
                 str(_llround(m.op_gap_mean_ns)), str(m.extra_ops)]
        out.append(",".join(cells))
    return "\n".join(out) + "\n"


def _llround(x: float) -> int:  # std::llround: half away from zero
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


def stream_table(streams) -> str:
    """print_stream_table (itertrace_main.cpp:61-77): the per-stream census as the CLI prints it
    (std::setw columns, right-aligned).  streams: (stream, class, counts[6], first, last)."""
    out = ["  %7s%11s%9s%7s%7s%7s%8s%7s%15s%15s" % ("stream", "class", "kernel", "htod", "dtoh", "dtod", "memset",
                                                    "other", "first_ns", "last_ns")]
    for stream, cls, c, first, last in streams:
        name = abi.CLASS_NAMES[cls] if 0 <= cls < len(abi.CLASS_NAMES) else "Assist"
        out.append("  %7d%11s%9d%7d%7d%7d%8d%7d%15d%15d" % (stream, name, c[0], c[1], c[2], c[3], c[4], c[5], first, last))
    return "\n".join(out) + "\n"


def inspect_csv(ctx: Context, text: bytes, trace_path: str = "trace.csv") -> str:
    """The CLI's `inspect` (run_inspect, itertrace_main.cpp:151-160) on the GPU: parse_trace_text
    (itt_parse_csv) + summarize_streams / classify_streams over the whole trace (no device
    filter, as there) on the device; returns the exact stdout text."""
    try:
        parsed = ctx.parse_csv(text, trace_path)
    except IttError as e:
        raise AnalyzeError(e.kind, str(e)) from e
    try:
        streams, _ = ctx.summarize_streams(parsed, filter_device=False)
        return ("trace: %s\nrows: %d parsed, %d skipped of %d\n" % (trace_path, parsed.rows_parsed, parsed.rows_skipped,
                                                                    parsed.rows_total)) + stream_table(streams)
    finally:
        parsed.free()
