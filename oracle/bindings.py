"""ctypes bindings for the CPU checkers (TEST INFRASTRUCTURE ONLY).

* ``Ref``    — oracle/_ref/libitertrace_ref.so: the unmodified reference headers compiled
               in place (oracle/Makefile).  Parity oracle + CPU baseline.
* ``Oracle`` — oracle/libitt_oracle.so: the C restatement (itt_oracle.c), pinned against
               ``Ref`` and the reference's known-answer tests.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_1707_03750_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
P = C.POINTER


class CheckerError(Exception):
    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status
        self.kind = abi.ERROR_KINDS[status - 1] if 1 <= status <= 12 else f"status{status}"


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


class _Common:
    prefix = ""

    def __init__(self, path):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        self.lib = C.CDLL(path)
        p = self.prefix
        L = self.lib
        getattr(L, p + "suffix_array").argtypes = [P(C.c_int32), C.c_uint64, C.c_int32, P(C.c_uint32), P(C.c_uint32)]
        getattr(L, p + "enumerate_repeats").argtypes = [P(C.c_int32), C.c_uint64, C.c_int32, C.c_int64, C.c_int64,
                                                        P(P(abi.itt_repeat)), P(C.c_uint64)]
        getattr(L, p + "mine_patterns").argtypes = [P(C.c_int32), C.c_uint64, C.c_uint32, P(abi.itt_mining_cfg),
                                                    C.c_uint32, C.c_int, P(abi.itt_pattern), C.c_char_p, C.c_uint64]
        getattr(L, p + "approx_match").argtypes = [P(C.c_int32), C.c_uint64, P(C.c_int32), C.c_uint64, C.c_int64,
                                                   P(P(abi.itt_span)), P(C.c_uint64)]
        getattr(L, p + "build_token_sequence").argtypes = [P(abi.itt_records), C.c_uint32, P(C.c_int32),
                                                           P(C.c_uint64), P(C.c_uint64), P(C.c_uint32), P(C.c_uint64)]
        getattr(L, p + "iteration_metrics").argtypes = [P(abi.itt_records), C.c_uint32, P(abi.itt_span), C.c_uint64,
                                                        P(abi.ref_iter), P(abi.itt_clamps)]
        getattr(L, p + "summarize_streams").argtypes = [P(abi.itt_records), C.c_int, P(abi.itt_stream_summary),
                                                        C.c_uint32, P(C.c_uint32), P(C.c_uint64)]
        self._free = getattr(L, p + "free")
        self._free.argtypes = [C.c_void_p]

    def _f(self, name):
        return getattr(self.lib, self.prefix + name)

    def suffix_array(self, tokens, term):
        t = _i32(tokens)
        n = t.shape[0]
        sa = np.zeros(n + 1, np.uint32)
        lcp = np.zeros(n + 1, np.uint32)
        rc = self._f("suffix_array")(t.ctypes.data_as(P(C.c_int32)), n, term, sa.ctypes.data_as(P(C.c_uint32)),
                                     lcp.ctypes.data_as(P(C.c_uint32)))
        if rc:
            raise CheckerError(rc, "suffix_array failed")
        return sa, lcp

    def enumerate_repeats(self, tokens, term, min_count, max_len):
        t = _i32(tokens)
        out = P(abi.itt_repeat)()
        cnt = C.c_uint64()
        self._f("enumerate_repeats")(t.ctypes.data_as(P(C.c_int32)), t.shape[0], term, min_count, max_len,
                                     C.byref(out), C.byref(cnt))
        res = [(out[i].start, out[i].length, out[i].count) for i in range(cnt.value)]
        self._free(out)
        return res

    def mine_patterns(self, tokens, n_names, loops, multi=False):
        """loops: list of (iterations, epsilon0) or (iterations, epsilon0, cap)."""
        t = _i32(tokens)
        cfgs = (abi.itt_mining_cfg * max(1, len(loops)))()
        for i, lp in enumerate(loops):
            cfgs[i].iterations = lp[0]
            cfgs[i].epsilon0 = lp[1] if len(lp) > 1 else 1
            cfgs[i].epsilon_cap = lp[2] if len(lp) > 2 else 0
        out = (abi.itt_pattern * max(1, len(loops)))()
        err = C.create_string_buffer(1024)
        rc = self._f("mine_patterns")(t.ctypes.data_as(P(C.c_int32)), t.shape[0], n_names, cfgs, len(loops),
                                      1 if multi else 0, out, err, 1024)
        if rc:
            raise CheckerError(rc, err.value.decode())
        res = []
        for i in range(len(loops) if multi else 1):
            p = out[i]
            res.append(dict(tokens=[p.tokens[j] for j in range(p.length)], count=p.count,
                            first_token=p.first_token, epsilon_used=p.epsilon_used))
            self._free(p.tokens)
        return res

    def approx_match(self, tokens, pattern, k0):
        t = _i32(tokens)
        p = _i32(pattern)
        out = P(abi.itt_span)()
        cnt = C.c_uint64()
        self._f("approx_match")(t.ctypes.data_as(P(C.c_int32)), t.shape[0], p.ctypes.data_as(P(C.c_int32)),
                                p.shape[0], k0, C.byref(out), C.byref(cnt))
        res = np.array([(out[i].start_token, out[i].end_token, out[i].extra) for i in range(cnt.value)],
                       dtype=np.int64).reshape(-1, 3)
        self._free(out)
        return res

    def build_token_sequence(self, recs: abi.Records, main_stream):
        c = recs.c()
        tok = np.zeros(max(1, recs.n), np.int32)
        ri = np.zeros(max(1, recs.n), np.uint64)
        names = np.zeros(max(1, recs.n), np.uint64)
        n = C.c_uint64()
        v = C.c_uint32()
        rc = self._f("build_token_sequence")(C.byref(c), main_stream, tok.ctypes.data_as(P(C.c_int32)),
                                             ri.ctypes.data_as(P(C.c_uint64)), C.byref(n), C.byref(v),
                                             names.ctypes.data_as(P(C.c_uint64)))
        if rc:
            raise CheckerError(rc, "build_token_sequence")
        return tok[:n.value].copy(), ri[:n.value].copy(), names[:v.value].copy()

    def iteration_metrics(self, recs: abi.Records, main_stream, spans):
        sp = (abi.itt_span * max(1, len(spans)))()
        for i, s in enumerate(spans):
            sp[i].start_token, sp[i].end_token, sp[i].extra = int(s[0]), int(s[1]), int(s[2])
        rows = (abi.ref_iter * max(1, len(spans)))()
        cl = abi.itt_clamps()
        c = recs.c()
        rc = self._f("iteration_metrics")(C.byref(c), main_stream, sp, len(spans), rows, C.byref(cl))
        if rc:
            raise CheckerError(rc, "iteration_metrics")
        return [rows[i] for i in range(len(spans))], (cl.negative_gap_clamps, cl.negative_interval_clamps)

    def summarize_streams(self, recs: abi.Records, filter_device=False):
        out = (abi.itt_stream_summary * 4096)()
        n = C.c_uint32()
        dropped = C.c_uint64()
        c = recs.c()
        rc = self._f("summarize_streams")(C.byref(c), 1 if filter_device else 0, out, 4096, C.byref(n),
                                          C.byref(dropped))
        if rc:
            raise CheckerError(rc, "summarize_streams")
        return [summary_tuple(out[i]) for i in range(n.value)], dropped.value


def summary_tuple(s):
    return (s.stream, s.cls, tuple(s.counts[k] for k in range(6)), s.first_start, s.last_end)


class Ref(_Common):
    prefix = "ref_"

    def __init__(self):
        super().__init__(os.path.join(HERE, "_ref", "libitertrace_ref.so"))
        L = self.lib
        L.ref_parse_csv.argtypes = [C.c_char_p, C.c_uint64, C.c_char_p, P(abi.ref_parsed)]
        L.ref_free_parsed.argtypes = [P(abi.ref_parsed)]
        L.ref_synth_csv.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_int64, C.c_int32,
                                    C.c_int32, P(C.c_uint64)]
        L.ref_synth_csv.restype = C.c_void_p
        L.ref_analyze_csv.argtypes = [C.c_char_p, C.c_uint64, C.c_char_p, P(abi.itt_analyze_opts), P(abi.ref_analysis)]
        self.lib.ref_analyze.argtypes = [P(abi.itt_records), P(abi.itt_analyze_opts), C.c_int, P(abi.ref_analysis)]
        self.lib.ref_free_analysis.argtypes = [P(abi.ref_analysis)]

    def parse_csv(self, text: bytes, label: str = "trace.csv") -> dict:
        """parse_trace_text (ingest.hpp:154-402), the reference itself."""
        return _ref_parse(self.lib, text, label)

    def synth_csv(self, seed=42, pattern_len=6, iterations=40, vocab_size=16, insert_prob=0.0, max_inserts=0,
                  inside_pattern=False, pathology=0) -> bytes:
        """The reference generator's CSV (synth.hpp:187)."""
        n = C.c_uint64()
        p = self.lib.ref_synth_csv(seed, pattern_len, iterations, vocab_size, insert_prob, max_inserts,
                                   1 if inside_pattern else 0, pathology, C.byref(n))
        if not p:
            raise ValueError("reference generator rejected the config")
        try:
            return C.string_at(p, n.value)
        finally:
            self._free(p)

    def analyze_csv(self, text: bytes, loops, label="trace.csv", epsilon0=1, k0=-1, main_stream=-1) -> dict:
        """parse_trace_text + analyze_trace: summary JSON / details CSV as the reference CLI writes them."""
        lp = (C.c_int64 * max(1, len(loops)))(*loops)
        opts = abi.itt_analyze_opts(lp, len(loops), epsilon0, k0, main_stream, 0)
        out = abi.ref_analysis()
        rc = self.lib.ref_analyze_csv(text, len(text), label.encode(), C.byref(opts), C.byref(out))
        try:
            if rc:
                return {"status": rc, "error": out.error.decode("utf-8", "surrogateescape")}
            return {"status": 0, "summary_json": out.summary_json.decode(), "details_csv": out.details_csv.decode(),
                    "warnings": out.warnings.decode().split("\n") if out.warnings else []}
        finally:
            self.lib.ref_free_analysis(C.byref(out))

    def analyze(self, recs: abi.Records, loops, epsilon0=1, k0=-1, main_stream=-1, staged=False):
        lp = (C.c_int64 * max(1, len(loops)))(*loops)
        opts = abi.itt_analyze_opts(lp, len(loops), epsilon0, k0, main_stream)
        out = abi.ref_analysis()
        c = recs.c()
        self.lib.ref_analyze(C.byref(c), C.byref(opts), 1 if staged else 0, C.byref(out))
        try:
            if out.status:
                raise CheckerError(out.status, (out.error or b"").decode())
            res = dict(
                streams=[summary_tuple(out.streams[i]) for i in range(out.n_streams)],
                main_stream=out.main_stream,
                warnings=(out.warnings or b"").decode().split("\n") if out.warnings else [],
                summary_json=(out.summary_json or b"").decode(),
                details_csv=(out.details_csv or b"").decode(),
                times={k: getattr(out.times, k) for k, _ in abi.ref_stage_times._fields_},
                loops=[],
            )
            for k in range(out.n_loops):
                lo = out.loops[k]
                res["loops"].append(dict(
                    iterations_declared=lo.iterations_declared, pattern_length=lo.pattern_length,
                    pattern_count=lo.pattern_count, epsilon_used=lo.epsilon_used, first_token=lo.first_token,
                    k0_used=lo.k0_used,
                    iters=[tuple(getattr(lo.iters[i], f) for f, _ in abi.ref_iter._fields_)
                           for i in range(lo.n_iterations)],
                    avg_interval_ns=lo.avg_interval_ns, avg_overlap=lo.avg_overlap,
                    avg_operation_ns=lo.avg_operation_ns, avg_size_bytes=lo.avg_size_bytes,
                    max_interval_ns=lo.max_interval_ns, insufficient_intervals=bool(lo.insufficient_intervals),
                    diagnosis=lo.diagnosis))
            return res
        finally:
            self.lib.ref_free_analysis(C.byref(out))


def _ref_parse(lib, text: bytes, label: str) -> dict:
    out = abi.ref_parsed()
    rc = lib.ref_parse_csv(text, len(text), label.encode(), C.byref(out))
    try:
        if rc:
            return {"status": rc, "error": out.error.decode("utf-8", "surrogateescape")}
        n = out.n

        def arr(ptr, dt, cnt):
            return np.ctypeslib.as_array(ptr, shape=(cnt,)).astype(dt, copy=True) if cnt else np.zeros(0, dt)
        name_off = arr(out.name_off, np.uint64, n + 1)
        dev_off = arr(out.device_off, np.uint64, n + 1)
        names = bytes(arr(out.name_bytes, np.uint8, int(name_off[-1]))) if n else b""
        devs = bytes(arr(out.device_bytes, np.uint8, int(dev_off[-1]))) if n else b""
        cols = ("Start", "Duration", "Size", "Throughput", "Device", "Stream", "Name")
        return {
            "status": 0, "n": n,
            "start_ns": arr(out.start_ns, np.int64, n), "duration_ns": arr(out.duration_ns, np.int64, n),
            "size_bytes": arr(out.size_bytes, np.int64, n), "flags": arr(out.flags, np.uint8, n),
            "stream": arr(out.stream, np.uint32, n), "row": arr(out.row, np.uint64, n),
            "names": [names[name_off[i]:name_off[i + 1]] for i in range(n)],
            "devices": [devs[dev_off[i]:dev_off[i + 1]].decode("utf-8", "surrogateescape") for i in range(n)],
            "rows_total": out.rows_total, "rows_parsed": out.rows_parsed, "rows_skipped": out.rows_skipped,
            "skips": list(zip([int(x) for x in arr(out.skip_line, np.uint64, out.n_skips)],
                              out.skip_reasons.decode("utf-8", "surrogateescape").split("\n") if out.n_skips else [])),
            "column": {cols[i]: int(out.column[i]) for i in range(7) if out.column[i] >= 0},
            "warnings": out.warnings.decode("utf-8", "surrogateescape").split("\n") if out.warnings else [],
        }
    finally:
        lib.ref_free_parsed(C.byref(out))


class Oracle(_Common):
    prefix = "orc_"

    def __init__(self):
        super().__init__(os.path.join(HERE, "libitt_oracle.so"))
        self.lib.orc_sort_records.argtypes = [C.c_uint64, P(C.c_int64), P(C.c_uint64)]
        self.lib.orc_classify.argtypes = [C.c_char_p, C.c_uint64, C.c_int]
        self.lib.orc_op_profile.argtypes = [P(C.c_int32), P(C.c_int64), P(C.c_int64), P(C.c_uint8), C.c_uint64,
                                            C.c_uint32, P(abi.itt_span), C.c_uint64, P(P(abi.itt_op_cell)),
                                            P(C.c_uint64)]

    def sort_records(self, start):
        s = np.ascontiguousarray(start, dtype=np.int64)
        perm = np.zeros(max(1, s.shape[0]), np.uint64)
        self.lib.orc_sort_records(s.shape[0], s.ctypes.data_as(P(C.c_int64)), perm.ctypes.data_as(P(C.c_uint64)))
        return perm[:s.shape[0]]

    def classify(self, name: bytes, has_tp: bool) -> int:
        return self.lib.orc_classify(name, len(name), 1 if has_tp else 0)

    def op_profile(self, tokens, tok_start, tok_end, tok_kind, n_ops, spans):
        """a12 cells (abi.OP_CELL_DTYPE) by the plain-loop restatement in itt_oracle.c."""
        t = _i32(tokens)
        ts = np.ascontiguousarray(tok_start, dtype=np.int64)
        te = np.ascontiguousarray(tok_end, dtype=np.int64)
        tk = np.ascontiguousarray(tok_kind, dtype=np.uint8)
        sp = (abi.itt_span * max(1, len(spans)))()
        for i, s in enumerate(spans):
            sp[i].start_token, sp[i].end_token, sp[i].extra = int(s[0]), int(s[1]), int(s[2])
        out = P(abi.itt_op_cell)()
        cnt = C.c_uint64()
        rc = self.lib.orc_op_profile(t.ctypes.data_as(P(C.c_int32)), ts.ctypes.data_as(P(C.c_int64)),
                                     te.ctypes.data_as(P(C.c_int64)), tk.ctypes.data_as(P(C.c_uint8)), t.shape[0],
                                     n_ops, sp, len(spans), C.byref(out), C.byref(cnt))
        if rc:
            raise CheckerError(rc, "op_profile")
        n = cnt.value
        res = np.zeros(n, abi.OP_CELL_DTYPE)
        if n:
            C.memmove(res.ctypes.data, out, n * C.sizeof(abi.itt_op_cell))
        self._free(out)
        return res


_ref = None
_orc = None


def ref() -> Ref:
    global _ref
    if _ref is None:
        _ref = Ref()
    return _ref


def oracle() -> Oracle:
    global _orc
    if _orc is None:
        _orc = Oracle()
    return _orc
