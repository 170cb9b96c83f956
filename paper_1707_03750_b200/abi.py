"""ctypes mirror of include/itertrace_cuda.h (the C-ABI of libitertrace_cuda.so).

Plain data only: struct layouts, status codes and a columnar ``Records`` holder that
produces an ``itt_records`` view over numpy arrays.  No compute lives here.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

ABI_VERSION = 2

# 1 + itertrace::ErrorKind (errors.hpp:8-21)
ERROR_KINDS = [
    "UnreadableFile", "MissingColumn", "TooManyBadRows", "EmptyTrace", "NoMainStream", "EmptyMainStream",
    "InvalidIterationCount", "NoPatternFound", "AmbiguousLoops", "NoIterations", "InvalidConfig", "IoError",
]
ITT_E_CUDA = 100
ITT_E_NCCL = 101
ITT_E_INVALID_ARGUMENT = 102

KIND_KERNEL = 0
KIND_NAMES = ["Kernel", "MemcpyHtoD", "MemcpyDtoH", "MemcpyDtoD", "Memset", "Other"]
CLASS_NAMES = ["Main", "CopyHtoD", "CopyDtoH", "CopyMixed", "Assist"]

REC_HAS_SIZE = 0x1
REC_HAS_THROUGHPUT = 0x2
MEM_HOST = 0
MEM_DEVICE = 1
MEM_HOST_STREAM_NAMES = 2  # host columns; names streamed through bounded device windows
MEM_DEVICE_HOST_NAMES = 3  # device columns; names streamed from (pinned) host memory
ORDER_UNKNOWN = 0
ORDER_SORTED = 1

P = C.POINTER


class itt_records(C.Structure):
    _fields_ = [
        ("n", C.c_uint64),
        ("start_ns", C.c_void_p),
        ("duration_ns", C.c_void_p),
        ("size_bytes", C.c_void_p),
        ("flags", C.c_void_p),
        ("stream", C.c_void_p),
        ("device", C.c_void_p),
        ("name_off", C.c_void_p),
        ("name_bytes", C.c_void_p),
        ("mem", C.c_int32),
        ("order", C.c_int32),
    ]


class itt_kernel_stat(C.Structure):
    _fields_ = [("name", C.c_char * 48), ("launches", C.c_uint64), ("total_ms", C.c_double), ("bytes", C.c_double)]


class itt_stream_summary(C.Structure):
    _fields_ = [
        ("stream", C.c_uint32),
        ("cls", C.c_int32),
        ("counts", C.c_int64 * 6),
        ("first_start", C.c_int64),
        ("last_end", C.c_int64),
    ]


class itt_census(C.Structure):
    _fields_ = [
        ("n_streams", C.c_uint32),
        ("streams", P(itt_stream_summary)),
        ("n_devices", C.c_uint32),
        ("majority_device", C.c_uint16),
        ("dropped_records", C.c_uint64),
        ("n_records", C.c_uint64),
    ]


class itt_tokens(C.Structure):
    _fields_ = [
        ("n", C.c_uint64),
        ("tokens", P(C.c_int32)),
        ("record_index", P(C.c_uint64)),
        ("n_names", C.c_uint32),
        ("name_row", P(C.c_uint64)),
    ]


class itt_repeat(C.Structure):
    _fields_ = [("start", C.c_int32), ("length", C.c_int32), ("count", C.c_int64)]


class itt_mining_cfg(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("epsilon0", C.c_int64), ("epsilon_cap", C.c_int64)]


class itt_pattern(C.Structure):
    _fields_ = [
        ("length", C.c_int64),
        ("tokens", P(C.c_int32)),
        ("count", C.c_int64),
        ("first_token", C.c_int64),
        ("epsilon_used", C.c_int64),
    ]


class itt_span(C.Structure):
    _fields_ = [("start_token", C.c_int64), ("end_token", C.c_int64), ("extra", C.c_int64)]


class itt_iter_row(C.Structure):
    _fields_ = [
        ("start_token", C.c_int64), ("end_token", C.c_int64), ("extra", C.c_int64),
        ("t_start", C.c_int64), ("t_end", C.c_int64),
        ("interval_ns", C.c_int64), ("copy_ns", C.c_int64), ("htod_bytes", C.c_int64),
        ("gap_sum", C.c_int64), ("gap_count", C.c_int64),
        ("has_interval", C.c_int32), ("pad_", C.c_int32),
    ]


class itt_clamps(C.Structure):
    _fields_ = [("negative_gap_clamps", C.c_int64), ("negative_interval_clamps", C.c_int64)]


# int (*)(void* user, const int32_t* tokens, uint64_t n, int32_t term, uint32_t cap, uint32_t* sa, uint32_t* lcp)
SA_PROVIDER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int32, C.c_uint32, C.c_void_p, C.c_void_p)


class itt_dsa_info(C.Structure):  # distributed suffix array (csrc/dist_driver.cu)
    _fields_ = [("rounds", C.c_int32), ("pad_", C.c_int32), ("groups", C.c_uint64), ("h_final", C.c_uint32),
                ("cap", C.c_uint32)]


class itt_summary(C.Structure):  # SummaryMetrics, metrics.hpp:33-42
    _fields_ = [
        ("avg_interval_ns", C.c_double),
        ("max_interval_ns", C.c_int64),
        ("avg_overlap", C.c_double),
        ("avg_operation_ns", C.c_double),
        ("avg_size_bytes", C.c_double),
        ("iterations_found", C.c_int64),
        ("iterations_declared", C.c_int64),
        ("insufficient_intervals", C.c_int32),
        ("pad_", C.c_int32),
    ]


class itt_analyze_opts(C.Structure):
    _fields_ = [
        ("loops", P(C.c_int64)),
        ("n_loops", C.c_uint32),
        ("epsilon0", C.c_int64),
        ("k0", C.c_int64),
        ("main_stream", C.c_int64),
        ("flags", C.c_uint32),
        ("sa_provider", SA_PROVIDER),
        ("sa_user", C.c_void_p),
    ]


ITT_ANALYZE_OP_PROFILE = 1
ITT_ANALYZE_OP_CELLS = 2
ITT_ANALYZE_BATCHED_SA = 4  # itt_batch_analyze: suffix arrays of the traces in flight built together
ITT_OP_PROFILE_AUTO, ITT_OP_PROFILE_SMEM, ITT_OP_PROFILE_SORT = 0, 1, 2


class itt_op_cell(C.Structure):
    """a12 (iteration, op) cell — include/itertrace_cuda.h itt_op_cell."""
    _fields_ = [
        ("iteration", C.c_uint32), ("op", C.c_int32), ("count", C.c_uint32), ("pad_", C.c_uint32),
        ("kernel_ns", C.c_int64), ("memcpy_ns", C.c_int64), ("idle_ns", C.c_int64),
    ]


class itt_op_total(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("count", C.c_int64), ("kernel_ns", C.c_int64), ("memcpy_ns", C.c_int64),
                ("idle_ns", C.c_int64)]


class itt_iter_op_total(C.Structure):
    _fields_ = [("distinct_ops", C.c_int64), ("kernel_ns", C.c_int64), ("memcpy_ns", C.c_int64), ("idle_ns", C.c_int64)]


# numpy views of the a12 structs
OP_CELL_DTYPE = np.dtype([("iteration", "<u4"), ("op", "<i4"), ("count", "<u4"), ("pad_", "<u4"),
                          ("kernel_ns", "<i8"), ("memcpy_ns", "<i8"), ("idle_ns", "<i8")])
OP_TOTAL_DTYPE = np.dtype([("iterations", "<i8"), ("count", "<i8"), ("kernel_ns", "<i8"), ("memcpy_ns", "<i8"),
                           ("idle_ns", "<i8")])
ITER_OP_TOTAL_DTYPE = np.dtype([("distinct_ops", "<i8"), ("kernel_ns", "<i8"), ("memcpy_ns", "<i8"), ("idle_ns", "<i8")])


class itt_loop_result(C.Structure):
    _fields_ = [
        ("iterations_declared", C.c_int64),
        ("pattern_length", C.c_int64),
        ("pattern_tokens", P(C.c_int32)),
        ("pattern_count", C.c_int64),
        ("epsilon_used", C.c_int64),
        ("first_token", C.c_int64),
        ("k0_used", C.c_int64),
        ("n_iterations", C.c_uint64),
        ("rows", P(itt_iter_row)),
        ("clamps", itt_clamps),
        ("op_totals", P(itt_op_total)),
        ("iter_op_totals", P(itt_iter_op_total)),
        ("n_op_cells", C.c_uint64),
        ("op_cells", P(itt_op_cell)),
    ]


class itt_parsed_trace(C.Structure):
    _fields_ = [
        ("records", itt_records),
        ("line", P(C.c_uint64)),
        ("n_device_labels", C.c_uint32),
        ("device_labels", P(C.c_char_p)),
        ("rows_total", C.c_uint64), ("rows_parsed", C.c_uint64), ("rows_skipped", C.c_uint64),
        ("n_skips", C.c_uint64),
        ("skip_line", P(C.c_uint64)),
        ("skip_reason", P(C.c_char_p)),
        ("column", C.c_int32 * 7),
        ("n_warnings", C.c_uint32),
        ("warnings", P(C.c_char_p)),
    ]


class itt_analysis(C.Structure):
    _fields_ = [
        ("census", itt_census),
        ("main_stream", C.c_uint32),
        ("n_main_streams", C.c_uint32),
        ("main_stream_override_non_main", C.c_int32),
        ("pad_", C.c_int32),
        ("n_tokens", C.c_uint64),
        ("n_names", C.c_uint32),
        ("name_row", P(C.c_uint64)),
        ("overlapping_kernels", C.c_int64),
        ("n_loops", C.c_uint32),
        ("loops", P(itt_loop_result)),
        ("owner", C.c_void_p),
    ]


# oracle/ref_api.h (test infrastructure structs; declared here so tests and bench share them)
class ref_iter(C.Structure):
    _fields_ = [
        ("index", C.c_int64), ("start_token", C.c_int64), ("end_token", C.c_int64), ("extra", C.c_int64),
        ("t_start", C.c_int64), ("t_end", C.c_int64), ("interval_ns", C.c_int64), ("htod_bytes", C.c_int64),
        ("has_interval", C.c_int32), ("has_overlap", C.c_int32),
        ("overlap_ratio", C.c_double), ("op_gap_mean_ns", C.c_double),
    ]


class ref_loop(C.Structure):
    _fields_ = [
        ("iterations_declared", C.c_int64), ("pattern_length", C.c_int64), ("pattern_count", C.c_int64),
        ("epsilon_used", C.c_int64), ("first_token", C.c_int64), ("k0_used", C.c_int64),
        ("pattern_tokens", P(C.c_int32)),
        ("n_iterations", C.c_uint64),
        ("iters", P(ref_iter)),
        ("avg_interval_ns", C.c_double), ("avg_overlap", C.c_double), ("avg_operation_ns", C.c_double),
        ("avg_size_bytes", C.c_double),
        ("max_interval_ns", C.c_int64),
        ("insufficient_intervals", C.c_int32), ("diagnosis", C.c_int32),
    ]


class ref_parsed(C.Structure):
    _fields_ = [
        ("status", C.c_int32), ("error", C.c_char_p), ("n", C.c_uint64),
        ("start_ns", P(C.c_int64)), ("duration_ns", P(C.c_int64)), ("size_bytes", P(C.c_int64)),
        ("flags", P(C.c_uint8)), ("stream", P(C.c_uint32)), ("row", P(C.c_uint64)),
        ("name_off", P(C.c_uint64)), ("name_bytes", P(C.c_uint8)),
        ("device_off", P(C.c_uint64)), ("device_bytes", P(C.c_uint8)),
        ("rows_total", C.c_uint64), ("rows_parsed", C.c_uint64), ("rows_skipped", C.c_uint64),
        ("n_skips", C.c_uint64), ("skip_line", P(C.c_uint64)), ("skip_reasons", C.c_char_p),
        ("column", C.c_int32 * 7), ("warnings", C.c_char_p),
    ]


class ref_stage_times(C.Structure):
    _fields_ = [(k, C.c_double) for k in
                ("order_ms", "filter_census_ms", "intern_ms", "mine_ms", "match_ms", "metrics_ms", "total_ms",
                 "analyze_ms")]


class ref_analysis(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("error", C.c_char_p),
        ("n_streams", C.c_uint32),
        ("streams", P(itt_stream_summary)),
        ("main_stream", C.c_uint32),
        ("n_tokens", C.c_uint64),
        ("n_names", C.c_uint32),
        ("n_loops", C.c_uint32),
        ("loops", P(ref_loop)),
        ("warnings", C.c_char_p),
        ("summary_json", C.c_char_p),
        ("details_csv", C.c_char_p),
        ("times", ref_stage_times),
    ]


def _ptr(a: np.ndarray | None) -> int | None:
    return None if a is None else a.ctypes.data


class Records:
    """Columnar trace records (host numpy arrays) — the itt_records of the C-ABI.

    Row i is TraceRecord i in source order.  ``names`` may be given as a list of str/bytes
    instead of (name_off, name_bytes).
    """

    def __init__(self, start_ns, duration_ns, stream, name_off=None, name_bytes=None, size_bytes=None, flags=None,
                 device=None, names=None, order=ORDER_UNKNOWN, keepalive=None):
        self.start_ns = np.ascontiguousarray(start_ns, dtype=np.int64)
        n = self.start_ns.shape[0]
        self.duration_ns = np.ascontiguousarray(duration_ns, dtype=np.int64)
        self.stream = np.ascontiguousarray(stream, dtype=np.uint32)
        self.size_bytes = (np.zeros(n, np.int64) if size_bytes is None
                           else np.ascontiguousarray(size_bytes, dtype=np.int64))
        self.flags = np.zeros(n, np.uint8) if flags is None else np.ascontiguousarray(flags, dtype=np.uint8)
        self.device = None if device is None else np.ascontiguousarray(device, dtype=np.uint16)
        if names is not None:
            bs = [s.encode() if isinstance(s, str) else bytes(s) for s in names]
            lens = np.fromiter((len(b) for b in bs), dtype=np.uint64, count=len(bs))
            self.name_off = np.zeros(n + 1, np.uint64)
            np.cumsum(lens, out=self.name_off[1:])
            self.name_bytes = np.frombuffer(b"".join(bs) or b"\0", dtype=np.uint8).copy()
        else:
            self.name_off = np.ascontiguousarray(name_off, dtype=np.uint64)
            self.name_bytes = np.ascontiguousarray(name_bytes, dtype=np.uint8)
        if self.name_bytes.size == 0:
            self.name_bytes = np.zeros(1, np.uint8)
        self.order = order
        self.mem = MEM_HOST  # or MEM_HOST_STREAM_NAMES (names streamed, not copied whole)
        self._keepalive = keepalive
        for a in (self.duration_ns, self.stream, self.size_bytes, self.flags):
            assert a.shape[0] == n
        assert self.name_off.shape[0] == n + 1

    @property
    def n(self) -> int:
        return int(self.start_ns.shape[0])

    def name(self, i: int) -> bytes:
        return self.name_bytes[int(self.name_off[i]):int(self.name_off[i + 1])].tobytes()

    def c(self) -> itt_records:
        return itt_records(self.n, _ptr(self.start_ns), _ptr(self.duration_ns), _ptr(self.size_bytes),
                           _ptr(self.flags), _ptr(self.stream), _ptr(self.device), _ptr(self.name_off),
                           _ptr(self.name_bytes), self.mem, self.order)

    def nbytes(self) -> int:
        tot = sum(a.nbytes for a in (self.start_ns, self.duration_ns, self.size_bytes, self.flags, self.stream,
                                     self.name_off, self.name_bytes))
        return tot + (self.device.nbytes if self.device is not None else 0)
