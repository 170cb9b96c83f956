"""ctypes binding of libitertrace_cuda.so (include/itertrace_cuda.h).

There is no CPU fallback: loading fails loudly when the in-tree library is missing, and
creating a context fails without an sm_100 device.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import abi

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libitertrace_cuda.so")
P = C.POINTER
_lib = None


class IttError(Exception):
    """A failed C-ABI call.  ``kind`` is the reference ErrorKind name for statuses 1..12."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status
        self.kind = abi.ERROR_KINDS[status - 1] if 1 <= status <= 12 else {
            abi.ITT_E_CUDA: "Cuda", abi.ITT_E_NCCL: "Nccl", abi.ITT_E_INVALID_ARGUMENT: "InvalidArgument"}.get(
                status, f"status{status}")


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is not built; run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    sig = {
        "itt_abi_version": ([], C.c_int),
        "itt_ctx_create": ([C.c_int, P(vp)], C.c_int),
        "itt_ctx_destroy": ([vp], C.c_int),
        "itt_last_error": ([vp], C.c_char_p),
        "itt_free": ([vp, vp], C.c_int),
        "itt_ctx_set_profiling": ([vp, C.c_int], C.c_int),
        "itt_ctx_reset_stats": ([vp], C.c_int),
        "itt_ctx_kernel_stats": ([vp, P(abi.itt_kernel_stat), C.c_uint32, P(C.c_uint32)], C.c_int),
        "itt_ctx_launch_count": ([vp, P(C.c_uint64)], C.c_int),
        "itt_batch_create": ([C.c_int, C.c_uint32, P(vp)], C.c_int),
        "itt_batch_destroy": ([vp], C.c_int),
        "itt_batch_analyze": ([vp, vp, C.c_uint64, vp, C.c_int, P(P(abi.itt_analysis)), P(C.c_int)], C.c_int),
        "itt_batch_error": ([vp, C.c_uint64], C.c_char_p),
        "itt_batch_launch_count": ([vp, P(C.c_uint64)], C.c_int),
        "itt_batch_free": ([vp, P(P(abi.itt_analysis)), C.c_uint64], C.c_int),
        "itt_parse_csv": ([vp, C.c_char_p, C.c_uint64, C.c_char_p, P(P(abi.itt_parsed_trace))], C.c_int),
        "itt_free_parsed": ([vp, P(abi.itt_parsed_trace)], C.c_int),
        "itt_ctx_mem_stats": ([vp, P(C.c_uint64), P(C.c_uint64), C.c_int], C.c_int),
        "itt_device_alloc": ([vp, C.c_uint64, P(vp)], C.c_int),
        "itt_device_free": ([vp, vp], C.c_int),
        "itt_memcpy_h2d": ([vp, vp, vp, C.c_uint64], C.c_int),
        "itt_memcpy_d2h": ([vp, vp, vp, C.c_uint64], C.c_int),
        "itt_memcpy": ([vp, vp, vp, C.c_uint64], C.c_int),
        "itt_compute_summary": ([vp, vp, C.c_uint64, C.c_int64, P(abi.itt_summary)], C.c_int),
        "itt_render_details_csv": ([vp, vp, C.c_uint64, P(C.c_void_p), P(C.c_uint64)], C.c_int),
        "itt_host_register": ([vp, vp, C.c_uint64], C.c_int),
        "itt_host_unregister": ([vp, vp], C.c_int),
        "itt_ctx_synchronize": ([vp], C.c_int),
        "itt_ctx_stream": ([vp, P(vp)], C.c_int),
        "itt_summarize_streams": ([vp, P(abi.itt_records), C.c_int, P(abi.itt_census)], C.c_int),
        "itt_select_main_stream": ([vp, P(abi.itt_census), P(C.c_uint32), P(C.c_uint32)], C.c_int),
        "itt_build_token_sequence": ([vp, P(abi.itt_records), C.c_uint32, P(P(abi.itt_tokens))], C.c_int),
        "itt_count_interval_overlaps": ([vp, P(abi.itt_records), C.c_uint32, P(C.c_int64)], C.c_int),
        "itt_radix_sort_pairs_u32": ([vp, vp, vp, C.c_uint64, C.c_int, C.c_int, C.c_int], C.c_int),
        "itt_suffix_array": ([vp, P(C.c_int32), C.c_uint64, C.c_int32, P(C.c_uint32), P(C.c_uint32)], C.c_int),
        "itt_suffix_array_capped": ([vp, vp, C.c_uint64, C.c_int32, C.c_uint32, vp, vp], C.c_int),
        "itt_enumerate_repeats": ([vp, P(C.c_int32), C.c_uint64, C.c_int32, C.c_int64, C.c_int64,
                                   P(P(abi.itt_repeat)), P(C.c_uint64)], C.c_int),
        "itt_mine_patterns": ([vp, P(C.c_int32), C.c_uint64, C.c_int32, P(abi.itt_mining_cfg), C.c_uint32, C.c_int,
                               P(P(abi.itt_pattern))], C.c_int),
        "itt_free_patterns": ([vp, P(abi.itt_pattern), C.c_uint32], C.c_int),
        "itt_mine_patterns_sa": ([vp, vp, C.c_uint64, C.c_int32, vp, vp, P(abi.itt_mining_cfg), C.c_uint32, C.c_int,
                                  P(P(abi.itt_pattern))], C.c_int),
        "itt_dsa_keys": ([vp, vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.c_int, vp, vp, C.c_uint64, C.c_int, vp, vp],
                         C.c_int),
        "itt_dsa_partition": ([vp, vp, vp, C.c_uint64, C.c_int, vp, vp, C.c_uint32, vp, C.c_uint32, vp, vp, P(C.c_uint64)],
                              C.c_int),
        "itt_dsa_sort": ([vp, vp, vp, C.c_uint64, C.c_int], C.c_int),
        "itt_dsa_ids": ([vp, vp, vp, C.c_uint64, C.c_int, C.c_uint64, C.c_uint32, vp, P(C.c_uint64)], C.c_int),
        "itt_dsa_scatter": ([vp, vp, C.c_uint64, C.c_uint64, vp], C.c_int),
        "itt_dsa_lcp_requests": ([vp, vp, C.c_uint64, C.c_uint64, C.c_int, C.c_uint64, vp, vp], C.c_int),
        "itt_dsa_kasai": ([vp, vp, C.c_uint64, C.c_uint64, C.c_uint64, vp, vp, C.c_uint32, vp], C.c_int),
        "itt_dsa_sample": ([vp, vp, vp, C.c_uint64, C.c_uint32, vp, vp], C.c_int),
        "itt_comm_nccl_unique_id": ([vp], C.c_int),
        "itt_comm_create_nccl": ([vp, C.c_int, C.c_int, vp, P(vp)], C.c_int),
        "itt_comm_create_local": ([C.c_int, P(vp)], C.c_int),
        "itt_comm_abort": ([vp], C.c_int),
        "itt_comm_destroy": ([vp], C.c_int),
        "itt_dsa_build": ([vp, vp, vp, C.c_uint64, C.c_int32, C.c_uint32, C.c_int, P(vp), P(vp), P(C.c_uint64),
                           P(C.c_uint64), P(abi.itt_dsa_info)], C.c_int),
        "itt_dsa_provider_create": ([vp, vp, C.c_int, P(vp)], C.c_int),
        "itt_dsa_provider_destroy": ([vp], C.c_int),
        "itt_dsa_serve": ([vp], C.c_int),
        "itt_dsa_stop": ([vp], C.c_int),
        "itt_dsa_last_info": ([vp, P(abi.itt_dsa_info)], C.c_int),
        "itt_approx_match": ([vp, P(C.c_int32), C.c_uint64, P(C.c_int32), C.c_uint64, C.c_int64, P(P(abi.itt_span)),
                              P(C.c_uint64)], C.c_int),
        "itt_op_profile": ([vp, P(C.c_int32), P(C.c_int64), P(C.c_int64), P(C.c_uint8), C.c_uint64, C.c_uint32,
                            P(abi.itt_span), C.c_uint64, C.c_int, vp, vp, P(P(abi.itt_op_cell)), P(C.c_uint64)],
                           C.c_int),
        "itt_iteration_metrics": ([vp, P(abi.itt_records), P(C.c_uint64), C.c_uint64, P(abi.itt_span), C.c_uint64,
                                   P(P(abi.itt_iter_row)), P(abi.itt_clamps)], C.c_int),
        "itt_analyze": ([vp, P(abi.itt_records), P(abi.itt_analyze_opts), P(P(abi.itt_analysis))], C.c_int),
        "itt_free_analysis": ([vp, P(abi.itt_analysis)], C.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    if L.itt_abi_version() != abi.ABI_VERSION:
        raise RuntimeError("libitertrace_cuda.so ABI version mismatch")
    _lib = L
    return L


def exported_symbols() -> list[str]:
    """Entry points declared in include/itertrace_cuda.h (checked by the CPU test suite)."""
    hdr = os.path.join(os.path.dirname(_HERE), "include", "itertrace_cuda.h")
    import re
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(itt_\w+)\s*\(", open(hdr).read(), re.M)))


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _ptr(a, t):
    return a.ctypes.data_as(P(t))


class DeviceRecords:
    """Trace columns resident in HBM (allocated through the context).  names_host=True keeps
    name_bytes in (registered, pinned) host memory, streamed chunk by chunk into the hash pass —
    for traces whose names do not fit in HBM next to the pipeline (C5)."""

    def __init__(self, ctx: "Context", recs: abi.Records, names_host: bool = False):
        self.ctx = ctx
        self.n = recs.n
        self.order = recs.order
        self.bufs = {}
        self.mapped = None
        cols = dict(start_ns=recs.start_ns, duration_ns=recs.duration_ns, size_bytes=recs.size_bytes, flags=recs.flags,
                    stream=recs.stream, name_off=recs.name_off, name_bytes=recs.name_bytes)
        if recs.device is not None:
            cols["device"] = recs.device
        self.names_pinned = False
        if names_host:
            a = cols.pop("name_bytes")
            try:
                ctx.register_host(a)  # pinned: full-speed chunk copies that overlap the hash pass
                self.names_pinned = True
            except IttError:
                pass  # the OS refused to lock that much memory: streamed from pageable memory
            self.mapped = a
            self.names_ptr = C.c_void_p(a.ctypes.data)
        for k, a in cols.items():
            p = C.c_void_p()
            ctx._check(lib().itt_device_alloc(ctx.h, max(1, a.nbytes), C.byref(p)))
            ctx._check(lib().itt_memcpy_h2d(ctx.h, p, a.ctypes.data, a.nbytes))
            self.bufs[k] = p
        if names_host:
            self.bufs["name_bytes"] = self.names_ptr
        self.nbytes = sum(a.nbytes for a in cols.values())  # bytes resident in HBM

    def c(self) -> abi.itt_records:
        b = self.bufs
        return abi.itt_records(self.n, b["start_ns"], b["duration_ns"], b["size_bytes"], b["flags"], b["stream"],
                               b.get("device"), b["name_off"], b["name_bytes"],
                               abi.MEM_DEVICE_HOST_NAMES if self.mapped is not None else abi.MEM_DEVICE, self.order)

    def free(self):
        for k, p in self.bufs.items():
            if not (k == "name_bytes" and self.mapped is not None):
                lib().itt_device_free(self.ctx.h, p)
        if self.mapped is not None:
            if self.names_pinned:
                self.ctx.unregister_host(self.mapped)
            self.mapped = None
        self.bufs = {}


class Context:
    def __init__(self, device: int = 0):
        L = lib()
        h = C.c_void_p()
        rc = L.itt_ctx_create(device, C.byref(h))
        if rc != 0:
            raise IttError(rc, f"itt_ctx_create({device}) failed: no usable sm_100 device")
        self.h = h
        self.device = device

    def close(self):
        if self.h:
            lib().itt_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != 0:
            raise IttError(rc, lib().itt_last_error(self.h).decode(errors="replace"))

    # ---------------------------------------------------------------- profiling
    def set_profiling(self, on: bool):
        self._check(lib().itt_ctx_set_profiling(self.h, 1 if on else 0))

    def reset_stats(self):
        self._check(lib().itt_ctx_reset_stats(self.h))

    def kernel_stats(self) -> dict:
        arr = (abi.itt_kernel_stat * 256)()
        n = C.c_uint32()
        self._check(lib().itt_ctx_kernel_stats(self.h, arr, 256, C.byref(n)))
        return {arr[i].name.decode(): dict(launches=arr[i].launches, total_ms=arr[i].total_ms, bytes=arr[i].bytes)
                for i in range(min(n.value, 256))}

    def launch_count(self) -> int:
        v = C.c_uint64()
        self._check(lib().itt_ctx_launch_count(self.h, C.byref(v)))
        return v.value

    def mem_stats(self, reset=False) -> tuple:
        """(bytes in use, high-water mark) of the context's device pool."""
        u, h = C.c_uint64(), C.c_uint64()
        self._check(lib().itt_ctx_mem_stats(self.h, C.byref(u), C.byref(h), 1 if reset else 0))
        return u.value, h.value

    def stream_ptr(self) -> int:
        v = C.c_void_p()
        self._check(lib().itt_ctx_stream(self.h, C.byref(v)))
        return v.value or 0

    def synchronize(self):
        self._check(lib().itt_ctx_synchronize(self.h))

    def parse_csv(self, text: bytes, label: str = "trace.csv") -> "ParsedTrace":
        """itt_parse_csv: parse_trace_text on the GPU."""
        out = P(abi.itt_parsed_trace)()
        self._check(lib().itt_parse_csv(self.h, text, len(text), label.encode(), C.byref(out)))
        return ParsedTrace(self, out)

    def upload(self, recs: abi.Records, names_host: bool = False) -> DeviceRecords:
        return DeviceRecords(self, recs, names_host)

    def register_host(self, arr: np.ndarray):
        self._check(lib().itt_host_register(self.h, arr.ctypes.data, arr.nbytes))

    def unregister_host(self, arr: np.ndarray):
        self._check(lib().itt_host_unregister(self.h, arr.ctypes.data))

    # ---------------------------------------------------------------- primitives
    def radix_sort_pairs(self, keys, vals, begin_bit=0, end_bit=32):
        """Stable sort of (u32 key, u32 value) host arrays; returns sorted copies."""
        k = np.array(keys, dtype=np.uint32, copy=True)
        v = np.array(vals, dtype=np.uint32, copy=True)
        self._check(lib().itt_radix_sort_pairs_u32(self.h, k.ctypes.data, v.ctypes.data, k.shape[0], begin_bit, end_bit,
                                                   abi.MEM_HOST))
        return k, v

    def radix_sort_device(self, keys_ptr, vals_ptr, n, begin_bit=0, end_bit=32):
        self._check(lib().itt_radix_sort_pairs_u32(self.h, keys_ptr, vals_ptr, n, begin_bit, end_bit, abi.MEM_DEVICE))

    # ---------------------------------------------------------------- hot path
    def suffix_array(self, tokens, term: int, want_lcp: bool = True):
        t = _i32(tokens)
        n = t.shape[0]
        sa = np.zeros(n + 1, np.uint32)
        lcp = np.zeros(n + 1, np.uint32) if want_lcp else None
        self._check(lib().itt_suffix_array(self.h, _ptr(t, C.c_int32), n, term, _ptr(sa, C.c_uint32),
                                           _ptr(lcp, C.c_uint32) if want_lcp else None))
        return sa, lcp

    def suffix_array_device(self, tokens_ptr: int, n: int, term: int, sa_ptr: int, lcp_ptr: int = 0,
                            cap: int = 0xFFFFFFFF):
        """itt_suffix_array_capped on device (or host) addresses; lcp_ptr = 0: no LCP."""
        self._check(lib().itt_suffix_array_capped(self.h, C.c_void_p(tokens_ptr), n, term, cap, C.c_void_p(sa_ptr),
                                                  C.c_void_p(lcp_ptr) if lcp_ptr else None))

    def enumerate_repeats(self, tokens, term, min_count, max_len):
        t = _i32(tokens)
        out = P(abi.itt_repeat)()
        cnt = C.c_uint64()
        self._check(lib().itt_enumerate_repeats(self.h, _ptr(t, C.c_int32), t.shape[0], term, min_count, max_len,
                                                C.byref(out), C.byref(cnt)))
        res = [(out[i].start, out[i].length, out[i].count) for i in range(cnt.value)]
        lib().itt_free(self.h, C.cast(out, C.c_void_p))
        return res

    def mine_patterns(self, tokens, term, loops, multi=False):
        t = _i32(tokens)
        cfgs = (abi.itt_mining_cfg * max(1, len(loops)))()
        for i, lp in enumerate(loops):
            cfgs[i].iterations = lp[0]
            cfgs[i].epsilon0 = lp[1] if len(lp) > 1 else 1
            cfgs[i].epsilon_cap = lp[2] if len(lp) > 2 else 0
        out = P(abi.itt_pattern)()
        self._check(lib().itt_mine_patterns(self.h, _ptr(t, C.c_int32), t.shape[0], term, cfgs, len(loops),
                                            1 if multi else 0, C.byref(out)))
        k = len(loops) if multi else 1
        res = [dict(tokens=[out[i].tokens[j] for j in range(out[i].length)], count=out[i].count,
                    first_token=out[i].first_token, epsilon_used=out[i].epsilon_used) for i in range(k)]
        lib().itt_free_patterns(self.h, out, k)
        return res

    # ---------------------------------------------------------------- host finish (report.cu)
    def compute_summary(self, rows: np.ndarray, iterations_declared: int):
        """compute_summary (metrics.hpp:166-202) over analyze_raw rows ([n, 11] int64)."""
        r = np.ascontiguousarray(rows, dtype=np.int64)
        out = abi.itt_summary()
        self._check(lib().itt_compute_summary(self.h, C.c_void_p(r.ctypes.data) if r.size else None, r.shape[0],
                                              iterations_declared, C.byref(out)))
        return out

    def render_details_csv(self, rows: np.ndarray) -> str:
        """details_to_csv (report.hpp:191-220) of analyze_raw rows, rendered natively."""
        r = np.ascontiguousarray(rows, dtype=np.int64)
        p = C.c_void_p()
        n = C.c_uint64()
        self._check(lib().itt_render_details_csv(self.h, C.c_void_p(r.ctypes.data) if r.size else None, r.shape[0],
                                                 C.byref(p), C.byref(n)))
        try:
            return C.string_at(p, n.value).decode()
        finally:
            lib().itt_free(self.h, p)

    def mine_patterns_sa(self, tokens_ptr, n, term, sa_ptr, lcp_ptr, loops, multi=False):
        """mine_pattern(s) over a suffix array built elsewhere (device pointers: tokens[n],
        sa[n+1], lcp[n+1] capped at >= max L_max + 1), e.g. the distributed one (dist_sa.py)."""
        cfgs = (abi.itt_mining_cfg * max(1, len(loops)))()
        for i, lp in enumerate(loops):
            cfgs[i].iterations = lp[0]
            cfgs[i].epsilon0 = lp[1] if len(lp) > 1 else 1
            cfgs[i].epsilon_cap = lp[2] if len(lp) > 2 else 0
        out = P(abi.itt_pattern)()
        self._check(lib().itt_mine_patterns_sa(self.h, C.c_void_p(tokens_ptr), n, term, C.c_void_p(sa_ptr),
                                               C.c_void_p(lcp_ptr), cfgs, len(loops), 1 if multi else 0, C.byref(out)))
        k = len(loops) if multi else 1
        res = [dict(tokens=[out[i].tokens[j] for j in range(out[i].length)], count=out[i].count,
                    first_token=out[i].first_token, epsilon_used=out[i].epsilon_used) for i in range(k)]
        lib().itt_free_patterns(self.h, out, k)
        return res

    def approx_match(self, tokens, pattern, k0):
        t = _i32(tokens)
        p = _i32(pattern)
        out = P(abi.itt_span)()
        cnt = C.c_uint64()
        self._check(lib().itt_approx_match(self.h, _ptr(t, C.c_int32), t.shape[0], _ptr(p, C.c_int32), p.shape[0], k0,
                                           C.byref(out), C.byref(cnt)))
        res = np.array([(out[i].start_token, out[i].end_token, out[i].extra) for i in range(cnt.value)],
                       dtype=np.int64).reshape(-1, 3)
        lib().itt_free(self.h, C.cast(out, C.c_void_p))
        return res

    def build_token_sequence(self, recs, main_stream):
        c = recs.c()
        out = P(abi.itt_tokens)()
        self._check(lib().itt_build_token_sequence(self.h, C.byref(c), main_stream, C.byref(out)))
        o = out[0]
        n = o.n
        tok = np.ctypeslib.as_array(o.tokens, shape=(n,)).copy() if n else np.zeros(0, np.int32)
        ri = np.ctypeslib.as_array(o.record_index, shape=(n,)).copy() if n else np.zeros(0, np.uint64)
        names = (np.ctypeslib.as_array(o.name_row, shape=(o.n_names,)).copy() if o.n_names
                 else np.zeros(0, np.uint64))
        for p in (o.tokens, o.record_index, o.name_row):
            lib().itt_free(self.h, C.cast(p, C.c_void_p))
        lib().itt_free(self.h, C.cast(out, C.c_void_p))
        return tok, ri, names

    def count_interval_overlaps(self, recs, stream):
        c = recs.c()
        v = C.c_int64()
        self._check(lib().itt_count_interval_overlaps(self.h, C.byref(c), stream, C.byref(v)))
        return v.value

    def summarize_streams(self, recs, filter_device=False):
        c = recs.c()
        out = abi.itt_census()
        self._check(lib().itt_summarize_streams(self.h, C.byref(c), 1 if filter_device else 0, C.byref(out)))
        from_c = [(s.stream, s.cls, tuple(s.counts[k] for k in range(6)), s.first_start, s.last_end)
                  for s in (out.streams[i] for i in range(out.n_streams))]
        info = dict(n_devices=out.n_devices, majority_device=out.majority_device, dropped=out.dropped_records,
                    n_records=out.n_records)
        lib().itt_free(self.h, C.cast(out.streams, C.c_void_p))
        return from_c, info

    def iteration_metrics(self, recs, record_index, spans):
        c = recs.c()
        ri = np.ascontiguousarray(record_index, dtype=np.uint64)
        sp = (abi.itt_span * max(1, len(spans)))()
        for i, s in enumerate(spans):
            sp[i].start_token, sp[i].end_token, sp[i].extra = int(s[0]), int(s[1]), int(s[2])
        rows = P(abi.itt_iter_row)()
        cl = abi.itt_clamps()
        self._check(lib().itt_iteration_metrics(self.h, C.byref(c), _ptr(ri, C.c_uint64), ri.shape[0], sp, len(spans),
                                                C.byref(rows), C.byref(cl)))
        out = [abi.itt_iter_row.from_buffer_copy(rows[i]) for i in range(len(spans))]
        lib().itt_free(self.h, C.cast(rows, C.c_void_p))
        return out, (cl.negative_gap_clamps, cl.negative_interval_clamps)

    def analyze_raw(self, recs, loops, epsilon0=1, k0=-1, main_stream=-1, op_profile=False, sa_provider=None,
                    native_provider=None) -> dict:
        """itt_analyze: device pipeline up to the per-loop integer aggregates.  The per-iteration
        rows (and the a12 op profile: op_profile=True for the per-op / per-iteration totals,
        "cells" for the (iteration, op) grid as well) are zero-copy numpy views of the library's
        pinned output blocks; the analysis is released (blocks back to the context) when the
        last view is dropped."""
        c = recs.c()
        lp = (C.c_int64 * max(1, len(loops)))(*loops)
        flags = 0
        if op_profile:
            flags |= abi.ITT_ANALYZE_OP_PROFILE
        if op_profile == "cells":
            flags |= abi.ITT_ANALYZE_OP_CELLS
        opts = abi.itt_analyze_opts(lp, len(loops), epsilon0, k0, main_stream, flags)
        if sa_provider is not None:  # fn(tokens_ptr, n, term, cap, sa_ptr, lcp_ptr); raises on failure
            failure = []

            def _cb(user, tok, n, term, cap, sa, lcp):
                try:
                    sa_provider(tok, n, term, cap, sa, lcp)
                    return 0
                except BaseException as e:  # noqa: BLE001 (reported after the call returns)
                    failure.append(e)
                    return 1
            opts.sa_provider = abi.SA_PROVIDER(_cb)
        if native_provider is not None:  # the C++/NCCL distributed suffix array (dist_native.Provider)
            opts.sa_provider = C.cast(lib().itt_dsa_provide, abi.SA_PROVIDER)
            opts.sa_user = native_provider.handle
        out = P(abi.itt_analysis)()
        rc = lib().itt_analyze(self.h, C.byref(c), C.byref(opts), C.byref(out))
        if sa_provider is not None and failure:
            raise failure[0]
        self._check(rc)
        owner = _AnalysisOwner(self, out)
        a = out[0]
        res = dict(
            streams=[(s.stream, s.cls, tuple(s.counts[k] for k in range(6)), s.first_start, s.last_end)
                     for s in (a.census.streams[i] for i in range(a.census.n_streams))],
            n_devices=a.census.n_devices, majority_device=a.census.majority_device,
            dropped=a.census.dropped_records, main_stream=a.main_stream, n_main_streams=a.n_main_streams,
            override_non_main=bool(a.main_stream_override_non_main), n_tokens=a.n_tokens, n_names=a.n_names,
            name_row=np.ctypeslib.as_array(a.name_row, shape=(a.n_names,)).tolist() if a.n_names else [],
            overlapping_kernels=a.overlapping_kernels,
            loops=[])
        for k in range(a.n_loops):
            L = a.loops[k]
            if L.n_iterations:
                buf = (C.c_int64 * (L.n_iterations * 11)).from_address(C.cast(L.rows, C.c_void_p).value)
                buf._owner = owner  # keeps the analysis (and the context) alive while views exist
                rows = np.frombuffer(buf, dtype=np.int64).reshape(L.n_iterations, 11)
            else:
                rows = np.zeros((0, 11), np.int64)
            res["loops"].append(dict(
                iterations_declared=L.iterations_declared, pattern_length=L.pattern_length,
                pattern_tokens=(np.ctypeslib.as_array(L.pattern_tokens, shape=(L.pattern_length,)).tolist()
                                if L.pattern_length else []),
                pattern_count=L.pattern_count, epsilon_used=L.epsilon_used, first_token=L.first_token,
                k0_used=L.k0_used, rows=rows,
                clamps=(L.clamps.negative_gap_clamps, L.clamps.negative_interval_clamps)))
            if op_profile:
                res["loops"][-1]["op_totals"] = _view(L.op_totals, a.n_names, abi.OP_TOTAL_DTYPE, owner)
                res["loops"][-1]["iter_op_totals"] = _view(L.iter_op_totals, L.n_iterations, abi.ITER_OP_TOTAL_DTYPE,
                                                           owner)
                res["loops"][-1]["op_cells"] = _view(L.op_cells, L.n_op_cells, abi.OP_CELL_DTYPE, owner)
        return res

    def op_profile(self, tokens, tok_start, tok_end, tok_kind, n_ops, spans, method=abi.ITT_OP_PROFILE_AUTO,
                   cells=True):
        """itt_op_profile (a12) over token-level arrays -> (cells | None, op_totals, iter_totals)."""
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        ts = np.ascontiguousarray(tok_start, dtype=np.int64)
        te = np.ascontiguousarray(tok_end, dtype=np.int64)
        tk = np.ascontiguousarray(tok_kind, dtype=np.uint8)
        sp = (abi.itt_span * max(1, len(spans)))()
        for i, s in enumerate(spans):
            sp[i].start_token, sp[i].end_token, sp[i].extra = int(s[0]), int(s[1]), int(s[2])
        out = P(abi.itt_op_cell)()
        cnt = C.c_uint64()
        ot = np.zeros(max(1, n_ops), abi.OP_TOTAL_DTYPE)
        it = np.zeros(max(1, len(spans)), abi.ITER_OP_TOTAL_DTYPE)
        self._check(lib().itt_op_profile(self.h, _ptr(t, C.c_int32), _ptr(ts, C.c_int64), _ptr(te, C.c_int64),
                                         _ptr(tk, C.c_uint8), t.shape[0], n_ops, sp, len(spans), method,
                                         ot.ctypes.data, it.ctypes.data, C.byref(out) if cells else None,
                                         C.byref(cnt)))
        res = None
        if cells:
            n = cnt.value
            res = np.zeros(n, abi.OP_CELL_DTYPE)
            if n:
                C.memmove(res.ctypes.data, out, n * C.sizeof(abi.itt_op_cell))
            lib().itt_free(self.h, out)
        return res, ot[:n_ops], it[:len(spans)]


class ParsedTrace:
    """itt_parse_csv result: records resident in HBM (source line order) + the IngestReport.
    Pass it to Context.analyze_raw like any record set."""

    def __init__(self, ctx: "Context", ptr):
        self.ctx = ctx
        self.ptr = ptr
        p = ptr[0]
        self.n = int(p.records.n)
        self.rows_total, self.rows_parsed, self.rows_skipped = int(p.rows_total), int(p.rows_parsed), int(p.rows_skipped)
        self.column = {k: int(p.column[i]) for i, k in enumerate(
            ("Start", "Duration", "Size", "Throughput", "Device", "Stream", "Name")) if p.column[i] >= 0}
        self.device_labels = [p.device_labels[i].decode("utf-8", "surrogateescape") for i in range(p.n_device_labels)]
        self.skips = [(int(p.skip_line[i]), p.skip_reason[i].decode("utf-8", "surrogateescape")) for i in range(p.n_skips)]
        self.warnings = [p.warnings[i].decode("utf-8", "surrogateescape") for i in range(p.n_warnings)]
        self.line = np.ctypeslib.as_array(p.line, shape=(self.n,)).copy() if self.n else np.zeros(0, np.uint64)

    def c(self) -> abi.itt_records:
        return self.ptr[0].records

    def columns(self) -> dict:
        """Host copies of the device columns (tests)."""
        r = self.ptr[0].records
        out = {}
        for name, dt, cnt in (("start_ns", np.int64, self.n), ("duration_ns", np.int64, self.n),
                              ("size_bytes", np.int64, self.n), ("flags", np.uint8, self.n),
                              ("stream", np.uint32, self.n), ("device", np.uint16, self.n),
                              ("name_off", np.uint64, self.n + 1)):
            a = np.zeros(max(1, cnt), dt)
            self.ctx._check(lib().itt_memcpy_d2h(self.ctx.h, a.ctypes.data, C.cast(getattr(r, name), C.c_void_p),
                                                a.nbytes if cnt else 0))
            out[name] = a[:cnt]
        nb = int(out["name_off"][-1]) if self.n else 0
        b = np.zeros(max(1, nb), np.uint8)
        self.ctx._check(lib().itt_memcpy_d2h(self.ctx.h, b.ctypes.data, C.cast(r.name_bytes, C.c_void_p), nb))
        out["name_bytes"] = b[:nb]
        self.ctx.synchronize()
        return out

    def free(self):
        if self.ptr is not None and self.ctx.h:
            lib().itt_free_parsed(self.ctx.h, self.ptr)
        self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Batch:
    """Native batch executor (itt_batch_*): `workers` C++ threads, one context each, on `device`."""

    def __init__(self, device: int = 0, workers: int = 8):
        h = C.c_void_p()
        rc = lib().itt_batch_create(device, workers, C.byref(h))
        if rc != 0:
            raise IttError(rc, f"itt_batch_create({device}, {workers}) failed")
        self.h = h
        self.workers = workers

    def close(self):
        if self.h:
            lib().itt_batch_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def launch_count(self) -> int:
        v = C.c_uint64()
        lib().itt_batch_launch_count(self.h, C.byref(v))
        return v.value

    def analyze(self, traces, loops, epsilon0=1, k0=-1, main_stream=-1, summarize=None, batched_sa=False):
        """Analyze every trace (abi.Records or DeviceRecords); returns per-trace results:
        summarize(itt_analysis) if given (read while the analyses are alive), else
        (status, pattern_length, pattern_count, iterations) of loop 0; errors as IttError.
        batched_sa: the suffix arrays of the traces in flight are built in one doubling sequence."""
        n = len(traces)
        recs = (abi.itt_records * max(1, n))(*[t.c() for t in traces])
        lp = (C.c_int64 * max(1, len(loops)))(*loops)
        opts = abi.itt_analyze_opts(lp, len(loops), epsilon0, k0, main_stream,
                                    abi.ITT_ANALYZE_BATCHED_SA if batched_sa else 0)
        out = (P(abi.itt_analysis) * max(1, n))()
        st = (C.c_int * max(1, n))()
        rc = lib().itt_batch_analyze(self.h, recs, n, C.byref(opts), 0, out, st)
        if rc != 0:
            raise IttError(rc, "itt_batch_analyze failed")
        try:
            res = []
            for i in range(n):
                if st[i] != 0:
                    res.append(IttError(st[i], lib().itt_batch_error(self.h, i).decode(errors="replace")))
                elif summarize is not None:
                    res.append(summarize(out[i][0]))
                else:
                    L = out[i][0].loops[0]
                    res.append((0, L.pattern_length, L.pattern_count, L.n_iterations))
            return res
        finally:
            lib().itt_batch_free(self.h, out, n)


def _view(ptr, n, dtype, owner):
    """Zero-copy numpy view of a library-owned pinned block (kept alive by `owner`)."""
    if not n or not ptr:
        return np.zeros(0, dtype)
    buf = (C.c_uint8 * (n * dtype.itemsize)).from_address(C.cast(ptr, C.c_void_p).value)
    buf._owner = owner
    return np.frombuffer(buf, dtype=dtype)


class _AnalysisOwner:
    def __init__(self, ctx: Context, ptr):
        self.ctx = ctx
        self.ptr = ptr

    def __del__(self):
        try:
            if self.ctx.h:  # after close() the context already released its pinned blocks
                lib().itt_free_analysis(self.ctx.h, self.ptr)
        except Exception:
            pass


# column order of analyze_raw()["loops"][k]["rows"] (itt_iter_row as int64 words; the last word
# packs has_interval | pad)
ROW_FIELDS = ["start_token", "end_token", "extra", "t_start", "t_end", "interval_ns", "copy_ns", "htod_bytes",
              "gap_sum", "gap_count", "has_interval"]
