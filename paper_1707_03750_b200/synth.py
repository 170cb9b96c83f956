"""Deterministic TF-like trace generator (ctypes over libitt_synth.so; include/itt_synth.h).

Test/bench infrastructure: produces the columnar records of the BASELINE configs
(SURVEY §8(d)).  Host only, no CUDA.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .abi import ORDER_UNKNOWN, Records

_HERE = os.path.dirname(os.path.abspath(__file__))


class itt_synth_cfg(C.Structure):
    _fields_ = [
        ("seed", C.c_uint64), ("iterations", C.c_int64), ("body_len", C.c_int64), ("vocab", C.c_int64),
        ("init_ops", C.c_int64), ("noise_frac", C.c_double), ("shuffle_window", C.c_int64),
        ("minority_frac", C.c_double), ("name_min", C.c_int64), ("name_max", C.c_int64),
        ("kdur_lo", C.c_int64), ("kdur_hi", C.c_int64), ("intra_lo", C.c_int64), ("intra_hi", C.c_int64),
        ("inter_lo", C.c_int64), ("inter_hi", C.c_int64), ("htod_lo", C.c_int64), ("htod_hi", C.c_int64),
        ("body_inserts", C.c_int64), ("insert_prob", C.c_double), ("extra_stream_frac", C.c_double),
    ]


class itt_synth_trace(C.Structure):
    _fields_ = [
        ("n", C.c_uint64), ("start_ns", C.c_void_p), ("duration_ns", C.c_void_p), ("size_bytes", C.c_void_p),
        ("flags", C.c_void_p), ("stream", C.c_void_p), ("device", C.c_void_p), ("name_off", C.c_void_p),
        ("name_bytes", C.c_void_p), ("name_bytes_len", C.c_uint64), ("n_main", C.c_uint64), ("n_htod", C.c_uint64),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "libitt_synth.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        _lib = C.CDLL(path)
        _lib.itt_synth_default.argtypes = [C.POINTER(itt_synth_cfg)]
        _lib.itt_synth_generate.argtypes = [C.POINTER(itt_synth_cfg), C.POINTER(itt_synth_trace)]
        _lib.itt_synth_free.argtypes = [C.POINTER(itt_synth_trace)]
        _lib.itt_synth_to_csv.argtypes = [C.POINTER(itt_synth_trace), C.POINTER(C.c_void_p), C.POINTER(C.c_uint64)]
    return _lib


class _Owner:
    def __init__(self, t):
        self.t = t

    def __del__(self):
        try:
            lib().itt_synth_free(C.byref(self.t))
        except Exception:
            pass


# BASELINE.json configs; C5 is the distributed 1B case.
CONFIGS = {
    "C1": dict(iterations=100, body_len=200, vocab=150, seed=1),
    "C2": dict(iterations=50_000, body_len=200, vocab=150, seed=2, noise_frac=0.05, shuffle_window=64),
    "C3": dict(iterations=20_000, body_len=5_000, vocab=4_096, seed=3),
    "C4": dict(iterations=500, body_len=200, vocab=150, seed=1000),
    "C5": dict(iterations=500_000, body_len=2_000, vocab=4_096, seed=5),
}


def generate(**kw) -> tuple[Records, dict]:
    """Generate a trace; returns (Records, info).  Keyword names follow itt_synth_cfg."""
    cfg = itt_synth_cfg()
    lib().itt_synth_default(C.byref(cfg))
    for k, v in kw.items():
        setattr(cfg, k, v)
    t = itt_synth_trace()
    rc = lib().itt_synth_generate(C.byref(cfg), C.byref(t))
    if rc != 0:
        raise RuntimeError(f"itt_synth_generate failed ({rc})")
    owner = _Owner(t)
    n = int(t.n)

    def arr(ptr, dtype, count):
        if count == 0:
            return np.zeros(0, dtype)
        return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(np.ctypeslib.as_ctypes_type(dtype))), shape=(count,))

    recs = Records(
        start_ns=arr(t.start_ns, np.int64, n), duration_ns=arr(t.duration_ns, np.int64, n),
        stream=arr(t.stream, np.uint32, n), name_off=arr(t.name_off, np.uint64, n + 1),
        name_bytes=arr(t.name_bytes, np.uint8, max(1, int(t.name_bytes_len))),
        size_bytes=arr(t.size_bytes, np.int64, n), flags=arr(t.flags, np.uint8, n),
        device=arr(t.device, np.uint16, n), order=ORDER_UNKNOWN, keepalive=owner)
    info = dict(n=n, n_main=int(t.n_main), n_htod=int(t.n_htod), name_bytes=int(t.name_bytes_len))
    return recs, info


def to_csv(recs: Records) -> bytes:
    """Profiler CSV text of a generated trace (the reference's format; itt_synth_to_csv)."""
    owner = recs._keepalive
    p, n = C.c_void_p(), C.c_uint64()
    if lib().itt_synth_to_csv(C.byref(owner.t), C.byref(p), C.byref(n)) != 0:
        raise RuntimeError("itt_synth_to_csv failed")
    try:
        return C.string_at(p, n.value)
    finally:
        C.CDLL(None).free(p)


def generate_config(name: str, **override) -> tuple[Records, dict]:
    kw = dict(CONFIGS[name])
    kw.update(override)
    return generate(**kw)
