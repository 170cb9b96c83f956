"""CPU: the native host finish (report.cu: itt_compute_summary, itt_render_details_csv — SURVEY
§8f row 4) equals the Python restatement of compute_summary (metrics.hpp:166-202) and
details_to_csv (report.hpp:191-220), which the GPU tests pin to the reference byte for byte:
every summary double bit for bit, the CSV byte for byte, on random rows with the edge cases
(first row without interval, zero and negative-clamped intervals, no gaps, huge values) and at
C5's 500K iterations.  Host functions only: called with a NULL context (no GPU needed)."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from paper_1707_03750_b200 import abi, cuda, itertrace


def _rows(n, seed):
    rng = np.random.default_rng(seed)
    r = np.zeros((n, 11), np.int64)
    r[:, 0] = np.arange(n) * 200
    r[:, 1] = r[:, 0] + rng.integers(150, 260, n)
    r[:, 2] = rng.integers(0, 5, n)
    r[:, 3] = np.arange(n) * 10**6 + rng.integers(0, 1000, n)
    r[:, 4] = r[:, 3] + rng.integers(10**5, 9 * 10**5, n)
    r[:, 5] = rng.choice([0, 1, 7, 4000, 11999, 10**12], n)
    r[:, 6] = rng.integers(0, 5000, n)
    r[:, 7] = rng.integers(0, 9000, n)
    r[:, 8] = rng.integers(0, 3 * 10**9, n)
    r[:, 9] = rng.choice([0, 1, 3, 199, 1999], n)
    r[:, 10] = rng.integers(0, 2, n)
    r[0, 10] = 0
    return r


def _native(rows, iters):
    L = cuda.lib()
    r = np.ascontiguousarray(rows)
    out = abi.itt_summary()
    rc = L.itt_compute_summary(None, C.c_void_p(r.ctypes.data) if r.size else None, r.shape[0], iters, C.byref(out))
    p, n = C.c_void_p(), C.c_uint64()
    rc2 = L.itt_render_details_csv(None, C.c_void_p(r.ctypes.data) if r.size else None, r.shape[0], C.byref(p), C.byref(n))
    assert rc2 == 0
    text = C.string_at(p, n.value).decode()
    L.itt_free(None, p)
    return rc, out, text


@pytest.mark.parametrize("n,seed", [(1, 1), (2, 2), (37, 3), (5000, 4), (500_000, 5)])
def test_native_finish_matches_restatement(n, seed):
    rows = _rows(n, seed)
    items = itertrace.rows_to_metrics(rows)
    want = itertrace.compute_summary(items, n + 3)
    rc, got, text = _native(rows, n + 3)
    assert rc == 0
    for f in ("avg_interval_ns", "avg_overlap", "avg_operation_ns", "avg_size_bytes"):
        assert float(getattr(got, f)).hex() == float(getattr(want, f)).hex(), f
    assert got.max_interval_ns == want.max_interval_ns
    assert (got.iterations_found, got.iterations_declared) == (want.iterations_found, want.iterations_declared)
    assert bool(got.insufficient_intervals) == want.insufficient_intervals
    if n <= 5000:
        assert text == itertrace.details_to_csv(items)
    else:  # the interpreted renderer takes seconds here: spot-check blocks against it
        lines = text.split("\n")
        for a in (0, 16383, 16384, 250_000, n - 3):
            assert lines[1 + a: 1 + a + 3] == itertrace.details_to_csv(items[a: a + 3]).split("\n")[1:4][: len(lines[1 + a: 1 + a + 3])] \
                or a + 3 > n
        assert len(lines) == n + 2


def test_native_summary_no_iterations():
    rc, _, text = _native(np.zeros((0, 11), np.int64), 5)
    assert rc == 1 + abi.ERROR_KINDS.index("NoIterations")
    assert text == itertrace.DETAILS_HEADER + "\n"
