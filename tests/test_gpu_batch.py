"""GPU: the native batch executor (itt_batch_*, C4) with and without batched suffix arrays
(ITT_ANALYZE_BATCHED_SA: the traces in flight share one doubling sequence over their
concatenation, separators above every token).  Every trace's full result (pattern, counts,
per-iteration integer rows) must equal the single-trace analyze, including traces of
different lengths, alphabets and iteration counts in one wave, and a trace that fails before
its suffix-array stage (it leaves the wave without blocking the others)."""
from __future__ import annotations

import numpy as np
import pytest

from paper_1707_03750_b200 import abi, cuda, synth

pytestmark = pytest.mark.gpu


def _summ(a):
    out = []
    for k in range(a.n_loops):
        L = a.loops[k]
        rows = np.ctypeslib.as_array(C.cast(L.rows, C.POINTER(C.c_int64)), shape=(L.n_iterations * 11,)).copy() \
            if L.n_iterations else np.zeros(0, np.int64)
        out.append((L.pattern_length, [L.pattern_tokens[j] for j in range(L.pattern_length)], L.pattern_count,
                    L.first_token, L.epsilon_used, L.n_iterations, rows.tobytes()))
    return out


import ctypes as C  # noqa: E402


@pytest.mark.parametrize("workers", [1, 3, 8])
def test_batched_suffix_arrays_match_single_trace(ctx, workers):
    traces, loops = [], []
    for t in range(13):
        iters = 20 + 7 * (t % 4)
        recs, _ = synth.generate(seed=500 + t, iterations=iters, body_len=10 + 5 * (t % 3), vocab=8 + t)
        traces.append(recs)
        loops.append(iters)
    # one loop count for the whole batch call: group traces by their count
    b = cuda.Batch(0, workers)
    try:
        for iters in sorted(set(loops)):
            group = [tr for tr, l in zip(traces, loops) if l == iters]
            want = b.analyze(group, [iters], summarize=_summ)
            got = b.analyze(group, [iters], summarize=_summ, batched_sa=True)
            assert got == want
            single = [_summ_single(ctx, tr, iters) for tr in group]
            assert [g[0][:6] for g in got] == [s_[:6] for s_ in single]
    finally:
        b.close()


def _summ_single(ctx, tr, iters):
    r = ctx.analyze_raw(tr, [iters])
    L = r["loops"][0]
    return (L["pattern_length"], L["pattern_tokens"], L["pattern_count"], L["first_token"], L["epsilon_used"],
            L["rows"].shape[0])


def test_batched_wave_survives_a_failing_trace(ctx):
    good = [synth.generate(seed=700 + t, iterations=30, body_len=12, vocab=9)[0] for t in range(5)]
    bad = abi.Records(np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0, np.uint32), names=[])  # EmptyTrace
    b = cuda.Batch(0, 4)
    try:
        res = b.analyze(good[:2] + [bad] + good[2:], [30], batched_sa=True)
        assert isinstance(res[2], cuda.IttError) and res[2].kind == "EmptyTrace"
        want = b.analyze(good, [30])
        assert [r for i, r in enumerate(res) if i != 2] == want
    finally:
        b.close()
