"""a12 — the second-level per-op profile (definition: itt_op_cell in
include/itertrace_cuda.h).

The reference has no such function, so parity cannot be pinned to a reference output directly.
The chain of evidence instead:
  * the oracle (orc_op_profile) restates the definition with plain loops and is checked against
    an independent pure-Python brute force (CPU tests below);
  * its idle column is pinned to the REFERENCE: for every golden trace, sum over ops of idle_ns
    in iteration k, divided by the iteration's gap count, equals the reference's op_gap_mean_ns
    (metrics.hpp:145-160) bit for bit, and sum over ops of count equals the span length;
  * the device (both the shared-memory and the sort path) must equal the oracle cell for cell.
"""
from __future__ import annotations

import random

import numpy as np
import pytest

from paper_1707_03750_b200 import abi, synth
from paper_1707_03750_b200.itertrace import reduce_cells

gpu = pytest.mark.gpu


def brute_cells(tokens, ts, te, kind, spans):
    out = []
    for k, (s, e, _x) in enumerate(spans):
        acc = {}
        for j in range(s, e + 1):
            v = int(tokens[j])
            c = acc.setdefault(v, [0, 0, 0, 0])
            c[0] += 1
            c[1 if kind[j] == abi.KIND_KERNEL else 2] += int(te[j]) - int(ts[j])
            if j > s:
                c[3] += max(0, int(ts[j]) - int(te[j - 1]))
        for v in sorted(acc):
            out.append((k, v, *acc[v]))
    return out


def as_tuples(cells):
    return [(int(c["iteration"]), int(c["op"]), int(c["count"]), int(c["kernel_ns"]), int(c["memcpy_ns"]),
             int(c["idle_ns"])) for c in cells]


def random_tokens(rng, n, n_ops, n_spans):
    tokens = np.array([rng.randrange(n_ops) for _ in range(n)], np.int32)
    ts = np.cumsum([rng.randrange(0, 50) for _ in range(n)]).astype(np.int64)
    te = ts + np.array([rng.randrange(0, 80) for _ in range(n)], np.int64)  # overlaps -> negative gaps
    kind = np.array([rng.choice([0, 0, 0, 1, 2, 3, 4, 5]) for _ in range(n)], np.uint8)
    cuts = sorted(rng.sample(range(n + 1), min(n + 1, 2 * n_spans)))
    spans = []
    for a, b in zip(cuts[0::2], cuts[1::2]):
        if b > a:
            spans.append((a, b - 1, rng.randrange(3)))
    return tokens, ts, te, kind, spans


def token_arrays(O, recs, main_stream):
    """Main-stream token columns in (start,row) order, by the oracle (streams.hpp:147-169)."""
    perm = O.sort_records(recs.start_ns).astype(np.int64)
    tok, ri, names = O.build_token_sequence(recs, main_stream)
    rows = perm[ri.astype(np.int64)]
    ts = recs.start_ns[rows]
    te = ts + recs.duration_ns[rows]
    kind = np.array([O.classify(recs.name(r), bool(recs.flags[r] & abi.REC_HAS_THROUGHPUT)) for r in rows], np.uint8)
    return tok, ts, te, kind, len(names)


# ---------------------------------------------------------------- CPU: the oracle itself
def test_oracle_matches_brute_force(O):
    rng = random.Random(17)
    for trial in range(60):
        n = rng.randrange(1, 300)
        n_ops = rng.randrange(1, 40)
        tokens, ts, te, kind, spans = random_tokens(rng, n, n_ops, rng.randrange(0, 12))
        got = as_tuples(O.op_profile(tokens, ts, te, kind, n_ops, spans))
        assert got == brute_cells(tokens, ts, te, kind, spans), trial


def test_oracle_idle_column_is_pinned_to_the_reference_gap_means(O, trace_cases):
    """sum_v idle(k, v) / gap_count(k) == the reference's op_gap_mean_ns (golden, bitwise)."""
    checked = 0
    for c in trace_cases:
        if "error" in c or any("MultiDeviceTrace" in w for w in c["warnings"]):
            continue
        recs, _ = synth.generate(**c["generator"])
        tok, ts, te, kind, n_ops = token_arrays(O, recs, c["main_stream"])
        for G in c["loops_out"][:1]:
            spans = [(x[1], x[2], x[3]) for x in G["iters"]]
            cells = O.op_profile(tok, ts, te, kind, n_ops, spans)
            idle = np.zeros(len(spans), np.int64)
            cnt = np.zeros(len(spans), np.int64)
            np.add.at(idle, cells["iteration"].astype(np.int64), cells["idle_ns"])
            np.add.at(cnt, cells["iteration"].astype(np.int64), cells["count"].astype(np.int64))
            for k, x in enumerate(G["iters"]):
                s, e = x[1], x[2]
                assert cnt[k] == e - s + 1
                mean = float(idle[k]) / float(e - s) if e > s else 0.0
                assert mean.hex() == x[11], (c["name"], k)
                checked += 1
    assert checked > 100


# ---------------------------------------------------------------- GPU: device vs oracle
@gpu
@pytest.mark.parametrize("method", [abi.ITT_OP_PROFILE_SMEM, abi.ITT_OP_PROFILE_SORT])
def test_device_op_profile_random(ctx, O, method):
    rng = random.Random(5 + method)
    for trial in range(40):
        n = rng.randrange(1, 3000)
        n_ops = rng.choice([1, 2, 7, 150, 4112, 7936])
        tokens, ts, te, kind, spans = random_tokens(rng, n, n_ops, rng.randrange(0, 40))
        want = O.op_profile(tokens, ts, te, kind, n_ops, spans)
        got, ot, it = ctx.op_profile(tokens, ts, te, kind, n_ops, spans, method)
        assert as_tuples(got) == as_tuples(want), (trial, method)
        wo, wi = reduce_cells(want, n_ops, len(spans))
        assert np.array_equal(ot, wo) and np.array_equal(it, wi), (trial, method)
        none, ot2, it2 = ctx.op_profile(tokens, ts, te, kind, n_ops, spans, method, cells=False)
        assert none is None and np.array_equal(ot2, wo) and np.array_equal(it2, wi), (trial, method)


@gpu
def test_device_op_profile_edges(ctx, O):
    # one-token spans, a span covering everything, op ids above the shared-memory table (AUTO -> sort)
    tokens = np.array([3, 3, 1, 0, 3, 2], np.int32)
    ts = np.array([0, 5, 5, 20, 21, 40], np.int64)
    te = np.array([4, 9, 30, 21, 22, 41], np.int64)
    kind = np.array([0, 1, 0, 0, 5, 2], np.uint8)
    for spans in ([(0, 0, 0)], [(0, 5, 0)], [(0, 1, 0), (2, 2, 1), (4, 5, 0)], []):
        for method in (abi.ITT_OP_PROFILE_AUTO, abi.ITT_OP_PROFILE_SMEM, abi.ITT_OP_PROFILE_SORT):
            got, ot, it = ctx.op_profile(tokens, ts, te, kind, 4, spans, method)
            want = O.op_profile(tokens, ts, te, kind, 4, spans)
            assert as_tuples(got) == as_tuples(want)
            wo, wi = reduce_cells(want, 4, len(spans))
            assert np.array_equal(ot, wo) and np.array_equal(it, wi)
    big = 100000  # n_ops beyond the shared-memory table: AUTO takes the sort path
    rng = random.Random(3)
    t2 = np.array([rng.randrange(big) for _ in range(5000)], np.int32)
    ts2 = np.arange(5000, dtype=np.int64) * 10
    te2 = ts2 + 7
    k2 = np.zeros(5000, np.uint8)
    sp2 = [(0, 999, 0), (1500, 4999, 2)]
    got, ot, it = ctx.op_profile(t2, ts2, te2, k2, big, sp2)
    want = O.op_profile(t2, ts2, te2, k2, big, sp2)
    assert as_tuples(got) == as_tuples(want)
    wo, wi = reduce_cells(want, big, len(sp2))
    assert np.array_equal(ot, wo) and np.array_equal(it, wi)
    from paper_1707_03750_b200.cuda import IttError
    with pytest.raises(IttError):  # overlapping spans
        ctx.op_profile(tokens, ts, te, kind, 4, [(0, 3, 0), (3, 5, 0)])
    with pytest.raises(IttError):  # op id outside [0, n_ops)
        ctx.op_profile(tokens, ts, te, kind, 3, [(0, 5, 0)])
    with pytest.raises(IttError):  # shared-memory path forced beyond its table
        ctx.op_profile(t2, ts2, te2, k2, big, sp2, abi.ITT_OP_PROFILE_SMEM)


@gpu
def test_analyze_op_profile_golden_traces(ctx, O, trace_cases):
    """itt_analyze with ITT_ANALYZE_OP_PROFILE: cells == oracle over the reference's token
    sequence and spans; idle sums reproduce the reference's gap means bit for bit."""
    from paper_1707_03750_b200 import itertrace
    checked = 0
    for c in trace_cases:
        if "error" in c or any("MultiDeviceTrace" in w for w in c["warnings"]):
            continue
        recs, _ = synth.generate(**c["generator"])
        o = c["opts"]
        r = itertrace.analyze_trace(ctx, recs, c["loops"], epsilon0=o.get("epsilon0", 1), k0=o.get("k0"),
                                    main_stream=o.get("main_stream"), op_profile="cells")
        assert r.summary_json() == c["summary_json"]  # the reference outputs are unchanged
        tok, ts, te, kind, n_ops = token_arrays(O, recs, r.main_stream)
        for p, items in zip(r.op_profiles, r.details):
            spans = [(m.start_token, m.end_token, m.extra_ops) for m in items]
            want = O.op_profile(tok, ts, te, kind, n_ops, spans)
            assert as_tuples(p.cells) == as_tuples(want), c["name"]
            wo, wi = reduce_cells(want, n_ops, len(spans))
            assert np.array_equal(p.per_op, wo) and np.array_equal(p.per_iteration, wi), c["name"]
            for m, it in zip(items, p.per_iteration):
                gc = m.end_token - m.start_token
                mean = float(int(it["idle_ns"])) / float(gc) if gc > 0 else 0.0
                assert mean.hex() == m.op_gap_mean_ns.hex()
            assert p.per_op_csv().count("\n") == 1 + int((wo["count"] > 0).sum())
            checked += 1
    assert checked >= 5


@gpu
def test_analyze_op_profile_c2_scale(ctx):
    """Full C2 (10M tokens): shared-memory cells == sort-path cells over the same tokens, and the
    per-iteration sums equal the rows' gap sums and span lengths."""
    from paper_1707_03750_b200 import cuda
    recs, info = synth.generate_config("C2")
    d = ctx.upload(recs)
    raw = ctx.analyze_raw(d, [synth.CONFIGS["C2"]["iterations"]], op_profile="cells")
    L = raw["loops"][0]
    cells = L["op_cells"]
    rows = L["rows"]
    wo, wi = reduce_cells(cells, raw["n_names"], rows.shape[0])
    assert np.array_equal(L["op_totals"], wo) and np.array_equal(L["iter_op_totals"], wi)
    raw2 = ctx.analyze_raw(d, [synth.CONFIGS["C2"]["iterations"]], op_profile=True)  # totals only
    assert len(raw2["loops"][0]["op_cells"]) == 0
    assert np.array_equal(raw2["loops"][0]["op_totals"], wo) and np.array_equal(raw2["loops"][0]["iter_op_totals"], wi)
    I = rows.shape[0]
    assert I == synth.CONFIGS["C2"]["iterations"]
    it = cells["iteration"].astype(np.int64)
    assert np.all(np.diff(it) >= 0)
    same = np.diff(it) == 0
    assert np.all(np.diff(cells["op"].astype(np.int64))[same] > 0)  # (iteration, op) order, no duplicates
    cnt = np.zeros(I, np.int64)
    idle = np.zeros(I, np.int64)
    np.add.at(cnt, it, cells["count"].astype(np.int64))
    np.add.at(idle, it, cells["idle_ns"])
    fi = cuda.ROW_FIELDS
    assert np.array_equal(cnt, rows[:, fi.index("end_token")] - rows[:, fi.index("start_token")] + 1)
    assert np.array_equal(idle, rows[:, fi.index("gap_sum")])
