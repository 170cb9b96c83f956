"""GPU parity at BASELINE sizes through size-independent properties (the CPU reference is too
slow at 10M tokens: its metrics stage alone is O(I*H)).

  * SA: a permutation, and sorted by the O(n) Burkhardt-Karkkainen test
    (t[SA[k-1]], ISA[SA[k-1]+1]) < (t[SA[k]], ISA[SA[k]+1]);
  * LCP: direct comparison on sampled adjacent pairs (mismatch right after LCP symbols);
  * mining: the mined period is the planted body, count = I, first occurrence after the init
    prefix, spans = the planted iterations;
  * aggregates: sampled iterations recomputed by brute force with the reference's definitions
    (metrics.hpp:109-164) over ALL HtoD records, doubles compared bit for bit.
"""
from __future__ import annotations

import numpy as np
import pytest

from paper_1707_03750_b200 import itertrace, synth

pytestmark = pytest.mark.gpu


def _sorted_view(recs):
    order = np.lexsort((np.arange(recs.n), recs.start_ns))  # (start, row) — ingest.hpp:396-400
    return order


def _check_sa(ctx, tokens, term, rng, n_lcp_samples=40):
    sa, lcp = ctx.suffix_array(tokens, term)
    n = tokens.size
    np_ = n + 1
    assert np.array_equal(np.sort(sa), np.arange(np_, dtype=np.uint32))
    text = np.empty(np_, np.int64)
    text[:n] = tokens
    text[n] = term
    isa = np.empty(np_ + 1, np.int64)
    isa[sa.astype(np.int64)] = np.arange(np_)
    isa[np_] = -1
    a, b = sa[:-1].astype(np.int64), sa[1:].astype(np.int64)
    ta, tb = text[a], text[b]
    ra, rb = isa[a + 1], isa[b + 1]
    assert np.all((ta < tb) | ((ta == tb) & (ra < rb)))
    assert lcp[0] == 0
    for k in rng.integers(1, np_, n_lcp_samples):
        l = int(lcp[k])
        x, y = int(sa[k - 1]), int(sa[k])
        assert np.array_equal(text[x:x + l], text[y:y + l])
        assert x + l >= np_ or y + l >= np_ or text[x + l] != text[y + l]
    return sa, lcp


def _brute_metrics(recs, order, tok_rows, htod_rows, spans, ks):
    start = recs.start_ns[order]
    end = start + recs.duration_ns[order]
    ts, te = start[tok_rows], end[tok_rows]
    hs, he = start[htod_rows], end[htod_rows]
    hz = np.where(recs.flags[order][htod_rows] & 1, recs.size_bytes[order][htod_rows], 0)
    out = {}
    for k in ks:
        s, e, x = spans[k]
        t0, t1 = int(ts[s]), int(te[e])
        row = {"t": (t0, t1)}
        if k > 0:
            lo = int(te[spans[k - 1][1]])
            iv = max(0, t0 - lo)
            row["interval"] = iv
            if iv > 0:
                a = np.maximum(hs, lo)
                b = np.minimum(he, t0)
                m = b > a
                segs = sorted(zip(a[m].tolist(), b[m].tolist()))
                tot, cl, ch, op = 0, 0, 0, False
                for p, q in segs:
                    if not op or p > ch:
                        if op:
                            tot += ch - cl
                        cl, ch, op = p, q, True
                    else:
                        ch = max(ch, q)
                if op:
                    tot += ch - cl
                row["overlap"] = float(tot) / float(iv)
        lo_b = int(te[spans[k - 1][1]]) if k > 0 else -1
        row["bytes"] = int(hz[(hs > lo_b) & (hs <= t1)].sum())
        g = ts[s + 1:e + 1] - te[s:e]
        row["gap"] = float(np.maximum(g, 0).sum()) / float(e - s) if e > s else 0.0
        out[k] = row
    return out


@pytest.mark.parametrize("config", ["C2", "C3-lite"])
def test_full_size_properties(ctx, config):
    rng = np.random.default_rng(7)
    if config == "C2":
        recs, info = synth.generate_config("C2")
        iters, body_len, init = 50_000, 200, 16
    else:  # V = 4096, 5000-op body (the C3 shape at 2,000 iterations = 10M tokens)
        recs, info = synth.generate_config("C3", iterations=2_000)
        iters, body_len, init = 2_000, 5_000, 16
    tokens, ri, names = ctx.build_token_sequence(recs, 13)
    assert tokens.size == info["n_main"] == init + iters * body_len
    # first appearance: ids are 0..V-1 in order of first use
    first = np.unique(tokens, return_index=True)[1]
    assert np.array_equal(np.argsort(first), np.arange(names.size))
    _check_sa(ctx, tokens, int(names.size), rng)

    r = itertrace.analyze_trace(ctx, recs, [iters])
    L = r.loops[0]
    assert (L.pattern_length, L.pattern_count, L.first_occurrence_token, L.epsilon_used) == (body_len, iters, init, 1)
    assert L.pattern_tokens == tokens[init:init + body_len].tolist()
    items = r.details[0]
    assert len(items) == iters
    starts = np.array([m.start_token for m in items])
    ends = np.array([m.end_token for m in items])
    assert np.array_equal(starts, init + body_len * np.arange(iters))
    assert np.array_equal(ends, starts + body_len - 1)
    assert all(m.extra_ops == 0 for m in items)

    order = _sorted_view(recs)
    srt_stream = recs.stream[order]
    tok_rows = np.nonzero(srt_stream == 13)[0]
    names_sorted = [recs.name(int(i)) for i in order[:1]]  # noqa: F841 (keeps the view warm)
    htod_mask = np.array([b"memcpy htod" in recs.name(int(i)).lower() for i in order[np.nonzero(srt_stream != 13)[0]]])
    htod_rows = np.nonzero(srt_stream != 13)[0][htod_mask]
    spans = [(m.start_token, m.end_token, m.extra_ops) for m in items]
    ks = sorted(set([0, 1, iters - 1] + rng.integers(0, iters, 60).tolist()))
    want = _brute_metrics(recs, order, tok_rows, htod_rows, spans, ks)
    for k in ks:
        m, w = items[k], want[k]
        assert (m.t_start, m.t_end) == w["t"], k
        assert m.interval_ns == w.get("interval"), k
        assert (m.overlap_ratio is None) == ("overlap" not in w)
        if m.overlap_ratio is not None:
            assert m.overlap_ratio.hex() == w["overlap"].hex(), k
        assert m.htod_bytes == w["bytes"], k
        assert m.op_gap_mean_ns.hex() == w["gap"].hex(), k


def test_repeated_runs_are_deterministic(ctx):
    recs, _ = synth.generate_config("C2", iterations=5_000)
    a = ctx.analyze_raw(recs, [5_000])
    b = ctx.analyze_raw(recs, [5_000])
    assert a["name_row"] == b["name_row"] and a["streams"] == b["streams"]
    assert np.array_equal(a["loops"][0]["rows"], b["loops"][0]["rows"])


def test_c2_host_columns_overlapped_upload_matches_resident(ctx):
    """Large host inputs take the overlapped upload (columns on the copy stream, names streamed in
    64 MiB chunks into the hash pass): same analysis as device-resident columns."""
    recs, info = synth.generate_config("C2")
    d = ctx.upload(recs)
    try:
        want = ctx.analyze_raw(d, [50_000], op_profile=True)
    finally:
        d.free()
    got = ctx.analyze_raw(recs, [50_000], op_profile=True)
    assert got["streams"] == want["streams"] and got["name_row"] == want["name_row"]
    a, b = got["loops"][0], want["loops"][0]
    assert a["pattern_tokens"] == b["pattern_tokens"] and np.array_equal(a["rows"], b["rows"])
    assert np.array_equal(a["op_totals"], b["op_totals"])
