"""CPU: pin the C restatement (oracle/itt_oracle.c) to the reference.

Three sources of truth, all reference-derived:
  * the committed golden fixtures (tests/golden/*.json, generated from oracle/_ref);
  * the reference's own known-answer tests (test_suffix_tree.cpp, test_mine.cpp,
    test_match.cpp, test_metrics.cpp, test_streams.cpp), restated here;
  * the compiled reference itself (oracle/_ref) on seeded random inputs.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import records_from_ops
from oracle.bindings import CheckerError
from paper_1707_03750_b200 import synth


def _mine(X, tokens, loops, multi):
    n_names = max(tokens) + 1 if len(tokens) else 0
    try:
        return {"ok": X.mine_patterns(tokens, n_names, [tuple(l) for l in loops], multi=multi)}
    except CheckerError as e:
        return {"error": e.kind, "message": str(e)}


def test_oracle_matches_golden_token_cases(O, token_cases):
    for c in token_cases:
        sa, lcp = O.suffix_array(c["tokens"], c["term"])
        assert sa.tolist() == c["sa"], c["name"]
        assert lcp.tolist() == c["lcp"], c["name"]
        for r in c["repeats"]:
            got = sorted(O.enumerate_repeats(c["tokens"], c["term"], r["min_count"], r["max_len"]))
            assert [list(x) for x in got] == r["out"], (c["name"], r)
        for m in c["mine"]:
            got = _mine(O, c["tokens"], m["loops"], m["multi"])
            want = {k: m[k] for k in ("ok", "error", "message") if k in m}
            assert got == want, (c["name"], m["loops"])
        for m in c["match"]:
            assert O.approx_match(c["tokens"], m["pattern"], m["k0"]).tolist() == m["spans"], (c["name"], m)


def test_oracle_matches_reference_random(O, R):
    rng = np.random.default_rng(4242)
    for trial in range(120):
        n = int(rng.integers(1, 300))
        a = int(rng.integers(1, 6))
        s = rng.integers(0, a, n).astype(np.int32)
        if trial % 3 == 0:
            per = rng.integers(0, a, int(rng.integers(1, 8)))
            s = np.tile(per, n // len(per) + 1)[:n].astype(np.int32)
        sa1, l1 = R.suffix_array(s, a)
        sa2, l2 = O.suffix_array(s, a)
        assert np.array_equal(sa1, sa2) and np.array_equal(l1, l2)
        mc, ml = int(rng.integers(2, 5)), int(rng.integers(1, 12))
        assert sorted(R.enumerate_repeats(s, -1, mc, ml)) == sorted(O.enumerate_repeats(s, -1, mc, ml))
        it = int(rng.integers(2, 8))
        assert _mine(R, s.tolist(), [(it, 1)], False) == _mine(O, s.tolist(), [(it, 1)], False)
        p = s[: int(rng.integers(1, 6))]
        k0 = int(rng.integers(0, 3))
        assert np.array_equal(R.approx_match(s, p, k0), O.approx_match(s, p, k0))


# ---------------------------------------------------------------- reference known answers
def test_banana_suffix_order_and_repeats(O):
    # test_suffix_tree.cpp:34-45 and test_mine.cpp:50-84 (terminator -1)
    tok = [ord(c) for c in "banana"]
    sa, lcp = O.suffix_array(tok, -1)
    assert len(sa) == 7  # 7 leaves
    assert sorted(O.enumerate_repeats(tok, -1, 2, 10)) == sorted([(1, 1, 3), (1, 3, 2), (2, 2, 2)])  # a, ana, na
    got = {(tuple(tok[s:s + l]), c) for s, l, c in O.enumerate_repeats(tok, -1, 2, 2)}
    assert got == {((ord("a"),), 3), ((ord("n"), ord("a")), 2), ((ord("a"), ord("n")), 2)}
    assert O.enumerate_repeats(tok, -1, 99, 10) == []


def test_mine_known_answers(O):
    # test_mine.cpp:114-165
    p = O.mine_patterns([900, 901, 1, 2, 3, 1, 2, 3, 1, 2, 3], 902, [(3, 1)])[0]
    assert p == {"tokens": [1, 2, 3], "count": 3, "first_token": 2, "epsilon_used": 1}
    assert O.mine_patterns([1, 2, 1, 2, 1, 2], 3, [(3, 1)])[0]["tokens"] == [1]
    body = [1000 + i for i in range(30)] + [1, 2, 3] * 7
    p = O.mine_patterns(body, 1030, [(10, 1)])[0]
    assert (p["tokens"], p["count"], p["epsilon_used"]) == ([1, 2, 3], 7, 4)
    with pytest.raises(CheckerError) as e:
        O.mine_patterns([1, 2, 3, 4, 5, 6], 7, [(3, 1)])
    assert e.value.kind == "NoPatternFound"
    for iters in (3, 1):
        with pytest.raises(CheckerError) as e:
            O.mine_patterns([1, 2], 3, [(iters, 1)])
        assert e.value.kind == "InvalidIterationCount"
    two = [10, 11] * 50 + [20, 21, 22] * 20
    ps = O.mine_patterns(two, 23, [(50, 1), (20, 1)], multi=True)
    assert [(p["tokens"], p["count"]) for p in ps] == [([10, 11], 50), ([20, 21, 22], 20)]
    with pytest.raises(CheckerError) as e:
        O.mine_patterns([1000, 1001] + [1, 2, 3] * 10, 1002, [(10, 1), (10, 1)], multi=True)
    assert e.value.kind == "InvalidConfig"
    with pytest.raises(CheckerError) as e:
        O.mine_patterns([1000 + i for i in range(40)] + [1, 2, 3] * 10, 1040, [(10, 1), (11, 1)], multi=True)
    assert e.value.kind == "AmbiguousLoops"


def test_match_known_answers(O):
    # test_match.cpp:21-76
    assert O.approx_match([1, 2, 3, 1, 2, 9, 3, 1, 2, 3], [1, 2, 3], 1).tolist() == [[0, 2, 0], [3, 6, 1], [7, 9, 0]]
    assert O.approx_match([4, 5, 6, 7], [4, 5, 6, 7], 0).tolist() == [[0, 3, 0]]
    assert O.approx_match([1, 9, 9, 2, 9, 9, 3], [1, 2, 3], 1).tolist() == []


def test_default_k0_table():
    # test_match.cpp:186-192; default_k0 = (l + 3) / 4 (match.hpp:19-21)
    assert [(l + 3) // 4 for l in (1, 4, 5, 8, 9)] == [1, 1, 2, 2, 3]


def _htod(start, dur, size):
    return (14, "[CUDA memcpy HtoD]", start, dur, size, 1e9)


def _metrics(X, ops, spans):
    recs = records_from_ops(ops)
    rows, clamps = X.iteration_metrics(recs, 13, spans)
    return rows, clamps


@pytest.mark.parametrize("use_ref", [False, True])
def test_metrics_known_answers(O, R, use_ref):
    X = R if use_ref else O
    # interval 15, overlap 5/15, bytes 1000 (test_metrics.cpp:65-91)
    rows, _ = _metrics(X, [(13, "a", 0, 10), (13, "b", 12, 8), _htod(25, 5, 1000), (13, "a", 35, 10), (13, "b", 47, 3)],
                       [(0, 1, 0), (2, 3, 0)])
    assert not rows[0].has_interval and not rows[0].has_overlap
    assert rows[1].interval_ns == 15 and rows[1].overlap_ratio == 5.0 / 15.0 and rows[1].htod_bytes == 1000
    # zero overlap vs absent (test_metrics.cpp:93-119)
    rows, _ = _metrics(X, [(13, "a", 0, 10), (13, "a", 30, 10)], [(0, 0, 0), (1, 1, 0)])
    assert rows[1].has_overlap and rows[1].overlap_ratio == 0.0
    rows, _ = _metrics(X, [(13, "a", 0, 10), (13, "a", 10, 10)], [(0, 0, 0), (1, 1, 0)])
    assert rows[1].has_interval and rows[1].interval_ns == 0 and not rows[1].has_overlap
    # union 12/20 and clipping 15/20 (test_metrics.cpp:121-151)
    rows, _ = _metrics(X, [(13, "a", 0, 20), _htod(22, 8, 100), _htod(26, 8, 100), (13, "a", 40, 10)], [(0, 0, 0), (1, 1, 0)])
    assert rows[1].overlap_ratio == 12.0 / 20.0
    rows, _ = _metrics(X, [(13, "a", 0, 20), _htod(25, 100, 100), (13, "a", 40, 10)], [(0, 0, 0), (1, 1, 0)])
    assert rows[1].overlap_ratio == 15.0 / 20.0
    # byte attribution 111 / 555 / 0 (test_metrics.cpp:153-176)
    rows, _ = _metrics(X, [_htod(0, 2, 111), (13, "a", 10, 10), _htod(25, 5, 222), (13, "a", 40, 10), _htod(45, 5, 333),
                           (13, "a", 60, 10), _htod(90, 5, 999)], [(0, 0, 0), (1, 1, 0), (2, 2, 0)])
    assert [r.htod_bytes for r in rows] == [111, 555, 0]
    # op-gap mean 3.0 and the negative clamp counter (test_metrics.cpp:178-202)
    rows, _ = _metrics(X, [(13, "a", 0, 10), (13, "b", 14, 6), (13, "c", 22, 8)], [(0, 2, 0)])
    assert rows[0].op_gap_mean_ns == 3.0
    rows, clamps = _metrics(X, [(13, "a", 0, 12), (13, "b", 10, 5)], [(0, 1, 0)])
    assert rows[0].op_gap_mean_ns == 0.0 and clamps[0] == 1


def test_streams_known_answers(O, R):
    # first-appearance ids (test_streams.cpp:180-186) and the 100K replay (test_streams.cpp:204-225)
    recs = records_from_ops([(13, "A", 0, 10), (13, "B", 10, 10), (13, "A", 20, 10)])
    tok, ri, names = O.build_token_sequence(recs, 13)
    assert tok.tolist() == [0, 1, 0] and len(names) == 2
    rng = np.random.default_rng(33)
    n = 100_000
    ops = [(13, "op%d" % int(rng.integers(0, 512)), i * 20, 10) for i in range(n)]
    recs = records_from_ops(ops)
    tok, ri, names = O.build_token_sequence(recs, 13)
    replay = {}
    for i in range(n):
        nm = recs.name(int(ri[i]))
        want = replay.setdefault(nm, len(replay))
        assert tok[i] == want
    rt, rri, rn = R.build_token_sequence(recs, 13)
    assert np.array_equal(rt, tok) and np.array_equal(rri, ri)


def test_oracle_matches_golden_traces(O, trace_cases):
    for c in trace_cases:
        recs, info = synth.generate(**c["generator"])
        assert info == c["info"], c["name"]  # the generator is deterministic across machines
        tok, ri, names = O.build_token_sequence(recs, 13)
        sha = int(np.bitwise_xor.reduce(tok.astype(np.uint64) * np.arange(1, tok.size + 1, dtype=np.uint64)))
        assert (tok.size, names.size, sha) == (c["n_tokens"], c["n_names"], c["tokens_sha"]), c["name"]
        if "loops_out" not in c or c["opts"].get("main_stream") is not None or c["generator"].get("minority_frac"):
            continue
        L = c["loops_out"][0]
        spans = [(it[1], it[2], it[3]) for it in L["iters"]]
        rows, _ = O.iteration_metrics(recs, 13, spans)
        for r, it in zip(rows, L["iters"]):
            assert (r.t_start, r.t_end, r.htod_bytes) == (it[4], it[5], it[7])
            assert float(r.op_gap_mean_ns).hex() == it[11]
            if r.has_overlap:
                assert float(r.overlap_ratio).hex() == it[10]


def test_classifier_precedence(O):
    # trace.hpp:103-113 / test_trace.cpp:9-45
    K = O.classify
    assert K(b"[CUDA memcpy HtoD]", True) == 1 and K(b"[CUDA memcpy DtoH]", True) == 2
    assert K(b"[CUDA MEMCPY dtod]", False) == 3 and K(b"[CUDA memset]", True) == 4
    assert K(b"volta_sgemm", False) == 0 and K(b"volta_sgemm", True) == 5
    assert K(b"memcpy_kernel_htod_memset", False) == 1  # copy marker wins over memset
    assert K(b"memcpyish", False) == 0 and K(b"", False) == 0
