"""GPU parity: the CUDA path (through the C-ABI) against the reference.

Bit-exact bar: SA, LCP, repeats, mined pattern (tokens/count/first_token/epsilon_used), error
kinds and messages, spans, token ids, stream census, integer per-iteration aggregates, and
the doubles derived from them (compared via float.hex()).  Oracles: the committed golden
fixtures (generated from the reference) and the compiled reference (oracle/_ref) live.
"""
from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import records_from_ops
from oracle.bindings import CheckerError
from paper_1707_03750_b200 import cuda, itertrace, synth

pytestmark = pytest.mark.gpu


def _mine(X, tokens, term, loops, multi):
    try:
        return {"ok": X.mine_patterns(tokens, term, [tuple(l) for l in loops], multi=multi)}
    except (cuda.IttError, CheckerError) as e:
        return {"error": e.kind, "message": str(e)}


# ---------------------------------------------------------------- token level (golden)
def test_golden_token_cases(ctx, token_cases):
    for c in token_cases:
        sa, lcp = ctx.suffix_array(c["tokens"], c["term"])
        assert sa.tolist() == c["sa"], c["name"]
        assert lcp.tolist() == c["lcp"], c["name"]
        for r in c["repeats"]:
            got = sorted(ctx.enumerate_repeats(c["tokens"], c["term"], r["min_count"], r["max_len"]))
            assert [list(x) for x in got] == r["out"], (c["name"], r)
        n_names = max(c["tokens"]) + 1
        for m in c["mine"]:
            got = _mine(ctx, c["tokens"], n_names, m["loops"], m["multi"])
            want = {k: m[k] for k in ("ok", "error", "message") if k in m}
            assert got == want, (c["name"], m["loops"])
        for m in c["match"]:
            assert ctx.approx_match(c["tokens"], m["pattern"], m["k0"]).tolist() == m["spans"], (c["name"], m)


def _random_string(rng, n, a, periodic):
    s = rng.integers(0, a, n)
    if periodic:
        per = rng.integers(0, a, int(rng.integers(1, max(2, min(n, 400)))))
        s = np.tile(per, n // len(per) + 1)[:n]
        s[rng.integers(0, n, int(rng.integers(0, 4)))] = a - 1  # sparse defects
    return s.astype(np.int32)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random_vs_reference(ctx, R, seed):
    rng = np.random.default_rng(seed)
    for trial in range(60):
        n = int(rng.integers(1, 6000)) if trial % 4 else int(rng.integers(1, 40))
        a = int(rng.integers(1, 300))
        s = _random_string(rng, n, a, trial % 2 == 0)
        sa, lcp = ctx.suffix_array(s, a)
        rsa, rlcp = R.suffix_array(s, a)
        assert np.array_equal(sa, rsa) and np.array_equal(lcp, rlcp), (seed, trial, n, a)
        mc, ml = int(rng.integers(2, 6)), int(rng.integers(1, 60))
        assert sorted(ctx.enumerate_repeats(s, a, mc, ml)) == sorted(R.enumerate_repeats(s, a, mc, ml))
        it = int(rng.integers(2, 80))
        assert _mine(ctx, s, a, [(it, 1)], False) == _mine(R, s, a, [(it, 1)], False), (seed, trial)
        assert _mine(ctx, s, a, [(it, 2), (it + 3, 1)], True) == _mine(R, s, a, [(it, 2), (it + 3, 1)], True)
        p = s[int(rng.integers(0, n)):][: int(rng.integers(1, 40))]
        k0 = int(rng.integers(0, 6))
        assert np.array_equal(ctx.approx_match(s, p, k0), R.approx_match(s, p, k0)), (seed, trial)


def test_alphabet_and_terminator_edge_cases(ctx, R):
    cases = [
        ([], 0), ([5], 6), ([5], -1), ([3] * 1000, 4), ([3] * 1000, -7), (list(range(2000)), 2000),
        (list(range(2000, 0, -1)), 0), ([7, 1 << 30, 7, 1 << 30, 7], 3), ([-5, -5, -2, -5, -5, -2], 0),
        ([1, 2] * 3000, 3), ([0, 0, 1] * 2000 + [2], 5),
    ]
    for s, term in cases:
        sa, lcp = ctx.suffix_array(s, term)
        rsa, rlcp = R.suffix_array(s, term)
        assert np.array_equal(sa, rsa) and np.array_equal(lcp, rlcp), (s[:10], term)
    with pytest.raises(cuda.IttError) as e:  # a terminator that occurs in the text is not unique
        ctx.suffix_array([1, 2, 3], 2)
    assert e.value.kind == "InvalidConfig"


def test_match_greedy_skip_semantics(ctx, R):
    rng = np.random.default_rng(606)  # test_match.cpp:78-102, with longer strings
    for _ in range(300):
        s = rng.integers(0, 4, int(rng.integers(1, 2000))).astype(np.int32)
        p = s[: int(rng.integers(1, 70))] if rng.integers(0, 2) else rng.integers(0, 4, int(rng.integers(1, 70)))
        k0 = int(rng.integers(0, 5))
        assert np.array_equal(ctx.approx_match(s, p, k0), R.approx_match(s, p, k0))
    # overlapping successes force the successor chain off the fast path
    s = np.array([1, 1, 2, 1, 2, 2] * 500, np.int32)
    for p, k0 in (([1, 2], 1), ([1, 1, 2], 2), ([1, 2, 2], 3)):
        assert np.array_equal(ctx.approx_match(s, p, k0), R.approx_match(s, p, k0))


# ---------------------------------------------------------------- records level
def test_row_order_fast_path_and_fallback(ctx, R):
    """(start,row) ordering: already sorted, locally shuffled (block fast path), globally shuffled
    (radix fallback), and heavy start ties across block boundaries (stability)."""
    rng = np.random.default_rng(21)
    n = 5000
    base = np.sort(rng.integers(0, 4000, n))  # many equal starts
    variants = {"sorted": base.copy()}
    loc = base.copy()
    for b in range(0, n, 64):
        seg = loc[b:b + 64].copy()
        rng.shuffle(seg)
        loc[b:b + 64] = seg
    variants["local"] = loc
    glob = base.copy()
    rng.shuffle(glob)
    variants["global"] = glob
    variants["ties"] = np.repeat(np.arange(n // 500), 500)[::-1].copy()
    # blocks spanning >= 2^24 ns take the 64-bit-key bitonic path, narrow ones the packed 32-bit
    # key: wide and mixed spans (incl. negative starts), locally shuffled
    wide = np.sort(rng.integers(-(1 << 40), 1 << 40, n))
    mixed = np.sort(np.concatenate([rng.integers(0, 3000, n // 2), rng.integers(1 << 30, 1 << 36, n - n // 2)]))
    for nm, arr in (("wide_local", wide), ("mixed_local", mixed)):
        v = arr.copy()
        for b in range(0, n, 64):
            seg = v[b:b + 64].copy()
            rng.shuffle(seg)
            v[b:b + 64] = seg
        variants[nm] = v
    for name, starts in variants.items():
        ops = [(13 if i % 3 else 14, "op%d" % (i % 17) if i % 3 else "[CUDA memcpy HtoD]", int(s), 3, 64, 1e9)
               for i, s in enumerate(starts)]
        recs = records_from_ops(ops)
        gt, gri, _ = ctx.build_token_sequence(recs, 13)
        rt, rri, _ = R.build_token_sequence(recs, 13)
        assert np.array_equal(gt, rt) and np.array_equal(gri, rri), name
        assert ctx.summarize_streams(recs)[0] == R.summarize_streams(recs)[0], name


def test_build_token_sequence_vs_reference(ctx, R):
    for kw in (dict(), dict(noise_frac=0.05, shuffle_window=64, seed=11), dict(minority_frac=0.1, seed=12),
               dict(vocab=2000, body_len=3000, iterations=20, seed=5)):
        recs, _ = synth.generate_config("C1", **kw)
        gt, gri, gn = ctx.build_token_sequence(recs, 13)
        rt, rri, rn = R.build_token_sequence(recs, 13)
        assert np.array_equal(gt, rt) and np.array_equal(gri, rri) and len(gn) == len(rn)
        for v in range(len(rn)):  # same name behind every id
            assert recs.name(int(gn[v])) == recs.name(int(rn[v]))
    with pytest.raises(cuda.IttError) as e:
        ctx.build_token_sequence(recs, 99)
    assert e.value.kind == "EmptyMainStream"


def test_long_names_staged_and_unstaged_intern_identically(ctx, R):
    """Warp groups whose names exceed the 4 KiB staging buffer hash from global memory; the same
    name must get the same id whichever path a record takes (and hash prefixes must not merge)."""
    rng = np.random.default_rng(5)
    long = ["L" * 300 + "#%d" % i for i in range(6)]
    short = ["k%d" % i for i in range(6)]
    prefix = ["L" * 300 + "#%d" % i + "x" for i in range(3)]  # share 303 bytes with long names
    ops, t = [], 0
    for blk in range(400):
        pool = long + prefix if blk % 3 == 0 else short + long[:2]
        for _ in range(32):
            ops.append((13, pool[int(rng.integers(0, len(pool)))], t, 5))
            t += 7
    recs = records_from_ops(ops)
    gt, gri, gn = ctx.build_token_sequence(recs, 13)
    rt, rri, rn = R.build_token_sequence(recs, 13)
    assert np.array_equal(gt, rt) and len(gn) == len(rn) == 15


def _adversarial_name_pool(rng):
    """Names of every length class the dictionary kernel splits on (0, < 16, chunk and 128-byte
    boundaries, > 128, > 300) and near-duplicates differing in one byte at the first, a chunk-edge,
    the middle and the last position, or by one extra byte (prefixes)."""
    pool = [""]
    for L in (1, 3, 4, 7, 8, 15, 16, 17, 31, 32, 33, 63, 64, 100, 127, 128, 129, 143, 144, 200, 255, 256, 257, 300, 520):
        base = bytes(rng.integers(33, 127, size=L, dtype=np.uint8)).decode()
        pool.append(base)
        pool.append(base + "x")
        for pos in {0, L // 2, L - 1, 15, 16, 127, 128, 129}:
            if 0 <= pos < L:
                ch = "A" if base[pos] != "A" else "B"
                pool.append(base[:pos] + ch + base[pos + 1:])
    return sorted(set(pool))


@pytest.mark.parametrize("force_collision", [False, True])
def test_dictionary_adversarial_names(ctx, R, force_collision, monkeypatch):
    """Exact dictionary on names built to break a hash-only scheme; with ITT_TEST_FORCE_COLLISION
    every name first lands in ONE slot, so the byte compares (copy, representative row, length)
    must catch every collision and the re-run must recover."""
    if force_collision:
        monkeypatch.setenv("ITT_TEST_FORCE_COLLISION", "1")
    rng = np.random.default_rng(77)
    pool = _adversarial_name_pool(rng)
    longs = [x for x in pool if len(x) > 200]
    ops, t = [], 0
    for blk in range(300):
        # some warp groups only long names (their bytes exceed the staging buffer), the rest mixed
        src = longs if blk % 5 == 0 else pool
        for _ in range(32 + int(rng.integers(0, 7))):  # ragged groups: every name alignment occurs
            ops.append((13, src[int(rng.integers(0, len(src)))], t, 5))
            t += 7
    recs = records_from_ops(ops)
    gt, gri, gn = ctx.build_token_sequence(recs, 13)
    rt, rri, rn = R.build_token_sequence(recs, 13)
    assert np.array_equal(gt, rt) and np.array_equal(gri, rri) and len(gn) == len(rn)


def test_token_replay_100k(ctx):
    # test_streams.cpp:204-225
    rng = np.random.default_rng(33)
    n = 100_000
    recs = records_from_ops([(13, "op%d" % int(rng.integers(0, 512)), i * 20, 10) for i in range(n)])
    tok, ri, names = ctx.build_token_sequence(recs, 13)
    replay = {}
    for i in range(n):
        assert tok[i] == replay.setdefault(recs.name(int(ri[i])), len(replay))


def test_summarize_streams_vs_reference(ctx, R):
    for kw in (dict(), dict(minority_frac=0.2, seed=3), dict(noise_frac=0.05, shuffle_window=64, seed=4),
               dict(extra_stream_frac=0.05, seed=6)):
        recs, _ = synth.generate_config("C1", **kw)
        for filt in (False, True):
            g, info = ctx.summarize_streams(recs, filt)
            r, dropped = R.summarize_streams(recs, filt)
            assert g == r and info["dropped"] == dropped, (kw, filt)
    assert ctx.count_interval_overlaps(records_from_ops([(13, "a", 0, 15), (13, "b", 10, 5)]), 13) == 1
    assert ctx.count_interval_overlaps(records_from_ops([(13, "a", 0, 5), (13, "b", 10, 5)]), 13) == 0


def _htod(start, dur, size):
    return (14, "[CUDA memcpy HtoD]", start, dur, size, 1e9)


def test_iteration_metrics_known_answers(ctx, R):
    cases = [
        ([(13, "a", 0, 10), (13, "b", 12, 8), _htod(25, 5, 1000), (13, "a", 35, 10), (13, "b", 47, 3)], [(0, 1, 0), (2, 3, 0)]),
        ([(13, "a", 0, 10), (13, "a", 30, 10)], [(0, 0, 0), (1, 1, 0)]),
        ([(13, "a", 0, 10), (13, "a", 10, 10)], [(0, 0, 0), (1, 1, 0)]),
        ([(13, "a", 0, 20), _htod(22, 8, 100), _htod(26, 8, 100), (13, "a", 40, 10)], [(0, 0, 0), (1, 1, 0)]),
        ([(13, "a", 0, 20), _htod(25, 100, 100), (13, "a", 40, 10)], [(0, 0, 0), (1, 1, 0)]),
        ([_htod(0, 2, 111), (13, "a", 10, 10), _htod(25, 5, 222), (13, "a", 40, 10), _htod(45, 5, 333), (13, "a", 60, 10),
          _htod(90, 5, 999)], [(0, 0, 0), (1, 1, 0), (2, 2, 0)]),
        ([(13, "a", 0, 10), (13, "b", 14, 6), (13, "c", 22, 8)], [(0, 2, 0)]),
        ([(13, "a", 0, 12), (13, "b", 10, 5)], [(0, 1, 0)]),
        # carry-in: a long copy that starts before the gap and covers it; negative interval
        ([(13, "a", 0, 50), _htod(5, 200, 7), (13, "a", 60, 10), (13, "b", 65, 30), (13, "a", 80, 5)],
         [(0, 0, 0), (1, 1, 0), (2, 3, 0)]),
    ]
    for ops, spans in cases:
        recs = records_from_ops(ops)
        _, ri, _ = ctx.build_token_sequence(recs, 13)
        rows, clamps = ctx.iteration_metrics(recs, ri, spans)
        rrows, rclamps = R.iteration_metrics(recs, 13, spans)
        assert clamps == rclamps, ops
        for g, r in zip(rows, rrows):
            m = itertrace.rows_to_metrics([[g.start_token, g.end_token, g.extra, g.t_start, g.t_end, g.interval_ns,
                                            g.copy_ns, g.htod_bytes, g.gap_sum, g.gap_count, g.has_interval]])[0]
            assert (m.t_start, m.t_end, m.htod_bytes) == (r.t_start, r.t_end, r.htod_bytes)
            assert (m.interval_ns is not None) == bool(r.has_interval) and (m.interval_ns or 0) == r.interval_ns
            assert (m.overlap_ratio is not None) == bool(r.has_overlap)
            if m.overlap_ratio is not None:
                assert m.overlap_ratio.hex() == float(r.overlap_ratio).hex()
            assert m.op_gap_mean_ns.hex() == float(r.op_gap_mean_ns).hex()


# ---------------------------------------------------------------- end to end (golden traces)
def test_golden_traces_end_to_end(ctx, trace_cases):
    for c in trace_cases:
        recs, info = synth.generate(**c["generator"])
        assert info == c["info"]
        o = c["opts"]
        try:
            r = itertrace.analyze_trace(ctx, recs, c["loops"], epsilon0=o.get("epsilon0", 1), k0=o.get("k0"),
                                        main_stream=o.get("main_stream"))
        except itertrace.AnalyzeError as e:
            assert (e.kind, str(e)) == (c.get("error"), c.get("message")), c["name"]
            continue
        assert "error" not in c, (c["name"], c.get("error"))
        assert [list(s[:2]) + [list(s[2])] + list(s[3:]) for s in r.streams] == c["streams"], c["name"]
        assert r.main_stream == c["main_stream"] and r.warnings == c["warnings"], c["name"]
        for L, G, items in zip(r.loops, c["loops_out"], r.details):
            assert (L.pattern_length, L.pattern_count, L.epsilon_used, L.first_occurrence_token, L.k0_used) == \
                (G["pattern_length"], G["pattern_count"], G["epsilon_used"], G["first_token"], G["k0_used"]), c["name"]
            assert len(items) == len(G["iters"])
            for m, x in zip(items, G["iters"]):
                assert [m.index, m.start_token, m.end_token, m.extra_ops, m.t_start, m.t_end] == x[:6]
                assert (m.interval_ns is not None) == bool(x[8]) and (m.interval_ns or 0) == x[6]
                assert m.htod_bytes == x[7]
                assert (m.overlap_ratio is not None) == bool(x[9])
                if m.overlap_ratio is not None:
                    assert m.overlap_ratio.hex() == x[10]
                assert m.op_gap_mean_ns.hex() == x[11]
        assert r.summary_json() == c["summary_json"], c["name"]
        assert r.details_csv(0) == c["details_csv"], c["name"]


def test_live_reference_end_to_end_random_configs(ctx, R):
    rng = np.random.default_rng(1003)  # acceptance.cpp:164-184 style sweep, on the TF-like generator
    for i in range(12):
        kw = dict(seed=77_000 + i, iterations=int(rng.integers(20, 400)), body_len=int(rng.integers(5, 120)),
                  vocab=int(rng.integers(3, 100)), init_ops=int(rng.integers(1, 20)),
                  noise_frac=float(rng.choice([0.0, 0.05])), shuffle_window=int(rng.choice([0, 16])),
                  body_inserts=int(rng.integers(0, 3)), insert_prob=float(rng.random() * 0.3))
        recs, _ = synth.generate(**kw)
        loops = [kw["iterations"]]
        try:
            r = itertrace.analyze_trace(ctx, recs, loops)
            got = (r.summary_json(), r.details_csv(0))
        except itertrace.AnalyzeError as e:
            got = (e.kind, str(e))
        try:
            ref = R.analyze(recs, loops)
            want = (ref["summary_json"], ref["details_csv"])
        except CheckerError as e:
            want = (e.kind, str(e))
        assert got == want, kw


def test_device_resident_inputs_match_host_inputs(ctx):
    recs, _ = synth.generate_config("C1", noise_frac=0.05, shuffle_window=64, seed=8)
    d = ctx.upload(recs)
    try:
        a = ctx.analyze_raw(recs, [100])
        b = ctx.analyze_raw(d, [100])
    finally:
        d.free()
    assert a["streams"] == b["streams"] and a["name_row"] == b["name_row"]
    assert np.array_equal(a["loops"][0]["rows"], b["loops"][0]["rows"])


def test_pinned_host_columns_match_device(ctx):
    """Pinned (registered) host columns: the size column is read in place by the compaction (zero-
    copy, HtoD rows only) instead of being copied — the per-iteration HtoD bytes must not change."""
    recs, _ = synth.generate_config("C1", noise_frac=0.05, shuffle_window=64, seed=9)
    d = ctx.upload(recs)
    cols = [recs.start_ns, recs.duration_ns, recs.size_bytes, recs.flags, recs.stream, recs.name_off, recs.name_bytes]
    for a in cols:
        ctx.register_host(a)
    try:
        a = ctx.analyze_raw(recs, [100])
        b = ctx.analyze_raw(d, [100])
    finally:
        for x in cols:
            ctx.unregister_host(x)
        d.free()
    assert np.array_equal(a["loops"][0]["rows"], b["loops"][0]["rows"])
    assert a["loops"][0]["rows"][:, 7].sum() > 0  # HtoD bytes present: the in-place sizes were read


@pytest.mark.parametrize("shuffle", [0, 64])
def test_late_durations_match_device(ctx, shuffle, monkeypatch):
    """Large pinned host traces send the duration column last over PCIe (after the streamed names)
    and fill stream ends, token ends and HtoD ends after the suffix array: census (last_end),
    overlapping kernels, per-iteration rows and the op profile must equal the device-resident
    call.  ITT_TEST_OVERLAP_MIN lowers the 256 MiB name threshold to this small trace; shuffled
    rows take the compaction path that waits for the copy instead."""
    monkeypatch.setenv("ITT_TEST_OVERLAP_MIN", "1")
    monkeypatch.setenv("ITT_STREAM_CHUNK", "65536")
    recs, _ = synth.generate_config("C1", noise_frac=0.05, shuffle_window=shuffle, seed=11, minority_frac=0.02)
    d = ctx.upload(recs)
    cols = [recs.start_ns, recs.duration_ns, recs.size_bytes, recs.flags, recs.stream, recs.name_off, recs.name_bytes]
    if recs.device is not None:
        cols.append(recs.device)
    for a in cols:
        ctx.register_host(a)
    from paper_1707_03750_b200 import abi
    try:
        a = ctx.analyze_raw(recs, [100], op_profile=True)
        recs.mem = abi.MEM_HOST_STREAM_NAMES  # streamed names: the same two-stream column copy
        try:
            s = ctx.analyze_raw(recs, [100], op_profile=True)
        finally:
            recs.mem = abi.MEM_HOST
        b = ctx.analyze_raw(d, [100], op_profile=True)
    finally:
        for x in cols:
            ctx.unregister_host(x)
        d.free()
    for x in (a, s):
        assert x["streams"] == b["streams"]
        assert x["overlapping_kernels"] == b["overlapping_kernels"]
        assert x["name_row"] == b["name_row"] and x["dropped"] == b["dropped"]
        assert x["loops"][0]["pattern_tokens"] == b["loops"][0]["pattern_tokens"]
        assert np.array_equal(x["loops"][0]["rows"], b["loops"][0]["rows"])
        assert np.array_equal(x["loops"][0]["op_totals"], b["loops"][0]["op_totals"])
    assert a["loops"][0]["rows"][:, 7].sum() > 0  # HtoD rows: their ends came from the late pass


@pytest.mark.parametrize("chunk", [None, "4096", "200000"])
def test_streamed_host_names_match_copied_names(ctx, chunk, monkeypatch):
    """ITT_MEM_HOST_STREAM_NAMES / ITT_MEM_DEVICE_HOST_NAMES: names streamed through bounded
    device windows (the C5 layout) — identical results, with many chunks (ITT_STREAM_CHUNK) so
    representatives from earlier chunks are verified from the arena."""
    from paper_1707_03750_b200 import abi
    if chunk:
        monkeypatch.setenv("ITT_STREAM_CHUNK", chunk)
    recs, _ = synth.generate_config("C1", noise_frac=0.05, shuffle_window=64, seed=9, name_max=160,
                                    minority_frac=0.02)
    a = ctx.analyze_raw(recs, [100], op_profile=True)
    recs.mem = abi.MEM_HOST_STREAM_NAMES
    try:
        b = ctx.analyze_raw(recs, [100], op_profile=True)
    finally:
        recs.mem = abi.MEM_HOST
    d = ctx.upload(recs, names_host=True)
    try:
        e = ctx.analyze_raw(d, [100], op_profile=True)
    finally:
        d.free()
    for x in (b, e):
        assert a["streams"] == x["streams"] and a["name_row"] == x["name_row"]
        assert a["loops"][0]["pattern_tokens"] == x["loops"][0]["pattern_tokens"]
        assert np.array_equal(a["loops"][0]["rows"], x["loops"][0]["rows"])
        assert np.array_equal(a["loops"][0]["op_totals"], x["loops"][0]["op_totals"])


def test_native_batch_executor_matches_single_trace_calls(ctx):
    """itt_batch_* (C4's executor): C++ worker threads with their own contexts give the same
    per-trace results as one-at-a-time itt_analyze, including per-trace errors."""
    from paper_1707_03750_b200 import batch
    traces = [synth.generate(iterations=20 + t % 5, body_len=15 + t % 4, vocab=12, seed=500 + t)[0] for t in range(24)]
    traces.append(records_from_ops([(13, "k", 0, 5)]))  # one token: mining fails for this trace
    ex = cuda.Batch(0, 4)
    try:
        got = ex.analyze(traces, [20], summarize=batch.summarize_c)
        assert ex.launch_count() > 0
    finally:
        ex.close()
    for t, g in zip(traces, got):
        try:
            want = batch.summarize(ctx.analyze_raw(t, [20]))
        except cuda.IttError as e:
            assert isinstance(g, cuda.IttError) and g.status == e.status and str(g) == str(e)
            continue
        assert g == want


def test_narrow_rank_levels(ctx, R):
    """u16 rank levels (used where the arrays outgrow L2; forced here for small inputs), including
    the fallback to u32 when a level's group count passes 2^16 (random strings)."""
    import os
    rng = np.random.default_rng(77)
    old = os.environ.get("ITT_NARROW_MIN_N")
    os.environ["ITT_NARROW_MIN_N"] = "0"
    try:
        for n, V in ((3000, 5), (20_000, 3), (150_000, 1000), (90_000, 2)):
            s = rng.integers(0, V, n).tolist()
            sa, lcp = ctx.suffix_array(s, V)
            rsa, rlcp = R.suffix_array(s, V)
            assert np.array_equal(sa, rsa) and np.array_equal(lcp, rlcp), (n, V)
        body = rng.integers(0, 40, 97).tolist()
        tok = np.array((body * 400)[:38_000], np.int32)
        assert ctx.mine_patterns(tok, 40, [(390, 1)]) == R.mine_patterns(tok, 40, [(390, 1)])
    finally:
        if old is None:
            os.environ.pop("ITT_NARROW_MIN_N", None)
        else:
            os.environ["ITT_NARROW_MIN_N"] = old
