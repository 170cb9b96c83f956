"""Bit-exact parity at BASELINE scale (the north star's "bit-exact vs the CPU reference on every
config").

* C2 (10.6M events) and C3 (100M events, V = 4096): the device path's outputs are hashed and
  compared with SHA-256 digests of what the UNMODIFIED reference produced on the same generated
  trace (tests/golden/baseline_digests.json, made in the CPU container by
  tests/golden/make_baseline_digests.py through oracle/_ref/ref_digest):
    - analyze_trace (pipeline.hpp:34-134): summary JSON exactly as the CLI writes it
      (report.hpp:304) and the details CSV (report.hpp:191-220), plus the pattern integers;
    - build_token_sequence (streams.hpp:147-169): the main-stream token ids;
    - the full suffix array (SuffixTree leaf order, suffix_tree.hpp:21-190) and its LCP (Kasai).
* C5 (1B events): the reference's tree does not fit this container (~400 B per token), so:
    - itt_suffix_array (full SA, 1,000,000,017 suffixes) is checked by the O(n)
      Burkhardt-Karkkainen test, on the device (torch as the checker);
    - the token ids equal the planted structure (16 init ids, then the mined body 500,000 times);
    - analyze finds the planted period and spans; sampled iterations are recomputed by brute force
      with the reference's definitions (metrics.hpp:109-164), doubles compared bit for bit.
The generator is deterministic (libitt_synth.so), so the box regenerates the same traces.
"""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

from paper_1707_03750_b200 import itertrace, synth

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
DIGESTS = os.path.join(HERE, "golden", "baseline_digests.json")


def _sha(b) -> str:
    return hashlib.sha256(b).hexdigest()


def _digests(config):
    with open(DIGESTS) as f:
        d = json.load(f)
    if config not in d:
        pytest.fail(f"{config} digests missing: run tests/golden/make_baseline_digests.py {config}")
    return d[config]


def _full_vs_reference(ctx, config):
    d = _digests(config)
    a, s = d["analyze"], d["sa"]
    iters = d["generator"]["iterations"]
    recs, info = synth.generate_config(config)
    assert info["n"] == a["events"]
    r = itertrace.analyze_trace(ctx, recs, [iters])
    L = r.loops[0]
    assert (L.pattern_length, L.pattern_count, L.epsilon_used, L.first_occurrence_token, L.k0_used,
            L.iterations_found) == (a["pattern_length"], a["pattern_count"], a["epsilon_used"], a["first_token"],
                                    a["k0_used"], a["iterations_found"])
    got = r.summary_json()
    assert got == a["summary_json"]  # readable diff on failure
    assert _sha(got.encode()) == a["summary_json_sha256"]
    csv = r.details_csv(0).encode()
    assert len(csv) == a["details_csv_bytes"]
    assert _sha(csv) == a["details_csv_sha256"]
    # token ids, then the full suffix array and LCP of tokens + [V]
    tokens, _, names = ctx.build_token_sequence(recs, s["main_stream"])
    assert tokens.size == s["tokens"] and names.size == s["terminator"]
    assert _sha(tokens.tobytes()) == s["tokens_i32_sha256"]
    sa, lcp = ctx.suffix_array(tokens, int(names.size))
    assert _sha(sa.tobytes()) == s["sa_u32_sha256"]
    assert _sha(lcp.tobytes()) == s["lcp_u32_sha256"]


def test_c2_full_vs_reference(ctx):
    _full_vs_reference(ctx, "C2")


def test_c3_full_vs_reference(ctx):
    _full_vs_reference(ctx, "C3")


def _bk_check_device(sa_t, text_t):
    """Burkhardt-Karkkainen: SA is a permutation of [0, n') and for every k
    (t[SA[k-1]], ISA[SA[k-1]+1]) < (t[SA[k]], ISA[SA[k]+1]) (ISA[n'] = -1).  int32 tensors on the GPU."""
    import torch
    np_ = sa_t.numel()
    isa = torch.full((np_ + 1,), -1, dtype=torch.int32, device=sa_t.device)
    step = 1 << 27
    for lo in range(0, np_, step):
        hi = min(np_, lo + step)
        isa[sa_t[lo:hi].long()] = torch.arange(lo, hi, dtype=torch.int32, device=sa_t.device)
    assert int((isa[:np_] < 0).sum()) == 0, "SA is not a permutation"
    for lo in range(1, np_, step):
        hi = min(np_, lo + step)
        a = sa_t[lo - 1:hi - 1].long()
        b = sa_t[lo:hi].long()
        ta, tb = text_t[a], text_t[b]
        ra, rb = isa[a + 1], isa[b + 1]
        ok = (ta < tb) | ((ta == tb) & (ra < rb))
        assert bool(ok.all()), f"suffixes out of order near SA position {lo + int((~ok).nonzero()[0])}"
    del isa


def _brute_rows(recs, record_index, htod_rows, spans, ks):
    """metrics.hpp:109-164 restated with plain loops for the sampled iterations ks (records are in
    (start,row) order already: the C5 generator emits them start-sorted, checked by the caller)."""
    start, dur = recs.start_ns, recs.duration_ns
    hs = start[htod_rows]
    he = hs + dur[htod_rows]
    hz = np.where(recs.flags[htod_rows] & 1, recs.size_bytes[htod_rows], 0)

    def tstart(i):
        return int(start[record_index[i]])

    def tend(i):
        r = record_index[i]
        return int(start[r] + dur[r])
    out = {}
    for k in ks:
        s, e, _ = spans[k]
        t0, t1 = tstart(s), tend(e)
        row = {"t": (t0, t1)}
        if k > 0:
            lo = tend(spans[k - 1][1])
            iv = max(0, t0 - lo)
            row["interval"] = iv
            if iv > 0:
                a = np.maximum(hs, lo)
                b = np.minimum(he, t0)
                m = b > a
                tot, cl, ch, op = 0, 0, 0, False
                for p, q in sorted(zip(a[m].tolist(), b[m].tolist())):
                    if not op or p > ch:
                        if op:
                            tot += ch - cl
                        cl, ch, op = p, q, True
                    else:
                        ch = max(ch, q)
                if op:
                    tot += ch - cl
                row["overlap"] = float(tot) / float(iv)
        lo_b = tend(spans[k - 1][1]) if k > 0 else -1
        row["bytes"] = int(hz[(hs > lo_b) & (hs <= t1)].sum())
        ri = record_index[s:e + 1]
        st = start[ri]
        en = st + dur[ri]
        g = st[1:] - en[:-1]
        row["gap"] = float(np.maximum(g, 0).sum()) / float(e - s) if e > s else 0.0
        out[k] = row
    return out


def test_c5_full_scale(ctx):
    """C5, 1B events on one B200: tokens, the full suffix array (BK test), analyze, sampled metrics."""
    import torch
    iters, body, init = 500_000, 2_000, 16
    recs, info = synth.generate_config("C5")
    n_tok = init + iters * body
    assert info["n_main"] == n_tok
    drecs = ctx.upload(recs, names_host=True)  # 83 GB of names stay in host memory, streamed
    try:
        res = ctx.analyze_raw(drecs, [iters])
        tokens, record_index, names = ctx.build_token_sequence(drecs, 13)
    finally:
        drecs.free()
    L = res["loops"][0]
    assert (L["pattern_length"], L["pattern_count"], L["first_token"], L["epsilon_used"]) == (body, iters, init, 1)
    pat = np.asarray(L["pattern_tokens"], np.int32)
    # token ids: first appearance order over the init prefix, then the body repeated
    assert tokens.size == n_tok
    assert np.array_equal(tokens[:init], np.arange(init, dtype=np.int32))
    assert np.array_equal(tokens[init:].reshape(iters, body), np.broadcast_to(pat, (iters, body)))
    rows = L["rows"]
    assert rows.shape[0] == iters
    starts = init + body * np.arange(iters)
    assert np.array_equal(rows[:, 0], starts) and np.array_equal(rows[:, 1], starts + body - 1)
    assert not rows[:, 2].any()  # extra ops
    # sampled per-iteration metrics against the reference's definitions
    chunk = 1 << 26
    for lo in range(0, recs.n - 1, chunk):
        seg = recs.start_ns[lo:min(recs.n, lo + chunk + 1)]
        assert np.all(seg[1:] >= seg[:-1]), "C5 records are expected in start order"
    other = np.nonzero(recs.stream != 13)[0]
    htod = other[np.array([b"memcpy htod" in recs.name(int(i)).lower() for i in other])]
    spans = [(int(x[0]), int(x[1]), int(x[2])) for x in rows[:, :3]]
    rng = np.random.default_rng(5)
    ks = sorted(set([0, 1, iters - 1] + rng.integers(0, iters, 40).tolist()))
    want = _brute_rows(recs, record_index, htod, spans, ks)
    for k in ks:
        m, w = itertrace.rows_to_metrics(rows[k:k + 1])[0], want[k]
        assert (m.t_start, m.t_end) == w["t"], k
        assert m.interval_ns == w.get("interval"), k
        assert (m.overlap_ratio is None) == ("overlap" not in w), k
        if m.overlap_ratio is not None:
            assert m.overlap_ratio.hex() == w["overlap"].hex(), k
        assert m.htod_bytes == w["bytes"], k
        assert m.op_gap_mean_ns.hex() == w["gap"].hex(), k
    del recs, record_index, rows, res
    # the full suffix array of tokens + [V] (1,000,000,017 suffixes), BK-checked on the device
    dev = torch.device("cuda", 0)
    np_ = n_tok + 1
    text_t = torch.empty(np_, dtype=torch.int32, device=dev)
    text_t[:n_tok].copy_(torch.from_numpy(tokens))
    text_t[n_tok] = int(names.size)
    del tokens
    sa_t = torch.empty(np_, dtype=torch.int32, device=dev)
    torch.cuda.synchronize()
    ctx.suffix_array_device(text_t.data_ptr(), n_tok, int(names.size), sa_t.data_ptr())
    _bk_check_device(sa_t, text_t)
