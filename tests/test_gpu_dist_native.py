"""The natively driven distributed suffix array (csrc/dist_driver.cu) against the reference.

* Virtual ranks (threads of one process on one device, LocalTransport): 1, 2, 3 and 5 ranks —
  including ranks that own no text position — build their slices of the full SA + LCP; the
  concatenation equals the reference tree's leaf order and depths (suffix_tree.hpp:21-190, via
  oracle/_ref) and itt_suffix_array.
* Capped (mining) builds: mining over the gathered SA/LCP equals the reference's mine_pattern
  (mine.hpp:119-127).
* itt_analyze with the suffix array distributed over 2 virtual ranks (itt_dsa_provide / serve)
  equals the single-device analyze, and so does the NCCL transport at one rank (the only NCCL
  shape one GPU can run; G > 1 needs more GPUs and is exercised by bench.py --dist-sa).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from oracle.bindings import CheckerError
from paper_1707_03750_b200 import cuda, dist_native, synth

pytestmark = pytest.mark.gpu


def _strings():
    rng = np.random.default_rng(77)
    out = [("random", rng.integers(0, 300, 50_000).astype(np.int32), 300),
           ("tiny", np.asarray([3, 1, 3], np.int32), 4), ("one", np.asarray([0], np.int32), 1)]
    body = rng.integers(0, 90, 137)
    per = np.tile(body, 200_000 // 137 + 1)[:200_000].astype(np.int32)
    out.append(("periodic", per, 90))
    sub = per.copy()
    sub[rng.integers(0, sub.size, 6)] = 89
    out.append(("periodic-subst", sub, 90))
    out.append(("a^n", np.zeros(20_000, np.int32), 1))
    return out


STRINGS = _strings()


def _to_host(ctx, ptr, n):
    out = np.zeros(max(1, n), np.uint32)
    if n:
        ctx._check(cuda.lib().itt_memcpy_d2h(ctx.h, out.ctypes.data, C.c_void_p(ptr), n * 4))
        ctx.synchronize()
    return out[:n]


def _dist(P, s, term, cap=0xFFFFFFFF):
    """Build over P virtual ranks; returns the gathered (sa, lcp) on the host."""
    import torch
    n = s.size
    text = torch.from_numpy(np.concatenate([s, [term]]).astype(np.int32)).cuda()
    ctxs = [cuda.Context(0) for _ in range(P)]
    try:
        def rank_fn(q, comm):
            part = dist_native.build(ctxs[q], comm, text.data_ptr(), n, term, cap)
            try:
                return part.kbase, _to_host(ctxs[q], part.sa_ptr, part.count), _to_host(ctxs[q], part.lcp_ptr, part.count)
            finally:
                part.free()
        parts = dist_native.run_local(P, rank_fn)
    finally:
        for cx in ctxs:
            cx.close()
    parts.sort(key=lambda t: t[0])
    kb = 0
    for k, sa, _ in parts:
        assert k == kb
        kb += sa.size
    return np.concatenate([p[1] for p in parts]), np.concatenate([p[2] for p in parts])


@pytest.mark.parametrize("P", [1, 2, 3, 5])
@pytest.mark.parametrize("name,s,term", STRINGS, ids=[x[0] for x in STRINGS])
def test_full_sa_over_virtual_ranks(ctx, R, P, name, s, term, monkeypatch):
    if P == 1:  # one rank takes the single-device doubling unless forced through the sample-sort rounds
        monkeypatch.setenv("ITT_DSA_FORCE_DIST", "1")
    sa, lcp = _dist(P, s, term)
    want_sa, want_lcp = ctx.suffix_array(s, term)
    assert np.array_equal(sa, want_sa), (name, P)
    assert np.array_equal(lcp, want_lcp), (name, P)
    if s.size <= 60_000:
        rsa, rlcp = R.suffix_array(s, term)
        assert np.array_equal(sa, rsa) and np.array_equal(lcp, rlcp), (name, P)


def _mine(X, *a):
    try:
        return {"ok": X.mine_patterns(*a)}
    except (cuda.IttError, CheckerError) as e:
        return {"error": e.kind, "message": str(e)}


@pytest.mark.parametrize("P", [2, 3])
def test_capped_mining_over_virtual_ranks(ctx, R, P):
    import torch
    for name, s, term in STRINGS[3:5]:
        it = s.size // 137
        cap = (s.size - 1) // it + 1  # L_max + 1 (mine.hpp:64-67)
        sa, lcp = _dist(P, s, term, cap)
        dt = torch.from_numpy(s).cuda()
        dsa = torch.from_numpy(sa.view(np.int32)).cuda()
        dlcp = torch.from_numpy(lcp.view(np.int32)).cuda()
        got = ctx.mine_patterns_sa(dt.data_ptr(), s.size, term, dsa.data_ptr(), dlcp.data_ptr(), [(it, 1)])
        want = R.mine_patterns(s, term, [(it, 1)])
        assert got == want, (name, P)


def _analyze_distributed(recs, iters, comms, ctx_an, ctxs):
    """Root (rank 0) analyzes; the other ranks serve the distributed suffix array."""
    import threading
    provs = [dist_native.Provider(ctxs[q], comms[q], root=0) for q in range(len(comms))]
    errs = []

    def serve(q):
        try:
            provs[q].serve()
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            comms[q].abort()
    ts = [threading.Thread(target=serve, args=(q,)) for q in range(1, len(comms))]
    for t in ts:
        t.start()
    try:
        res = ctx_an.analyze_raw(recs, [iters], native_provider=provs[0])
    finally:
        provs[0].stop()
        for t in ts:
            t.join()
    info = provs[0].last_info()
    for p in provs:
        p.close()
    if errs:
        raise errs[0]
    return res, info


def test_analyze_with_distributed_sa_over_virtual_ranks(ctx):
    recs, info = synth.generate_config("C2", iterations=2_000)
    want = ctx.analyze_raw(recs, [2_000])
    comms = dist_native.Comm.local(2)
    ctxs = [cuda.Context(0) for _ in range(2)]
    ctx_an = cuda.Context(0)
    try:
        got, dinfo = _analyze_distributed(recs, 2_000, comms, ctx_an, ctxs)
    finally:
        for cm in comms:
            cm.close()
        for cx in ctxs + [ctx_an]:
            cx.close()
    a, b = got["loops"][0], want["loops"][0]
    assert a["pattern_tokens"] == b["pattern_tokens"] and a["pattern_count"] == b["pattern_count"]
    assert np.array_equal(a["rows"], b["rows"])
    assert dinfo.rounds >= 1


@pytest.mark.parametrize("force", ["1", "0"])
def test_nccl_transport_at_one_rank(ctx, force, monkeypatch):
    """force=1: through the sample-sort rounds and NCCL exchanges; 0: one rank's shortcut."""
    import torch
    monkeypatch.setenv("ITT_DSA_FORCE_DIST", force)
    uid = dist_native.Comm.unique_id()
    cx = cuda.Context(0)
    comm = dist_native.Comm.nccl(cx, 1, 0, uid)
    try:
        s, term = STRINGS[3][1], STRINGS[3][2]
        text = torch.from_numpy(np.concatenate([s, [term]]).astype(np.int32)).cuda()
        part = dist_native.build(cx, comm, text.data_ptr(), s.size, term)
        sa, lcp = _to_host(cx, part.sa_ptr, part.count), _to_host(cx, part.lcp_ptr, part.count)
        part.free()
        want_sa, want_lcp = ctx.suffix_array(s, term)
        assert np.array_equal(sa, want_sa) and np.array_equal(lcp, want_lcp)
        recs, _ = synth.generate_config("C2", iterations=1_000)
        want = ctx.analyze_raw(recs, [1_000])
        ctx_an = cuda.Context(0)
        got, _ = _analyze_distributed(recs, 1_000, [comm], ctx_an, [cx])
        ctx_an.close()
        assert np.array_equal(got["loops"][0]["rows"], want["loops"][0]["rows"])
    finally:
        comm.close()
        cx.close()
