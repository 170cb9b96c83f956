"""Refinement rounds of the prefix doubling (sa.cu: k_refine_detect / k_refine_apply) against the
reference suffix tree (suffix_tree.hpp:21-190, leaf order + node depths, via oracle/_ref).

A doubling round that finds every group already ordered by its second key keeps the SA and only
splits groups; once it has run, levels hold group-head positions and a later round that does find
an inversion falls back to a full sort keyed by those positions.  The strings below are built to
walk every transition on the way: periodic texts (refinement from the second round on), periodic
texts with substitutions / insertions / a second loop (inversions after refinement started, so
head-keyed full rounds), and adversarial repetitive strings (Fibonacci, Thue-Morse, a^n).  SA and
LCP must equal the reference's exactly, and mining on them must too.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle.bindings import CheckerError
from paper_1707_03750_b200 import cuda

pytestmark = pytest.mark.gpu


def _periodic(rng, n, period, alphabet, init=16):
    body = rng.integers(init, init + alphabet, period)
    s = np.concatenate([np.arange(init), np.tile(body, n // period + 1)])[:n]
    return s.astype(np.int32), init + alphabet


def _fib(n):
    a, b = [0], [0, 1]
    while len(b) < n:
        a, b = b, b + a
    return np.asarray(b[:n], np.int32), 2


def _thue_morse(n):
    return np.asarray([bin(i).count("1") & 1 for i in range(n)], np.int32), 2


def _cases():
    rng = np.random.default_rng(2024)
    out = []
    for n, period, alpha in ((3_000, 7, 5), (40_000, 50, 40), (200_000, 200, 150), (300_000, 1_000, 900),
                             (120_000, 3, 2)):
        s, term = _periodic(rng, n, period, alpha)
        out.append((f"periodic-{n}-{period}", s, term))
        t = s.copy()
        t[rng.integers(16, n, 5)] = rng.integers(16, term, 5)  # substitutions
        out.append((f"subst-{n}-{period}", t, term))
        pos = np.sort(rng.integers(16, n, 4))
        ins = np.insert(s, pos, rng.integers(16, term, pos.size)).astype(np.int32)  # foreign ops inside iterations
        out.append((f"insert-{n}-{period}", ins, term))
        s2, _ = _periodic(rng, n // 2, period + 3, alpha)
        out.append((f"two-loops-{n}-{period}", np.concatenate([s, s2[16:]]).astype(np.int32), term))
    for n in (1_000, 100_000):
        out.append((f"fib-{n}", *_fib(n)))
        out.append((f"thue-morse-{n}", *_thue_morse(n)))
    out.append(("a^n", np.zeros(50_000, np.int32), 1))
    return out


CASES = _cases()


@pytest.mark.parametrize("name,s,term", CASES, ids=[c[0] for c in CASES])
def test_full_sa_lcp_vs_reference(ctx, R, name, s, term):
    sa, lcp = ctx.suffix_array(s, term)
    rsa, rlcp = R.suffix_array(s, term)
    assert np.array_equal(sa, rsa), name
    assert np.array_equal(lcp, rlcp), name


def _mine(X, s, term, loops, multi=False):
    try:
        return {"ok": X.mine_patterns(s, term, loops, multi=multi)}
    except (cuda.IttError, CheckerError) as e:
        return {"error": e.kind, "message": str(e)}


SMALL = [c for c in CASES if c[1].size <= 200_001]


@pytest.mark.parametrize("name,s,term", SMALL, ids=[c[0] for c in SMALL])
def test_capped_mining_vs_reference(ctx, R, name, s, term):
    """Mining builds the capped SA (the doubling stops at L_max + 1 symbols): same pattern as the
    reference for iteration counts that make the cap small (refinement then ends the doubling)."""
    for it in (max(2, s.size // 400), max(2, s.size // 60)):
        assert _mine(ctx, s, term, [(it, 1)]) == _mine(R, s, term, [(it, 1)]), (name, it)


@pytest.mark.parametrize("name,s,term", SMALL, ids=[c[0] for c in SMALL])
def test_capped_lcp_from_group_heads(ctx, R, name, s, term, monkeypatch):
    """Capped SA + LCP (what mining consumes): when the final groups are few, the LCP comes from the
    head bitmap + lifting (k_lcp_heads) instead of phi + capped Kasai.  Either way LCP must equal
    min(reference LCP, cap) and the suffixes must be grouped as in the reference (order inside a
    final group is by position)."""
    import torch
    rsa, rlcp = R.suffix_array(s, term)
    n = s.size
    for cap in (9, 65, 1025):
        got = {}
        for mode in ("0", "1"):
            monkeypatch.setenv("ITT_LCP_HEADS", mode)
            tok = torch.from_numpy(s).cuda()
            sa = torch.empty(n + 1, dtype=torch.int32, device="cuda")
            lcp = torch.empty(n + 1, dtype=torch.int32, device="cuda")
            ctx.suffix_array_device(tok.data_ptr(), n, term, sa.data_ptr(), lcp.data_ptr(), cap=cap)
            got[mode] = lcp.cpu().numpy().view(np.uint32)
        want = np.minimum(rlcp.astype(np.uint64), cap).astype(np.uint32)
        assert np.array_equal(got["0"], want), (name, cap)
        assert np.array_equal(got["1"], want), (name, cap)


def test_init_level_table_overflow_falls_back_to_scatter(ctx, R):
    """The first level comes from a (k-gram -> head) table filled in text order when the distinct
    k-grams fit it (64K entries, at most 64 probes); a random text over a large alphabet has more
    distinct k-grams than that, so the init update must fall back to the scatter — same SA/LCP."""
    rng = np.random.default_rng(4242)
    for n, alpha in ((300_000, 1_000), (150_000, 60_000)):
        s = rng.integers(0, alpha, n).astype(np.int32)
        sa, lcp = ctx.suffix_array(s, alpha)
        rsa, rlcp = R.suffix_array(s, alpha)
        assert np.array_equal(sa, rsa) and np.array_equal(lcp, rlcp), (n, alpha)
        assert _mine(ctx, s, alpha, [(50, 1)]) == _mine(R, s, alpha, [(50, 1)])
