"""CPU: the distributed suffix array's host driver (paper_1707_03750_b200/dist_sa.py) — partition
bounds, halo slices, splitters, split sizes, global ids, LCP routing and convergence — over
virtual ranks (threads) and over torch.distributed gloo with world size 2.  The per-element
device steps are the numpy test double (tests/dsa_numpy_ops.py, same contract as the itt_dsa_*
kernels); the checker is the oracle's suffix array / LCP (oracle/libitt_oracle.so, pinned to the
reference's SuffixTree).  The CUDA steps themselves are covered by tests/test_gpu_dist_sa.py."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1707_03750_b200 import dist_sa
from dsa_numpy_ops import NumpyOps


def _oracle_sa(tokens, term):
    from oracle.bindings import oracle
    return oracle().suffix_array(np.asarray(tokens, np.int32), term)


def _cases():
    rng = np.random.default_rng(7)
    out = [("tiny", [0], 1), ("two", [1, 0], 2)]
    for t in range(4):
        n = int(rng.integers(20, 300))
        V = int(rng.integers(2, 6))
        out.append((f"random{t}", rng.integers(0, V, n).tolist(), V))
    body = rng.integers(0, 5, 13).tolist()
    out.append(("periodic", (body * 23)[:290], 5))
    out.append(("runs", [0] * 150 + [1] * 3 + [0] * 60, 2))
    return out


def _run(P, tokens, term, cap=0xFFFFFFFF):
    text = torch.tensor(list(tokens) + [term], dtype=torch.int32)
    ops = NumpyOps()
    res = dist_sa.run_virtual(P, lambda ex, r: dist_sa.suffix_array_dist(ex, ops, text, len(tokens), term, cap))
    assert [r.kbase for r in res] == list(np.cumsum([0] + [r.sa.numel() for r in res])[:-1])
    sa = np.concatenate([r.sa.numpy().view(np.uint32) for r in res])
    lcp = np.concatenate([r.lcp.numpy().view(np.uint32) for r in res])
    return sa, lcp, res


@pytest.mark.parametrize("P", [1, 2, 3, 5])
def test_virtual_ranks_full_suffix_array(P):
    for name, tok, term in _cases():
        want_sa, want_lcp = _oracle_sa(tok, term)
        sa, lcp, _ = _run(P, tok, term)
        assert np.array_equal(sa, want_sa), name
        assert np.array_equal(lcp, want_lcp), name


def _groups_equal(sa, want_sa, lcp, cap):
    """Capped SA: same groups (runs with lcp >= cap), any order inside a group."""
    start = 0
    for k in range(1, len(sa) + 1):
        if k == len(sa) or lcp[k] < cap:
            if sorted(sa[start:k]) != sorted(want_sa[start:k]):
                return False
            start = k
    return True


@pytest.mark.parametrize("P", [2, 4])
def test_virtual_ranks_capped(P):
    for name, tok, term in _cases():
        want_sa, want_lcp = _oracle_sa(tok, term)
        for cap in (1, 3, 9):
            sa, lcp, res = _run(P, tok, term, cap)
            full = res[0].cap == 0xFFFFFFFF
            want = want_lcp if full else np.minimum(want_lcp, cap)
            assert np.array_equal(lcp, want), (name, cap)
            assert _groups_equal(sa, want_sa, lcp, 0xFFFFFFFF if full else cap), (name, cap)
            assert res[0].h_final >= cap or full


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cases, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ex = dist_sa.TorchExchange()
    ops = NumpyOps()
    got = []
    for name, tok, term, cap in cases:
        text = torch.tensor(list(tok) + [term], dtype=torch.int32)
        r = dist_sa.suffix_array_dist(ex, ops, text, len(tok), term, cap)
        sa = dist_sa.gather_to_root(ex, r.sa)
        lcp = dist_sa.gather_to_root(ex, r.lcp)
        if rank == 0:
            got.append((sa.numpy().view(np.uint32).tolist(), lcp.numpy().view(np.uint32).tolist()))
    if rank == 0:
        out.put(got)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_matches_oracle():
    cases = [(name, tok, term, 0xFFFFFFFF) for name, tok, term in _cases()[2:6]]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cases, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for (name, tok, term, _), (sa, lcp) in zip(cases, got):
        want_sa, want_lcp = _oracle_sa(tok, term)
        assert sa == want_sa.tolist(), name
        assert lcp == want_lcp.tolist(), name
