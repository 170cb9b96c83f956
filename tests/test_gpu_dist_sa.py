"""GPU: the distributed suffix array's device steps (itt_dsa_*, dist.cu) driven by dist_sa.py
over virtual ranks on one B200 (threads, one library context each; the exchange is a host-side
copy, so no kernel of one rank waits on another's).  Parity: SA and LCP bit-exact against the
single-GPU itt_suffix_array and the oracle (full), capped LCP = min(full LCP, cap) with the same
groups (capped), and mining over the gathered distributed SA/LCP (itt_mine_patterns_sa) equal to
itt_mine_patterns, including a planted-period trace of 2M tokens."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_1707_03750_b200 import cuda, dist_sa

pytestmark = pytest.mark.gpu


def _run(P, tokens, term, cap=0xFFFFFFFF):
    text = torch.tensor(np.concatenate([np.asarray(tokens, np.int32), [term]]), dtype=torch.int32, device="cuda")
    ctxs = [cuda.Context(0) for _ in range(P)]
    try:
        res = dist_sa.run_virtual(P, lambda ex, r: dist_sa.suffix_array_dist(ex, dist_sa.CudaOps(ctxs[r]), text,
                                                                             len(tokens), term, cap))
    finally:
        for c in ctxs:
            c.close()
    sa = torch.cat([r.sa for r in res]).cpu().numpy().view(np.uint32)
    lcp = torch.cat([r.lcp for r in res]).cpu().numpy().view(np.uint32)
    return sa, lcp, res


def _cases():
    rng = np.random.default_rng(11)
    out = [("one", [0], 1)]
    for t in range(6):
        n = int(rng.integers(50, 5000))
        V = int(rng.integers(2, 300))
        out.append((f"random{t}", rng.integers(0, V, n), V))
    body = rng.integers(0, 40, 57)
    out.append(("periodic", np.tile(body, 80)[:4500], 40))
    out.append(("runs", np.array([0] * 3000 + [1] + [0] * 100), 2))
    out.append(("random_200k", rng.integers(0, 1000, 200_000), 1000))
    return out


@pytest.mark.parametrize("P", [1, 2, 3, 4])
def test_dist_full_sa_matches_single_gpu(ctx, P):
    for name, tok, term in _cases():
        want_sa, want_lcp = ctx.suffix_array(tok, term)
        sa, lcp, _ = _run(P, tok, term)
        assert np.array_equal(sa, want_sa), (name, P)
        assert np.array_equal(lcp, want_lcp), (name, P)


def _groups_equal(sa, want_sa, lcp, cap):
    bounds = np.flatnonzero(np.concatenate([[True], lcp[1:] < cap, [True]]))
    return all(np.array_equal(np.sort(sa[a:b]), np.sort(want_sa[a:b])) for a, b in zip(bounds[:-1], bounds[1:]))


@pytest.mark.parametrize("P", [2, 4])
def test_dist_capped_sa(ctx, P):
    for name, tok, term in _cases():
        want_sa, want_lcp = ctx.suffix_array(tok, term)
        for cap in (2, 17, 201):
            sa, lcp, res = _run(P, tok, term, cap)
            full = res[0].cap == 0xFFFFFFFF
            assert np.array_equal(lcp, want_lcp if full else np.minimum(want_lcp, cap)), (name, cap)
            assert _groups_equal(sa, want_sa, lcp, 0xFFFFFFFF if full else cap), (name, cap)


def test_dist_mining_planted_period(ctx):
    rng = np.random.default_rng(3)
    V, body, iters = 150, 200, 10_000
    tok = np.concatenate([np.arange(150, 166) % V, np.tile(rng.integers(0, V, body), iters)]).astype(np.int32)
    tok[:16] = rng.integers(0, V, 16)
    n = tok.size
    loops = [(iters, 1)]
    cap = (n - 1) // iters + 1
    want = ctx.mine_patterns(tok, V, loops)
    for P in (2, 4):
        _, _, res = _run(P, tok, V, cap)
        sa = torch.cat([r.sa for r in res])
        lcp = torch.cat([r.lcp for r in res])
        dtok = torch.from_numpy(tok).cuda()
        got = ctx.mine_patterns_sa(dtok.data_ptr(), n, V, sa.data_ptr(), lcp.data_ptr(), loops)
        assert got == want, P
        assert len(got[0]["tokens"]) == body and got[0]["count"] == iters


@pytest.mark.parametrize("P", [2, 3])
def test_analyze_with_distributed_sa_provider(ctx, P):
    """itt_analyze with the suffix array built by P virtual ranks (itt_analyze_opts.sa_provider):
    summary JSON and details CSV byte-identical to the single-GPU analyze."""
    from paper_1707_03750_b200 import itertrace, synth
    for seed, cfg in ((5, "C1"), (9, "C1")):
        recs, _ = synth.generate_config(cfg, noise_frac=0.05, shuffle_window=64, seed=seed)
        want = itertrace.analyze_trace(ctx, recs, [100])
        ctxs = [cuda.Context(0) for _ in range(P)]
        main = cuda.Context(0)
        try:
            def body(ex, r):
                prov = dist_sa.DistributedSAProvider(ex, dist_sa.CudaOps(ctxs[r]))
                if r != 0:
                    prov.serve()
                    return None
                try:
                    return itertrace.analyze_trace(main, recs, [100], sa_provider=prov), prov.last
                finally:
                    prov.stop()
            got, last = dist_sa.run_virtual(P, body)[0]
        finally:
            for c in ctxs + [main]:
                c.close()
        assert last is not None and last.groups > 0
        assert got.summary_json() == want.summary_json()
        assert got.details_csv(0) == want.details_csv(0)


def _free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


@pytest.mark.parametrize("impl", ["native", "python"])
def test_nccl_provider_one_rank_bench(impl):
    """The NCCL path end to end at one rank (torch.distributed rendezvous, the provider inside
    itt_analyze): the native C++ driver (csrc/dist_driver.cu, ncclSend/Recv on the library
    stream) and dist_sa.py over torch.distributed; bench.py --dist-sa must report results equal to
    the single-GPU path."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                        "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--dist-sa",
                        "--dist-impl", impl, "--config", "C1", "--steps", "2", "--warmup", "1"], cwd=root,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["config"]["equal_to_single_gpu_path"] is True
    assert line["config"]["parallelism"] == "dist-sa1"


def test_bench_sharded_legs_one_rank():
    """bench.py's N>1 line shape at one rank: the replicas line plus the C4-sharded and the
    distributed-SA legs (the path a multi-GPU SCALE run takes)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                        "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--config", "C1",
                        "--sharded-legs", "--dist-config", "C1", "--traces", "64", "--distinct", "8", "--steps", "2",
                        "--warmup", "1", "--no-cpu-baseline", "--no-e2e", "--no-ingest", "--no-sa-full"], cwd=root,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["config"]["mined"]["pattern_length"] == 200
    assert line["c4_sharded"]["config"]["mined_ok"] is True
    assert line["dist_sa"]["config"]["equal_to_single_gpu_path"] is True
