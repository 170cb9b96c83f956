"""CPU: the batch-sharding path (C4) with world_size 2 over gloo.

Each rank analyzes its contiguous shard of independent traces with an injected per-trace
processor (here the C restatement oracle, since there is no GPU), results are gathered to rank 0
and must equal the single-process run.  On the GPU box the same code runs with
``batch.cuda_processor`` and NCCL.
"""
from __future__ import annotations

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1707_03750_b200 import batch


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_process(trace_cfg, loops):
    import numpy as np

    from oracle.bindings import oracle
    from paper_1707_03750_b200 import synth
    recs, _ = synth.generate(**trace_cfg)
    O = oracle()
    tok, ri, names = O.build_token_sequence(recs, 13)
    p = O.mine_patterns(tok, len(names), [(loops[0], 1)])[0]
    spans = O.approx_match(tok, np.asarray(p["tokens"]), (len(p["tokens"]) + 3) // 4)
    return {"pattern_length": len(p["tokens"]), "count": p["count"], "first_token": p["first_token"],
            "iterations": int(spans.shape[0])}


TRACES = [dict(seed=1000 + t, iterations=20 + t % 7, body_len=15 + t % 5, vocab=12) for t in range(11)]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = batch.shard_bounds(len(TRACES), world, rank)
    res = batch.run_shard(TRACES, lambda i: [TRACES[i]["iterations"]], lo, hi, _oracle_process, workers=2)
    got = batch.gather_to_root(res, world, rank)
    if rank == 0:
        out.put(got)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_bounds_partition():
    for n in (0, 1, 7, 8192, 8193):
        for world in (1, 2, 3, 4, 8):
            spans = [batch.shard_bounds(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_two_rank_gloo_batch_matches_single_process():
    want = batch.run_shard(TRACES, lambda i: [TRACES[i]["iterations"]], 0, len(TRACES), _oracle_process, workers=1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == want
    assert len(got) == len(TRACES)
