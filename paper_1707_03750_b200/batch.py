"""Batches of independent traces (BASELINE config C4: 8192 x 100K-event traces), sharded across
GPUs with no collective on the data path.

* rank r of G owns traces [r*T/G, (r+1)*T/G) — ``shard_bounds``;
* inside a rank, ``run_shard`` keeps ``workers`` traces in flight, one host thread and one
  library context (hence one CUDA stream) per worker: small traces are launch/latency bound, so
  concurrent streams fill the GPU;
* results (per-trace mined period + per-iteration integer rows) are gathered to rank 0 only when
  the caller asks (``gather_to_root``, torch.distributed object gather: NCCL on the GPU box,
  gloo in the CPU tests).

The per-trace processor is injectable so the sharding/gather logic is testable on the CPU.
"""
from __future__ import annotations

import concurrent.futures as cf
import threading
from typing import Callable, Sequence


def shard_bounds(n_items: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced split: sizes differ by at most one, every item owned exactly once."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def summarize(raw: dict) -> dict:
    """The part of an itt_analyze result that travels between ranks (small, picklable)."""
    out = {"main_stream": raw["main_stream"], "n_tokens": raw["n_tokens"], "loops": []}
    for L in raw["loops"]:
        rows = L["rows"]
        out["loops"].append({"pattern_length": L["pattern_length"], "pattern_count": L["pattern_count"],
                             "first_token": L["first_token"], "epsilon_used": L["epsilon_used"],
                             "iterations": int(rows.shape[0]),
                             "interval_sum": int(rows[:, 5].sum()) if rows.shape[0] else 0,
                             "htod_bytes": int(rows[:, 7].sum()) if rows.shape[0] else 0})
    return out


def summarize_c(a) -> dict:
    """summarize() over a live itt_analysis struct (the native batch path)."""
    import ctypes as C

    import numpy as np
    out = {"main_stream": a.main_stream, "n_tokens": a.n_tokens, "loops": []}
    for k in range(a.n_loops):
        L = a.loops[k]
        n = int(L.n_iterations)
        if n:
            buf = (C.c_int64 * (n * 11)).from_address(C.cast(L.rows, C.c_void_p).value)
            rows = np.frombuffer(buf, dtype=np.int64).reshape(n, 11)
            iv, hb = int(rows[:, 5].sum()), int(rows[:, 7].sum())
        else:
            iv = hb = 0
        out["loops"].append({"pattern_length": L.pattern_length, "pattern_count": L.pattern_count,
                             "first_token": L.first_token, "epsilon_used": L.epsilon_used, "iterations": n,
                             "interval_sum": iv, "htod_bytes": hb})
    return out


def run_shard_native(executor, traces: Sequence, loops: Sequence[int], lo: int, hi: int, batched_sa: bool = True) -> list:
    """traces[lo:hi] through the native executor (cuda.Batch: C++ worker threads, one context
    each) — the C4 hot path; same summaries as run_shard.  batched_sa: the suffix arrays of the
    traces in flight are built in one doubling sequence (ITT_ANALYZE_BATCHED_SA)."""
    return executor.analyze([traces[i] for i in range(lo, hi)], list(loops), summarize=summarize_c,
                            batched_sa=batched_sa)


def cuda_processor(device: int = 0) -> Callable:
    """Per-thread library contexts on `device`; returns process(trace, loops) -> summary dict."""
    from .cuda import Context
    local = threading.local()
    contexts = []
    lock = threading.Lock()

    def process(trace, loops):
        ctx = getattr(local, "ctx", None)
        if ctx is None:
            ctx = local.ctx = Context(device)
            with lock:
                contexts.append(ctx)
        return summarize(ctx.analyze_raw(trace, list(loops)))

    process.contexts = contexts
    return process


def run_shard(traces: Sequence, loops_of: Callable[[int], Sequence[int]], lo: int, hi: int,
              process: Callable, workers: int = 8) -> list:
    """Analyze traces[lo:hi] (global indices) with `workers` concurrent streams; ordered results."""
    idx = list(range(lo, hi))
    if workers <= 1:
        return [process(traces[i], loops_of(i)) for i in idx]
    with cf.ThreadPoolExecutor(max_workers=workers) as ex:
        return list(ex.map(lambda i: process(traces[i], loops_of(i)), idx))


def gather_to_root(results: list, world: int, rank: int) -> list | None:
    """Concatenate every rank's shard results on rank 0 in global trace order."""
    if world == 1:
        return results
    import torch.distributed as dist
    bucket = [None] * world if rank == 0 else None
    dist.gather_object(results, bucket, dst=0)
    if rank != 0:
        return None
    out = []
    for part in bucket:
        out.extend(part)
    return out
