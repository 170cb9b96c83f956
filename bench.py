#!/usr/bin/env python3
"""bench.py — trace events/sec of the B200 mining pipeline (intern -> SA -> LCP -> repeat ->
spans -> per-iteration aggregates) on the largest single-GPU BASELINE config, C3 (BASELINE.json
configs[2]: 100M-event TF-like trace, 20K iterations x 5000 ops, V=4096 distinct op names).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl cuda|reference] [--config C3]

* value : whole-job events/s with the columns already resident in HBM (device-timed with CUDA
          events on the library's stream; one step = one itt_analyze call = the full path).
* e2e   : the same metric through the C-ABI with pinned HOST buffers (H2D of every column and
          the D2H of the per-iteration rows inside the timed region).
* roofline : dominant kernel's algorithmic bytes / its CUDA-event launch time (profiled pass).
* cpu_baseline : the reference itself (oracle/_ref, compiled from the reference headers) on a
          bounded sample of the same workload, 1 host core (the reference is single-threaded).
* sa_full : the full suffix array + LCP (itt_suffix_array, cap = infinity) of the same tokens,
          device-resident, timed beside the step (the step itself builds the capped SA mining needs).
Under torchrun: C1-C3 run one replica per rank ("replicas only"); C4 shards the
batch; --dist-sa spreads one trace's suffix array over the ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "trace events/sec for SA+LCP+repeat mining+segmentation; % HBM roofline"
WORKLOADS = {
    "C1": ("C1: synthetic TF-like trace, 100 iterations x 200 ops (~20K events), V=150 body names + 16 init names",
           dict(), 100),
    "C2": ("C2: 10M-event trace, 50K iterations x 200 ops, V=150 (+16 init), 5% memcpy noise on streams 14/15, "
           "rows shuffled in windows of 64", dict(), 50_000),
    "C3": ("C3: 100M-event trace, 20K iterations x 5000 ops, V=4096 (+16 init)", dict(), 20_000),
    "C4": ("C4: batch of 8192 independent 100K-event traces (500 iterations x 200 ops, V=150 + 16 init), "
           "sharded across ranks", dict(), 500),
    "C5": ("C5: 1B-event trace, 500K iterations x 2000 ops, V=4096 (+16 init), on ONE B200: numeric columns "
           "resident in HBM, the 80 GB of names streamed from pinned host memory through 2 x 1 GB windows into the hash pass",
           dict(), 500_000),
}
# bounded CPU samples (same generator and shape, fewer iterations)
CPU_SAMPLE_ITERS = {"C1": 100, "C2": 10_000, "C3": 400, "C5": 1_000}
REF_ARM_ITERS = {"C1": 100, "C2": 2_000, "C3": 400, "C5": 250}  # ~1-4 s per reference step on one core


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons every 20 ms; only samples stamped inside the timed
    window (mark_start/mark_end) are summarised.  The sampler starts before the warm-up so it is
    producing rows by the time the timed region begins."""

    Q = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, interval_ms: int = 20):
        self.index = index
        self.interval_ms = interval_ms
        self.rows = []
        self.proc = None
        self.t0 = self.t1 = None

    def __enter__(self):
        if self.interval_ms <= 0:  # diagnosis only: no sampler (the JSON then has no clock samples)
            return self
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", str(self.interval_ms)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        import datetime
        for line in self.proc.stdout:
            r = [x.strip() for x in line.split(",")]
            try:
                ts = datetime.datetime.strptime(r[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except Exception:
                ts = time.time()
            self.rows.append((ts, r[1:]))

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()
        time.sleep(0.05)  # let the last in-window rows arrive

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = [r for ts, r in self.rows if self.t0 is None or (self.t0 - 0.02 <= ts <= (self.t1 or ts) + 0.02)]
        in_window = bool(rows)
        if not rows and self.rows and self.t0 is not None:  # window shorter than the interval: nearest samples
            near = sorted(self.rows, key=lambda tr: min(abs(tr[0] - self.t0), abs(tr[0] - (self.t1 or self.t0))))
            rows = [r for _, r in near[:2]]
        ok = [r for r in rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        sm = [float(r[0]) for r in ok]
        mx = [float(r[1]) for r in ok if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in ok for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(ok), "in_window": in_window, "interval_ms": self.interval_ms}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    return ws, int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


def make_trace(config: str, iterations: int | None = None):
    from paper_1707_03750_b200 import synth
    kw = {}
    if iterations is not None:
        kw["iterations"] = iterations
    return synth.generate_config(config, **kw)


def cpu_reference_run(config: str, iters: int, steps: int, warmup: int, full_iters: int | None = None):
    """Time the reference (oracle/_ref: the stock analyze_trace, pipeline.hpp:34-134) on a bounded
    sample, 1 core.  A step's time is the reference's own work as its CLI would do it after parsing:
    the (start,row) stable sort (ingest.hpp:396-400) + analyze_trace — not the marshalling of our
    columns into its AoS records and not the JSON/CSV rendering (the GPU step renders nothing).
    One extra staged run (the same stage calls with timers) gives the per-stage split, and from it
    an extrapolation to the full-size trace (labelled as such: linear stages scale with events,
    the metrics stage with I * H, i.e. quadratically in iterations, metrics.hpp:109-164)."""
    from oracle.bindings import ref
    recs, info = make_trace(config, iters)
    R = ref()
    times = []
    for s in range(warmup + steps):
        res = R.analyze(recs, [iters], staged=False)
        if s >= warmup:
            times.append((res["times"]["order_ms"] + res["times"]["analyze_ms"]) / 1000.0)
    ev = info["n"] / statistics.mean(times)
    stage = R.analyze(recs, [iters], staged=True)["times"]
    split = {k[:-3]: round(stage[k], 1) for k in ("order_ms", "filter_census_ms", "intern_ms", "mine_ms", "match_ms",
                                                  "metrics_ms")}
    sample = (f"{config}-shaped trace with {iters} iterations ({info['n']} events, {info['n_main']} tokens): stock "
              f"analyze_trace + the (start,row) sort, 1 core; stage split of one staged run (ms): "
              + ", ".join(f"{k}={v:.0f}" for k, v in split.items()))
    extra = {"stage_ms": split}
    if full_iters and full_iters > iters:
        f = full_iters / iters
        lin = sum(v for k, v in split.items() if k != "metrics")
        extra["extrapolated_full_size_s"] = round((lin * f + split["metrics"] * f * f) / 1000.0, 1)
        extra["extrapolation"] = (f"EXTRAPOLATED, not measured: {full_iters} iterations = {f:.0f}x the sample; "
                                  "linear stages x f, metrics x f^2")
    return ev, info, sample, times, extra


def _c4_ref_worker(seeds):
    """One host core: the reference (oracle/_ref) analyzing its own C4 traces; returns (events, s)."""
    from oracle.bindings import ref
    from paper_1707_03750_b200 import synth
    R = ref()
    kw = dict(synth.CONFIGS["C4"])
    ev, busy = 0, 0.0
    for sd in seeds:
        recs, info = synth.generate(**dict(kw, seed=sd))
        t0 = time.perf_counter()
        R.analyze(recs, [500], staged=False)
        busy += time.perf_counter() - t0
        ev += info["n"]
    return ev, busy


def c4_cpu_baseline(per_core: int = 2):
    """SURVEY §8d for C4: one reference process per host core over disjoint traces."""
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    seeds = [[1000 + c * per_core + k for k in range(per_core)] for c in range(cores)]
    with mp.get_context("spawn").Pool(cores) as p:
        res = p.map(_c4_ref_worker, seeds)
    ev = sum(r[0] for r in res)
    wall = max(r[1] for r in res)
    return {"value": ev / wall, "unit": "events/s", "cores": cores, "kind": "reference",
            "sample": f"{cores} reference processes x {per_core} C4 traces each ({ev} events; busy time of the slowest "
                      f"process {wall:.2f} s)"}


def bench_batch(args, world, rank, local, workload):
    """C4: every rank analyzes its contiguous shard of the batch; no collective on the data path
    (a barrier + max-over-ranks time bracket the timed region).  Strong scaling: the batch size is
    fixed, so per-rank work shrinks as N grows."""
    import concurrent.futures as cf

    import torch
    from paper_1707_03750_b200 import batch, cuda as itt, synth
    dev = local if world > 1 else 0
    torch.cuda.set_device(dev)
    lo, hi = batch.shard_bounds(args.traces, world, rank)
    pool_ids = sorted({t % args.distinct for t in range(lo, hi)})
    kw = dict(synth.CONFIGS["C4"])

    def gen(t):
        return t, synth.generate(**dict(kw, seed=1000 + t))
    with cf.ThreadPoolExecutor(8) as ex:
        pool = dict(ex.map(gen, pool_ids))
    up_ctx = itt.Context(dev)
    dev_pool = {t: (up_ctx.upload(recs), info) for t, (recs, info) in pool.items()}
    traces = [dev_pool[t % args.distinct][0] for t in range(args.traces)]  # global index -> resident trace
    events = sum(dev_pool[t % args.distinct][1]["n"] for t in range(lo, hi))
    loops_of = lambda i: [500]  # noqa: E731
    if args.batch_impl == "native":  # C++ worker threads (itt_batch_*), no interpreter between traces
        executor = itt.Batch(dev, args.workers)

        def one_pass():
            return batch.run_shard_native(executor, traces, [500], lo, hi)
        launch_count = executor.launch_count
    else:  # Python threads, one library context each
        process = batch.cuda_processor(dev)

        def one_pass():
            return batch.run_shard(traces, loops_of, lo, hi, process, workers=args.workers)
        launch_count = lambda: sum(c.launch_count() for c in process.contexts)  # noqa: E731

    for _ in range(max(1, args.warmup)):
        res = one_pass()
    l0 = launch_count()

    def bar():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)
    clk = ClockSampler(dev, args.clock_ms).__enter__()
    time.sleep(0.3)
    bar()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk.mark_start()
    e0.record()
    for _ in range(args.steps):
        res = one_pass()
    torch.cuda.synchronize(dev)
    e1.record()
    e1.synchronize()
    clk.mark_end()
    clk.__exit__()
    bar()
    ms = e0.elapsed_time(e1)
    ev_total = torch.tensor([float(events), ms], device=f"cuda:{dev}")
    if world > 1:
        t = ev_total.clone()
        torch.distributed.all_reduce(ev_total[0:1], op=torch.distributed.ReduceOp.SUM)
        torch.distributed.all_reduce(t[1:2], op=torch.distributed.ReduceOp.MAX)
        ev_total[1] = t[1]
    total_events, ms = float(ev_total[0].item()), float(ev_total[1].item())
    launches = (launch_count() - l0) // max(1, args.steps)
    ok = all(r["loops"][0]["pattern_length"] == 200 and r["loops"][0]["iterations"] == 500 for r in res)
    # e2e: the same batch from pinned HOST columns (each trace's H2D inside the timed region, the
    # per-iteration rows back to the host): the executor's own copies, native workers
    e2e = None
    if args.batch_impl == "native" and not args.no_e2e:
        fields = ["start_ns", "duration_ns", "size_bytes", "flags", "stream", "name_off", "name_bytes", "device"]
        registered = []
        try:
            for t in pool_ids:
                for f in fields:
                    a = getattr(pool[t][0], f, None)
                    if a is not None and a.nbytes:
                        try:
                            up_ctx.register_host(a)
                            registered.append(a)
                        except itt.IttError:
                            pass  # stays pageable (slower copies, same result)
            host_traces = [pool[t % args.distinct][0] for t in range(args.traces)]

            def one_pass_host():
                return batch.run_shard_native(executor, host_traces, [500], lo, hi)
            one_pass_host()
            bar()
            h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            h0.record()
            for _ in range(args.steps):
                res_h = one_pass_host()
            torch.cuda.synchronize(dev)
            h1.record()
            h1.synchronize()
            bar()
            ms_h = torch.tensor([h0.elapsed_time(h1)], device=f"cuda:{dev}")
            if world > 1:
                torch.distributed.all_reduce(ms_h, op=torch.distributed.ReduceOp.MAX)
            ms_h = float(ms_h.item())
            # pinned size columns are read in place (HtoD rows only, zero-copy), not copied whole
            pinned_ids = {id(a) for a in registered}
            h2d = sum(host_traces[i].nbytes() - (host_traces[i].size_bytes.nbytes if id(host_traces[i].size_bytes) in pinned_ids
                                                 else 0) for i in range(lo, hi))
            d2h = sum(sum(L["iterations"] * 88 for L in r["loops"]) for r in res_h)  # itt_iter_row: 11 x i64
            ok = ok and all(r["loops"][0]["pattern_length"] == 200 for r in res_h)
            e2e = {"value": total_events / (ms_h / args.steps / 1000.0), "unit": "events/s",
                   "h2d_bytes_per_step": int(h2d * (world if world > 1 else 1)), "d2h_bytes_per_step": int(d2h),
                   "ms_per_step": ms_h / args.steps, "pinned_columns": f"{len(registered)} registered"}
        finally:
            for a in registered:
                up_ctx.unregister_host(a)
    if rank == 0:
        line = {"metric": METRIC, "value": total_events / (ms / args.steps / 1000.0), "unit": "events/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
                "config": {"workload": workload, "traces": args.traces, "distinct_traces": args.distinct,
                           "events_per_step": int(total_events), "workers_per_gpu": args.workers, "executor": args.batch_impl,
                           "batched_suffix_arrays": args.batch_impl == "native",
                           "parallelism": f"shard{world}", "mined_ok": bool(ok)},
                "clocks": clk.summary(), "gpu_launches": int(launches), "e2e": e2e}
        if world == 1 and not args.no_cpu_baseline:
            try:
                line["cpu_baseline"] = c4_cpu_baseline()
            except Exception as e:  # noqa: BLE001 (the reference build is optional on the box)
                line["cpu_baseline"] = {"unavailable": str(e)[:200]}
        return line
    return None


def bench_dist_sa(args, world, rank, local, workload, iters):
    """One trace, suffix array over all ranks (SURVEY §8e C5 path): rank 0 runs itt_analyze on the
    trace with the distributed suffix array plugged in (itt_analyze_opts.sa_provider); every rank
    builds its share of the SA/LCP and rank 0 mines / matches / aggregates.  --dist-impl native
    (default): the C++ driver with NCCL on the library's streams (csrc/dist_driver.cu); python:
    dist_sa.py over torch.distributed."""
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    from paper_1707_03750_b200 import cuda as itt, dist_native, dist_sa
    dev = local
    ops_ctx = itt.Context(dev)
    if args.dist_impl == "native":
        uid = [dist_native.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = dist_native.Comm.nccl(ops_ctx, world, rank, uid[0])
        prov = dist_native.Provider(ops_ctx, comm, root=0)
        kw_of = lambda: dict(native_provider=prov)  # noqa: E731
    else:
        prov = dist_sa.DistributedSAProvider(dist_sa.TorchExchange(device=torch.device("cuda", dev)),
                                             dist_sa.CudaOps(ops_ctx))
        kw_of = lambda: dict(sa_provider=prov)  # noqa: E731
    if rank != 0:
        prov.serve()
        dist.barrier()
        return None
    ctx = itt.Context(dev)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=torch.device("cuda", dev))
    if args.iterations:
        iters = args.iterations
        workload += f" [DRY RUN: iterations overridden to {iters}]"
    recs, info = make_trace(args.config, args.iterations)
    drecs = ctx.upload(recs, names_host=args.config == "C5")
    n_events = info["n"]

    def step():
        return ctx.analyze_raw(drecs, [iters], **kw_of())

    for _ in range(max(3, args.warmup)):
        res = step()
    want = ctx.analyze_raw(drecs, [iters])  # single-GPU path: the distributed SA must not change a thing
    same = all(a["pattern_tokens"] == b["pattern_tokens"] and np.array_equal(a["rows"], b["rows"])
               for a, b in zip(res["loops"], want["loops"]))
    torch.cuda.synchronize(dev)
    ctx.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        res = step()
    e1.record(stream)
    e1.synchronize()
    ms_step = e0.elapsed_time(e1) / args.steps
    prov.stop()
    if args.dist_impl == "native":
        inf = prov.last_info()
        rounds, groups, cap = inf.rounds, inf.groups, inf.cap
    else:
        rounds, groups, cap = prov.last.rounds, prov.last.groups, prov.last.cap
    line = {"metric": METRIC, "value": n_events / (ms_step / 1000.0), "unit": "events/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": workload + " -- suffix array distributed over the ranks (sample-sort prefix doubling, "
                                              f"{args.dist_impl} driver)",
                       "events": n_events, "tokens": res["n_tokens"], "parallelism": f"dist-sa{world}",
                       "doubling_rounds": rounds, "groups": groups, "cap": cap,
                       "equal_to_single_gpu_path": bool(same)},
            "gpu_launches": None}
    dist.barrier()
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--config", default="C3", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--iterations", type=int, default=None,
                    help="override the workload's iteration count (smaller dry runs of C3/C5)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sa-full", action="store_true", help="skip timing the full (uncapped) suffix array")
    ap.add_argument("--no-ingest", action="store_true", help="skip the GPU CSV ingest measurement")
    ap.add_argument("--profile-steps", type=int, default=2)
    ap.add_argument("--clock-ms", type=int, default=200,
                    help="nvidia-smi sampling interval during the timed region (the profiling recipe's 200 ms: "
                         "NVML queries can stall the driver for milliseconds)")
    ap.add_argument("--traces", type=int, default=8192, help="C4: traces in the batch")
    ap.add_argument("--distinct", type=int, default=256, help="C4: distinct generated traces (batch cycles them)")
    ap.add_argument("--workers", type=int, default=64, help="C4: concurrent streams (host threads) per GPU")
    ap.add_argument("--dist-sa", action="store_true",
                    help="one trace with its suffix array distributed over all ranks (NCCL; C5's multi-GPU path)")
    ap.add_argument("--sharded-legs", action="store_true", help="add the N>1 sharded legs at N=1 too (tests)")
    ap.add_argument("--no-sharded-legs", action="store_true",
                    help="N>1: skip the C4-sharded and distributed-SA measurements added beside the replicas line")
    ap.add_argument("--dist-config", default="C3", choices=["C1", "C2", "C3", "C5"],
                    help="N>1: the trace whose suffix array the distributed-SA leg spreads over the ranks")
    ap.add_argument("--dist-impl", default="native", choices=["native", "python"],
                    help="--dist-sa driver: C++ with NCCL on the library streams, or dist_sa.py over torch.distributed")
    ap.add_argument("--batch-impl", default="native", choices=["native", "threads"],
                    help="C4 executor: native C++ worker threads (itt_batch_*) or Python threads")
    args = ap.parse_args()
    world, rank, local = dist_env()
    workload, _, iters = WORKLOADS[args.config]

    if args.impl == "reference":
        if rank != 0:
            return 0
        it = REF_ARM_ITERS[args.config]
        ev, info, sample, times, extra = cpu_reference_run(args.config, it, args.steps, max(1, args.warmup), iters)
        line = {"metric": METRIC, "value": ev, "unit": "events/s", "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1000 * statistics.mean(times), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic", "impl": "reference",
                "config": {"workload": workload, "sample_iterations": it, "events_per_step": info["n"]},
                "cpu_baseline": {"value": ev, "unit": "events/s", "cores": 1, "kind": "reference", "sample": sample,
                                 **extra},
                "e2e": {"value": ev, "unit": "events/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    import torch
    # a process group whenever ranks exchange anything: N>1, or the distributed suffix array
    pg = world > 1 or args.dist_sa or args.sharded_legs
    if pg:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        torch.cuda.set_device(local)
        torch.distributed.init_process_group("nccl", rank=rank, world_size=world)
    try:
        if args.config == "C4":
            line = bench_batch(args, world, rank, local, workload)
        elif args.dist_sa:
            line = bench_dist_sa(args, world, rank, local, workload, iters)
        else:
            line = bench_single(args, world, rank, local, workload, iters)
            if (world > 1 or args.sharded_legs) and not args.no_sharded_legs:
                # the configs that shard across GPUs, measured at this N beside the
                # replicas line: C4's batch split across ranks (strong scaling, no data-path
                # collective) and one trace's suffix array distributed over the ranks (NCCL)
                c4 = argparse.Namespace(**vars(args))
                c4.steps, c4.warmup, c4.config = max(1, min(args.steps, 3)), 1, "C4"
                leg_c4 = bench_batch(c4, world, rank, local, WORKLOADS["C4"][0])
                ds = argparse.Namespace(**vars(args))
                ds.steps, ds.warmup, ds.config = max(1, min(args.steps, 5)), 1, args.dist_config
                leg_ds = bench_dist_sa(ds, world, rank, local, WORKLOADS[ds.config][0], WORKLOADS[ds.config][2])
                if rank == 0:
                    line["c4_sharded"] = leg_c4
                    line["dist_sa"] = leg_ds
        if rank == 0 and line is not None:
            print(json.dumps(line), flush=True)
    finally:
        if pg:
            torch.distributed.destroy_process_group()
    return 0


def bench_single(args, world, rank, local, workload, iters):
    """C1/C2/C3/C5: one trace per rank (replicas: a trace's pipeline has no data-path exchange)."""
    import torch
    from paper_1707_03750_b200 import cuda as itt

    dev = local if world > 1 else 0
    torch.cuda.set_device(dev)
    ctx = itt.Context(dev)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=torch.device("cuda", dev))
    t_gen = time.perf_counter()
    if args.iterations:
        iters = args.iterations
        workload += f" [DRY RUN: iterations overridden to {iters}]"
    recs, info = make_trace(args.config, args.iterations)
    log(f"[rank {rank}] generated {args.config}: {info} in {time.perf_counter() - t_gen:.1f}s")
    n_events = info["n"]
    names_host = args.config == "C5"  # 80 GB of names do not fit in HBM beside the pipeline: streamed
    drecs = ctx.upload(recs, names_host=names_host)
    if names_host:
        log(f"[rank {rank}] names streamed from {'pinned' if drecs.names_pinned else 'PAGEABLE'} host memory")

    def step_device():
        return ctx.analyze_raw(drecs, [iters])

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)
        ctx.synchronize()

    def timed(fn, steps):
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            res = fn()
        e1.record(stream)
        e1.synchronize()
        barrier()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device=f"cuda:{dev}")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        return ms, res

    clk = ClockSampler(dev, args.clock_ms).__enter__()
    for _ in range(max(3, args.warmup)):
        res = step_device()
    # then keep warming for at least 1 s of steps (clocks ramp, caches of the block allocator fill):
    # a short warm-up at C1/C2 sizes left the first timed region ~10% slower than later ones
    t_w = time.perf_counter()
    extra_warmup = 0
    while time.perf_counter() - t_w < 1.0:
        res = step_device()
        extra_warmup += 1
    # correctness guard: the mined period must be the planted body
    assert res["loops"][0]["pattern_length"] == {"C1": 200, "C2": 200, "C3": 5000, "C5": 2000}[args.config] \
        or args.iterations
    l0 = ctx.launch_count()
    clk.mark_start()
    ms, res = timed(step_device, args.steps)
    clk.mark_end()
    clk.__exit__()
    launches = (ctx.launch_count() - l0) // max(1, args.steps)
    ms_step = ms / args.steps
    value = world * n_events / (ms_step / 1000.0)
    log(f"[rank {rank}] device-resident: {ms_step:.2f} ms/step, {value / 1e9:.3f}G events/s")

    # ---- roofline: profiled pass (per-kernel CUDA events on the library stream)
    ctx.set_profiling(True)
    ctx.reset_stats()
    for _ in range(args.profile_steps):
        step_device()
    stats = ctx.kernel_stats()
    ctx.set_profiling(False)
    tot = sum(s["total_ms"] for s in stats.values()) or 1.0
    top = max(stats.items(), key=lambda kv: kv[1]["total_ms"])
    name, st = top
    per_launch_bytes = st["bytes"] / st["launches"]
    avg_ms = st["total_ms"] / st["launches"]
    achieved = per_launch_bytes / (avg_ms / 1000.0) / 1e9
    peak, peak_kind = peaks()
    traffic = None
    prof_json = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof_json):
        try:
            pj = json.load(open(prof_json))
            # ncu bytes only describe the workload they were captured on
            if pj.get("workload") == args.config:
                traffic = pj.get("kernels", {}).get(name, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": peak, "peak_kind": peak_kind,
                "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                "share_of_step": st["total_ms"] / tot, "launches_per_step": st["launches"] / args.profile_steps}
    if traffic:
        # DRAM bytes the kernel really moves (ncu, same workload) over its live launch time: for the
        # random-access kernels (one 32-B sector per 4-B gather) this, not the algorithmic figure, is
        # how close the kernel runs to the memory system's limit
        roofline["traffic_GBps"] = traffic / (avg_ms / 1000.0) / 1e9
        roofline["traffic_frac"] = roofline["traffic_GBps"] / peak
        roofline["traffic_per_algorithmic_byte"] = traffic / per_launch_bytes
    # the random-access kernels are judged on sector efficiency too: the committed
    # ncu metrics pass of the same workload (scripts/sector_profile.sh)
    sect = os.path.join(ROOT, "profiles", "r01h_sector_efficiency.csv")
    kmap = {"sa_rank_update": "k_rank_update", "radix_onesweep": "k_onesweep", "lcp_plcp": "k_plcp", "lcp_phi": "k_phi",
            "lcp_gather": "k_lcp_gather", "ansv_intervals": "k_ansv"}
    if args.config == "C2" and os.path.exists(sect) and name in kmap:
        for ln in open(sect):
            f = ln.strip().split(",")
            if f and f[0] == kmap[name]:
                roofline["sector_efficiency"] = {"ld_bytes_per_sector_pct": float(f[5]), "st_bytes_per_sector_pct": float(f[6]),
                                                 "l2_hit_pct": float(f[4]), "source": "profiles/r01h_sector_efficiency.csv"}
    # the north star's radix-pass figure: 16 B per key-value pair per onesweep pass
    passes = [stats[k] for k in ("radix_onesweep", "radix_onesweep_w10") if k in stats]  # 8- and 10-bit digits
    if passes:
        pb, pms, pl = sum(x["bytes"] for x in passes), sum(x["total_ms"] for x in passes), sum(x["launches"] for x in passes)
        ra = pb / (pms / 1000.0) / 1e9
        roofline["radix_pass"] = {"achieved": ra, "frac": ra / peak, "passes_per_step": pl / args.profile_steps,
                                  "us_per_pass": 1000.0 * pms / pl}
    kernel_table = {k: {"ms_per_step": v["total_ms"] / args.profile_steps,
                        "GBps": (v["bytes"] / (v["total_ms"] / 1000.0) / 1e9) if v["total_ms"] > 0 else None}
                    for k, v in sorted(stats.items(), key=lambda kv: -kv[1]["total_ms"])}

    # ---- device memory: resident columns + the pipeline's high-water mark
    used0, _ = ctx.mem_stats(reset=True)
    step_device()
    _, high = ctx.mem_stats()
    memory = {"resident_columns_gb": drecs.nbytes / 1e9, "pool_high_water_gb": high / 1e9,
              "pipeline_peak_gb": (high - used0) / 1e9}

    # ---- a12 (the north star's per-op x per-iteration profile; no reference counterpart, so it
    # is reported as the increment over the reference-equivalent step, not inside `value`)
    def step_a12():
        return ctx.analyze_raw(drecs, [iters], op_profile=True)
    step_a12()
    ms_a12, _ = timed(step_a12, args.steps)
    ctx.set_profiling(True)
    ctx.reset_stats()
    step_a12()
    st_a12 = {k: v["total_ms"] for k, v in ctx.kernel_stats().items() if k.startswith("opprof")}
    ctx.set_profiling(False)
    op_profile = {"ms_per_step": ms_a12 / args.steps, "increment_ms": ms_a12 / args.steps - ms_step,
                  "events_per_s": world * n_events / (ms_a12 / args.steps / 1000.0),
                  "outputs": "per-op and per-iteration totals (cell grid on request)", "kernels_ms": st_a12}

    # ---- e2e through the C-ABI with pinned host buffers
    e2e = None
    if not args.no_e2e:
        fields = ["start_ns", "duration_ns", "size_bytes", "flags", "stream", "name_off"] + \
            ([] if names_host else ["name_bytes"]) + (["device"] if recs.device is not None else [])
        registered, staged = [], {}
        for f in fields:  # pinned for full-speed DMA: registered in place, else staged into cudaHostAlloc memory
            a = getattr(recs, f)
            try:
                ctx.register_host(a)
                registered.append(a)
            except itt.IttError as e:
                buf = torch.empty(a.nbytes, dtype=torch.uint8, pin_memory=True)
                view = buf.numpy().view(a.dtype)
                view[:] = a
                staged[f] = (buf, view)
                log(f"[rank {rank}] e2e: column {f} ({a.nbytes / 1e9:.2f} GB) not registrable ({e}); "
                    "staged into pinned memory instead")
        if staged:
            from paper_1707_03750_b200 import abi as _abi
            recs_e = _abi.Records(**{f: staged[f][1] if f in staged else getattr(recs, f) for f in
                                   ("start_ns", "duration_ns", "stream", "name_off", "name_bytes", "size_bytes",
                                    "flags", "device")}, order=recs.order, keepalive=(recs._keepalive, staged))
        else:
            recs_e = recs
        cols = fields
        if names_host:  # still registered by drecs; streamed again
            from paper_1707_03750_b200 import abi as _abi
            recs_e.mem = _abi.MEM_HOST_STREAM_NAMES
        try:
            def step_host():
                return ctx.analyze_raw(recs_e, [iters])
            step_host()
            ms_e, res_e = timed(step_host, args.steps)
        finally:
            for a in registered:
                ctx.unregister_host(a)
        d2h = sum(L["rows"].nbytes + 4 * L["pattern_length"] for L in res_e["loops"])
        # a pinned size column is read in place (HtoD rows only, zero-copy), not copied whole
        h2d = int(recs_e.nbytes()) - (int(recs.size_bytes.nbytes) if any(a is recs.size_bytes for a in registered) else 0)
        e2e = {"value": world * n_events / (ms_e / args.steps / 1000.0), "unit": "events/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": int(d2h),
               "ms_per_step": ms_e / args.steps,
               "pinned_columns": f"{len(registered)} registered + {len(staged)} staged of {len(cols)}"}
        log(f"[rank {rank}] e2e: {e2e['ms_per_step']:.2f} ms/step, {e2e['value'] / 1e9:.3f}G events/s")

    # ---- GPU CSV ingest: the same trace as profiler CSV text, parsed by
    # itt_parse_csv (host text -> HBM records), against the reference's parse_trace_text on a sample
    ingest = None
    if rank == 0 and not args.no_ingest and args.config in ("C1", "C2"):
        try:
            from paper_1707_03750_b200 import synth as _synth
            text = _synth.to_csv(recs)
            times = []
            for _ in range(3):
                t0 = time.perf_counter()
                pt = ctx.parse_csv(text, "bench.csv")
                times.append(time.perf_counter() - t0)
                assert pt.n == n_events and pt.rows_skipped == 0
                pt.free()
            ctx.set_profiling(True)
            ctx.reset_stats()
            ctx.parse_csv(text, "bench.csv").free()
            kst = {k: v["total_ms"] for k, v in ctx.kernel_stats().items() if k.startswith("ingest")}
            ctx.set_profiling(False)
            best = min(times)
            ingest = {"rows": n_events, "csv_bytes": len(text), "wall_ms": best * 1000,
                      "rows_per_s": n_events / best, "csv_GBps": len(text) / best / 1e9,
                      "kernels_ms": kst, "note": "wall time of itt_parse_csv on pageable host text (H2D inside)"}
            if not args.no_cpu_baseline:
                from oracle.bindings import ref as _ref
                sample = text[:text.index(b"\n", min(len(text) - 1, 200_000_000)) + 1]
                t0 = time.perf_counter()
                rp = _ref().parse_csv(sample, "bench.csv")
                dt = time.perf_counter() - t0
                ingest["reference_rows_per_s"] = rp["rows_total"] / dt
                ingest["reference_sample_rows"] = rp["rows_total"]
            log(f"[rank {rank}] ingest: {ingest['rows_per_s'] / 1e6:.1f}M rows/s ({ingest['csv_GBps']:.2f} GB/s of CSV)")
        except Exception as e:  # a failure here must not lose the main measurement
            ingest = {"error": repr(e)}

    # ---- the FULL suffix array + LCP (itt_suffix_array, cap = infinity) of the same tokens, device
    # resident: the step builds only the capped SA mining needs; this times the rest
    sa_full = None
    if not args.no_sa_full and args.config != "C5":
        try:
            tok_h, _, names_h = ctx.build_token_sequence(drecs, res["main_stream"])
            n_tok = int(tok_h.size)
            dev_t = torch.device("cuda", dev)
            tok_d = torch.from_numpy(tok_h).to(dev_t)
            sa_d = torch.empty(n_tok + 1, dtype=torch.int32, device=dev_t)
            lcp_d = torch.empty(n_tok + 1, dtype=torch.int32, device=dev_t)
            del tok_h
            torch.cuda.synchronize(dev)

            def step_sa():
                ctx.suffix_array_device(tok_d.data_ptr(), n_tok, int(names_h.size), sa_d.data_ptr(), lcp_d.data_ptr())
            step_sa()
            ms_sa, _ = timed(step_sa, 3)
            ctx.set_profiling(True)
            ctx.reset_stats()
            step_sa()
            st_sa = ctx.kernel_stats()
            ctx.set_profiling(False)
            rounds = st_sa.get("sa_rank_update", {}).get("launches", 0) - 1
            sa_full = {"ms": ms_sa / 3, "tokens": n_tok, "suffixes_per_s": (n_tok + 1) / (ms_sa / 3 / 1000.0),
                       "doubling_rounds": int(rounds),
                       "kernels_ms": {k: round(v["total_ms"], 3) for k, v in
                                      sorted(st_sa.items(), key=lambda kv: -kv[1]["total_ms"])[:6]}}
            del tok_d, sa_d, lcp_d
            log(f"[rank {rank}] full SA+LCP: {sa_full['ms']:.2f} ms ({rounds} doubling rounds)")
        except Exception as e:  # noqa: BLE001 (must not lose the main measurement)
            sa_full = {"error": repr(e)[:300]}

    # ---- CPU baseline (rank 0, N=1 only): the reference on a bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            ev, cinfo, sample, _, extra = cpu_reference_run(args.config, CPU_SAMPLE_ITERS[args.config], 1, 0, iters)
            cpu = {"value": ev, "unit": "events/s", "cores": 1, "kind": "reference", "sample": sample, **extra}
        except Exception as e:  # the reference library must be prebuilt in this container
            cpu = {"value": None, "unit": "events/s", "cores": 1, "kind": "reference", "sample": f"unavailable: {e}"}

    if rank == 0:
        L = res["loops"][0]
        line = {
            "metric": METRIC, "value": value, "unit": "events/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic", "warmup_extra_steps": extra_warmup,
            "config": {"workload": workload, "events": n_events, "tokens": info["n_main"],
                       "parallelism": f"replicas{world}" if world > 1 else "single",
                       "l2": "inputs larger than L2 (%.2f GB resident columns)" % (drecs.nbytes / 1e9),
                       "mined": {"pattern_length": L["pattern_length"], "pattern_count": L["pattern_count"],
                                 "iterations_found": int(L["rows"].shape[0])}},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary(),
            "gpu_launches": int(launches), "kernels": kernel_table, "op_profile": op_profile,
            "memory": memory, "ingest": ingest, "sa_full": sa_full,
        }
    drecs.free()
    return line if rank == 0 else None




if __name__ == "__main__":
    sys.exit(main())
