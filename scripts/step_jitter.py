"""Per-step times of the C2 device-resident analyze (CUDA events on the library stream), with
and without the nvidia-smi sampler running, to see where step-time jitter comes from."""
import os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1707_03750_b200 import cuda, synth
recs, info = synth.generate_config("C2")
ctx = cuda.Context(0)
d = ctx.upload(recs)
stream = torch.cuda.ExternalStream(ctx.stream_ptr())
for _ in range(3):
    ctx.analyze_raw(d, [50_000])
def run(tag, k=20):
    ts = []
    for _ in range(k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t = time.perf_counter()
        e0.record(stream); ctx.analyze_raw(d, [50_000]); e1.record(stream); e1.synchronize()
        ts.append((e0.elapsed_time(e1), 1000 * (time.perf_counter() - t)))
    print(tag, " ".join(f"{a:.2f}" for a, _ in ts), flush=True)
run("plain   ")
p = subprocess.Popen(["nvidia-smi", "--query-gpu=timestamp,clocks.sm", "--format=csv,noheader", "-lms", "20"],
                     stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
time.sleep(0.5)
run("smi20   ")
p.terminate()
run("plain   ")
