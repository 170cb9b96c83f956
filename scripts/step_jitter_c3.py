"""C3 step-time stability: 3 timed blocks of 10 analyzes each, without and with an nvidia-smi
clock sampler running (-lms 200 / 1000), device-timed with CUDA events on the library stream."""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1707_03750_b200 import cuda, synth  # noqa: E402

ctx = cuda.Context(0)
CFG = sys.argv[1] if len(sys.argv) > 1 else "C3"
IT = {"C2": 50_000, "C3": 20_000}[CFG]
recs, info = synth.generate_config(CFG)
d = ctx.upload(recs)
stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=torch.device("cuda", 0))
for _ in range(20):
    ctx.analyze_raw(d, [IT])


def block(k=10):
    ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(k):
        ctx.analyze_raw(d, [IT])
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / k


for mode in ("none", "200", "none", "1000", "none", "200"):
    p = None
    if mode != "none":
        q = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")  # bench.py's ClockSampler query
        p = subprocess.Popen(["nvidia-smi", "-i", "0", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", mode],
                             stdout=subprocess.DEVNULL)
        time.sleep(0.5)
    print(mode, [round(block(), 2) for _ in range(3)], flush=True)
    if p:
        p.terminate()
        p.wait()
