"""Where the C2 step's stream sits idle: ITT_TIMELINE=1 books the gap between consecutive
profiled launches as "gap:<prev>-><next>".  Prints kernel time, gap time and the largest gaps."""
import os, sys
os.environ["ITT_TIMELINE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_03750_b200 import cuda, synth

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
iters = {"C1": 100, "C2": 50_000, "C3": 20_000, "C4": 500}[cfg]
ctx = cuda.Context(0)
recs, info = synth.generate_config(cfg)
d = ctx.upload(recs)
for _ in range(3):
    ctx.analyze_raw(d, [iters])
steps = 5
ctx.set_profiling(True)
ctx.reset_stats()
for _ in range(steps):
    ctx.analyze_raw(d, [iters])
st = ctx.kernel_stats()
ctx.set_profiling(False)
kern = {k: v for k, v in st.items() if not k.startswith("gap:")}
gaps = {k: v for k, v in st.items() if k.startswith("gap:")}
kt = sum(v["total_ms"] for v in kern.values()) / steps
gt = sum(v["total_ms"] for v in gaps.values()) / steps
print(f"{cfg}: kernels {kt:.3f} ms/step, stream idle between launches {gt:.3f} ms/step "
      f"({sum(v['launches'] for v in gaps.values()) // steps} gaps/step)")
for k, v in sorted(gaps.items(), key=lambda kv: -kv[1]["total_ms"])[:25]:
    print(f"  {v['total_ms'] / steps * 1000:8.1f} us  x{v['launches'] // steps:<3d} {k}")
