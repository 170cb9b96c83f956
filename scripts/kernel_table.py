"""Per-kernel table of one analyze (default C3): launches, total ms, us/launch, declared GB/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_03750_b200 import cuda, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
ctx = cuda.Context(0)
recs, info = synth.generate_config(cfg)
it = synth.CONFIGS[cfg]["iterations"]
d = ctx.upload(recs)
for _ in range(3):
    ctx.analyze_raw(d, [it])
ctx.set_profiling(True)
ctx.reset_stats()
ctx.analyze_raw(d, [it])
st = ctx.kernel_stats()
tot = sum(v["total_ms"] for v in st.values())
print(f"{cfg}: kernel sum {tot:.3f} ms")
for k, v in sorted(st.items(), key=lambda kv: -kv[1]["total_ms"]):
    if v["total_ms"] < 0.02:
        continue
    print(f"{k:24s} {v['launches']:4d} {v['total_ms']:8.3f} ms {1000 * v['total_ms'] / v['launches']:9.1f} us "
          f"{v['bytes'] / (v['total_ms'] / 1000) / 1e9 if v['total_ms'] else 0:8.0f} GB/s")
