"""Two analyzes of a BASELINE trace (default C3), for ncu captures: python scripts/c3_once.py [C3] [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_03750_b200 import cuda, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
kw = {"iterations": int(sys.argv[2])} if len(sys.argv) > 2 else {}
recs, info = synth.generate_config(cfg, **kw)
it = kw.get("iterations", synth.CONFIGS[cfg]["iterations"])
ctx = cuda.Context(0)
d = ctx.upload(recs)
for _ in range(2):
    r = ctx.analyze_raw(d, [it])
ctx.synchronize()
print(cfg, info["n"], r["loops"][0]["pattern_length"], r["loops"][0]["pattern_count"])
