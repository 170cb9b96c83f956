import os, sys
sys.path.insert(0, "/root/repo")
from paper_1707_03750_b200 import cuda, synth
cfg = sys.argv[1]
ctx = cuda.Context(0)
recs, info = synth.generate_config(cfg)
it = synth.CONFIGS[cfg]["iterations"]
d = ctx.upload(recs)
for rep in range(4):
    ctx.set_profiling(True); ctx.reset_stats()
    ctx.analyze_raw(d, [it])
    st = ctx.kernel_stats()
    print(rep, {k: round(v["total_ms"], 3) for k, v in st.items() if k.startswith("intern")})
