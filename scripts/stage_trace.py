"""Per-stage wall times of one C2 itt_analyze (ITT_TRACE=1), device-resident inputs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_03750_b200 import cuda, synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
recs, info = synth.generate_config(cfg)
iters = synth.CONFIGS[cfg]["iterations"]
ctx = cuda.Context(0)
d = ctx.upload(recs)
for _ in range(3):
    ctx.analyze_raw(d, [iters], op_profile=bool(os.environ.get('OPPROF')))
os.environ["ITT_TRACE"] = "1"
print("---- traced run", file=sys.stderr)
t = time.perf_counter(); ctx.analyze_raw(d, [iters], op_profile=bool(os.environ.get('OPPROF'))); print("total %.2f ms" % (1000 * (time.perf_counter() - t)), file=sys.stderr)
