"""a12 op profile increment at C3: blocks of analyze with and without ITT_ANALYZE_OP_PROFILE."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1707_03750_b200 import cuda, synth  # noqa: E402

CFG = sys.argv[1] if len(sys.argv) > 1 else "C3"
IT = {"C2": 50_000, "C3": 20_000}[CFG]
ctx = cuda.Context(0)
recs, info = synth.generate_config(CFG)
d = ctx.upload(recs)
stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=torch.device("cuda", 0))


def block(k, **kw):
    ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(k):
        ctx.analyze_raw(d, [IT], **kw)
    e1.record(stream)
    e1.synchronize()
    return round(e0.elapsed_time(e1) / k, 2)


for _ in range(5):
    ctx.analyze_raw(d, [IT])
    ctx.analyze_raw(d, [IT], op_profile=True)
for kw in ({}, {"op_profile": True}, {}, {"op_profile": True}, {"op_profile": "cells"}):
    print(kw, [block(5, **kw) for _ in range(3)], flush=True)
ctx.set_profiling(True)
ctx.reset_stats()
ctx.analyze_raw(d, [IT], op_profile=True)
st = ctx.kernel_stats()
print({k: round(v["total_ms"], 3) for k, v in sorted(st.items(), key=lambda kv: -kv[1]["total_ms"])[:8]})
