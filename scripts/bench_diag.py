"""Why bench.py's timed bracket runs slower than a steady loop: time blocks of K analyzes under
variants (result held vs dropped, torch.cuda.synchronize in the barrier, block length)."""
import gc
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1707_03750_b200 import cuda, synth  # noqa: E402

CFG = sys.argv[1] if len(sys.argv) > 1 else "C2"
IT = {"C2": 50_000, "C3": 20_000}[CFG]
torch.cuda.set_device(0)
ctx = cuda.Context(0)
recs, info = synth.generate_config(CFG)
d = ctx.upload(recs)
stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=torch.device("cuda", 0))
for _ in range(30):
    ctx.analyze_raw(d, [IT])


def block(k, hold, tsync, gc_off=False):
    if tsync:
        torch.cuda.synchronize(0)
    ctx.synchronize()
    if gc_off:
        gc.disable()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    res = None
    for _ in range(k):
        r = ctx.analyze_raw(d, [IT])
        if hold:
            res = r
        del r
    e1.record(stream)
    e1.synchronize()
    if gc_off:
        gc.enable()
    del res
    return round(e0.elapsed_time(e1) / k, 3)


for name, kw in [("drop", dict(hold=False, tsync=False)), ("hold", dict(hold=True, tsync=False)),
                 ("hold+tsync", dict(hold=True, tsync=True)), ("drop", dict(hold=False, tsync=False)),
                 ("hold+gcoff", dict(hold=True, tsync=True, gc_off=True))]:
    print(name, [block(20, **kw) for _ in range(4)], flush=True)
