"""C3 end to end from pinned host columns: names copied whole (MEM_HOST) vs streamed through the
device windows while hashing (MEM_HOST_STREAM_NAMES); events/s of each."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1707_03750_b200 import abi, cuda, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
it = synth.CONFIGS[cfg]["iterations"]
ctx = cuda.Context(0)
recs, info = synth.generate_config(cfg)
cols = [recs.start_ns, recs.duration_ns, recs.size_bytes, recs.flags, recs.stream, recs.name_off, recs.name_bytes]
if recs.device is not None:
    cols.append(recs.device)
for a in cols:
    ctx.register_host(a)
stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=torch.device("cuda", 0))
for mode, name in ((abi.MEM_HOST, "copy names"), (abi.MEM_HOST_STREAM_NAMES, "stream names")):
    for chunk in ((None,) if mode == abi.MEM_HOST else ("", str(256 << 20), str(64 << 20))):
        if chunk:
            os.environ["ITT_STREAM_CHUNK"] = chunk
        recs.mem = mode
        for _ in range(2):
            ctx.analyze_raw(recs, [it])
        ctx.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(3):
            ctx.analyze_raw(recs, [it])
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"{name:13s} chunk={chunk or 'default'}: {ms:.1f} ms, {info['n'] / ms / 1e3:.0f}M events/s", flush=True)
