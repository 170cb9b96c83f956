"""Streamed-names probe: stage times of analyze with names in pinned host memory (C5 shape)."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1707_03750_b200 import cuda, synth
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000
recs, info = synth.generate_config("C5", iterations=iters)
print(info, flush=True)
ctx = cuda.Context(0)
d = ctx.upload(recs, names_host=os.environ.get("DEVNAMES") is None)
if os.environ.get("DEVNAMES") and os.environ.get("PIN"):
    ctx.register_host(recs.name_bytes)  # pinned but unused: does registration alone disturb timing?
L = cuda.lib()
p = C.c_void_p()
nb = recs.name_bytes.nbytes
ctx._check(L.itt_device_alloc(ctx.h, nb, C.byref(p)))
t = time.perf_counter(); ctx._check(L.itt_memcpy_h2d(ctx.h, p, recs.name_bytes.ctypes.data, nb)); ctx.synchronize()
print(f"plain copy of the registered names: {nb / (time.perf_counter() - t) / 1e9:.1f} GB/s", flush=True)
L.itt_device_free(ctx.h, p)
ctx.set_profiling(True)
for _ in range(8):
    ctx.reset_stats()
    t = time.perf_counter(); ctx.analyze_raw(d, [iters]); print("total %.1f ms" % (1000 * (time.perf_counter() - t)), flush=True)
    st = ctx.kernel_stats()
    top = sorted(st.items(), key=lambda kv: -kv[1]["total_ms"])[:4]
    print("   kernels " + ", ".join(f"{k}={v['total_ms']:.1f}ms/{v['launches']}" for k, v in top), flush=True)
