"""H2D bandwidth probe: torch pinned tensor vs cudaHostRegister'd numpy buffer (1 GiB chunks)."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1707_03750_b200 import cuda
ctx = cuda.Context(0)
GB = 1 << 30
for size in (GB, 4 * GB):
    src = torch.empty(size, dtype=torch.uint8).pin_memory()
    dst = torch.empty(size, dtype=torch.uint8, device="cuda")
    dst.copy_(src, non_blocking=True); torch.cuda.synchronize()
    t = time.perf_counter(); dst.copy_(src, non_blocking=True); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"torch pinned {size/GB:.0f} GiB: {size/dt/1e9:.1f} GB/s", flush=True)
    a = np.ones(size, np.uint8)
    t = time.perf_counter(); ctx.register_host(a); print(f"  register {size/GB:.0f} GiB: {time.perf_counter()-t:.2f}s")
    p = C.c_void_p()
    L = cuda.lib()
    ctx._check(L.itt_device_alloc(ctx.h, size, C.byref(p)))
    for rep in range(2):
        t = time.perf_counter(); ctx._check(L.itt_memcpy_h2d(ctx.h, p, a.ctypes.data, size)); ctx.synchronize(); dt = time.perf_counter() - t
        print(f"  registered numpy via itt_memcpy_h2d: {size/dt/1e9:.1f} GB/s", flush=True)
    ctx.unregister_host(a)
    t = time.perf_counter(); ctx._check(L.itt_memcpy_h2d(ctx.h, p, a.ctypes.data, size)); ctx.synchronize(); dt = time.perf_counter() - t
    print(f"  pageable numpy: {size/dt/1e9:.1f} GB/s", flush=True)
    L.itt_device_free(ctx.h, p)
