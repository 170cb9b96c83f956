"""How much host memory will cudaHostRegister pin on this box? (numpy buffers, filled)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1707_03750_b200 import cuda
ctx = cuda.Context(0)
for gb in [int(x) for x in sys.argv[1:]]:
    a = np.ones(gb << 30, np.uint8)
    t = time.perf_counter()
    try:
        ctx.register_host(a)
        print(f"{gb} GiB: registered in {time.perf_counter() - t:.1f}s", flush=True)
        ctx.unregister_host(a)
    except cuda.IttError as e:
        print(f"{gb} GiB: FAILED after {time.perf_counter() - t:.1f}s: {e}", flush=True)
    del a
