"""Onesweep radix pass sweep: per-pass time and GB/s (algorithmic 16 B/element/pass) for each
tile shape (ITT_RADIX_CFG), n = 10M keys, 24 and 32 key bits; validated against numpy."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1707_03750_b200 import cuda

ctx = cuda.Context(0)
n = int(os.environ.get("N", 10_000_001))
rng = np.random.default_rng(1)
res = {"cfg": int(os.environ.get("ITT_RADIX_CFG", "0")), "n": n}
for bits in (24, 32):
    keys = rng.integers(0, 1 << bits, n, dtype=np.uint64).astype(np.uint32)
    vals = np.arange(n, dtype=np.uint32)
    want = np.argsort(keys, kind="stable")
    dk = torch.from_numpy(keys.view(np.int32)).cuda()
    dv = torch.from_numpy(vals.view(np.int32)).cuda()
    for rep in range(4):
        k2 = dk.clone(); v2 = dv.clone(); torch.cuda.synchronize()
        ctx.set_profiling(rep == 3); ctx.reset_stats()
        ctx.radix_sort_device(k2.data_ptr(), v2.data_ptr(), n, 0, bits)
    st = ctx.kernel_stats(); ctx.set_profiling(False)
    one = st["radix_onesweep"]
    ok = np.array_equal(v2.cpu().numpy().view(np.uint32), want)
    res[f"bits{bits}"] = {"ok": bool(ok), "passes": one["launches"], "us_per_pass": 1000 * one["total_ms"] / one["launches"],
                          "GBps": one["bytes"] / (one["total_ms"] / 1000) / 1e9,
                          "hist_us": 1000 * st.get("radix_hist", {}).get("total_ms", 0)}
print(json.dumps(res))
