"""Rank-update experiment: per-launch time of sa_rank_update with parts disabled (ITT_RANK_EXP:
1 = no second-key gather, 2 = no look-back, 4 = no scatter).  Timing only; results are wrong."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1707_03750_b200 import cuda
rng = np.random.default_rng(1)
body = rng.permutation(166)[:150].tolist() + rng.integers(0, 166, 50).tolist()
tokens = np.tile(np.array(body, np.int32), 50_000)
ctx = cuda.Context(0)
def run():
    try:
        ctx.suffix_array(tokens, 166)
    except cuda.IttError:
        pass
run()
ctx.set_profiling(True)
ctx.reset_stats()
run()
st = ctx.kernel_stats()
for k in ("sa_rank_update", "radix_onesweep"):
    v = st[k]
    print(f"exp={os.environ.get('ITT_RANK_EXP', '0')} {k}: {v['launches']} launches, {1000 * v['total_ms'] / v['launches']:.1f} us/launch")
