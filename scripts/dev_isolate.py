import sys, numpy as np
sys.path.insert(0, "/root/repo")
from paper_1707_03750_b200 import cuda, synth
from oracle.bindings import ref
ctx = cuda.Context(0); R = ref()
recs, info = synth.generate_config("C1", body_inserts=2, insert_prob=0.3, seed=13)
rt, rri, rn = R.build_token_sequence(recs, 13)
gt, gri, gn = ctx.build_token_sequence(recs, 13)
print("tokens equal", np.array_equal(rt, gt), "ri", np.array_equal(rri, gri), "names", np.array_equal(rn, gn), len(rn), len(gn))
if not np.array_equal(rt, gt):
    d = np.nonzero(rt != gt)[0]; print("first diff", d[:10], rt[d[:10]], gt[d[:10]])
V = len(rn)
sa, lcp = ctx.suffix_array(rt, V); rsa, rlcp = R.suffix_array(rt, V)
print("sa equal", np.array_equal(sa, rsa), "lcp equal", np.array_equal(lcp, rlcp))
print("mine gpu", [(len(p["tokens"]), p["count"], p["first_token"], p["epsilon_used"]) for p in ctx.mine_patterns(rt, V, [(100, 1)])])
print("mine ref", [(len(p["tokens"]), p["count"], p["first_token"], p["epsilon_used"]) for p in R.mine_patterns(rt, V, [(100, 1)])])
g = sorted(ctx.enumerate_repeats(rt, V, 2, 200)); r = sorted(R.enumerate_repeats(rt, V, 2, 200))
print("repeats equal", g == r, len(g), len(r))
if g != r:
    sg, sr = set(g), set(r); print("only gpu", sorted(sg - sr)[:10]); print("only ref", sorted(sr - sg)[:10])
# larger random strings
rng = np.random.default_rng(3); bad = 0
for t in range(30):
    n = int(rng.integers(2000, 30000)); a = int(rng.integers(2, 50))
    s = rng.integers(0, a, n).astype(np.int32)
    if t % 2: 
        per = rng.integers(0, a, int(rng.integers(5, 300))); s = np.tile(per, n // len(per) + 1)[:n].astype(np.int32)
        s[rng.integers(0, n, 20)] = a - 1
    sa, lcp = ctx.suffix_array(s, a); rsa, rlcp = R.suffix_array(s, a)
    ok1 = np.array_equal(sa, rsa) and np.array_equal(lcp, rlcp)
    g = sorted(ctx.enumerate_repeats(s, a, 2, 50)); r = sorted(R.enumerate_repeats(s, a, 2, 50))
    it = int(rng.integers(2, 60))
    def run(f):
        try: return f()
        except Exception as e: return ("E", getattr(e, "kind", None), str(e))
    gm = run(lambda: ctx.mine_patterns(s, a, [(it, 1)])); rm = run(lambda: R.mine_patterns(s, a, [(it, 1)]))
    if not (ok1 and g == r and gm == rm):
        bad += 1; print("big fail", t, n, a, ok1, g == r, gm == rm, len(g), len(r))
print("big random bad", bad)
