"""Development parity sweep: CUDA path vs the reference (oracle/_ref) on random + synthetic inputs."""
import sys, time, traceback
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_1707_03750_b200 import cuda, synth
from oracle.bindings import ref, CheckerError

ctx = cuda.Context(0)
R = ref()
rng = np.random.default_rng(7)
fails = 0
def check(name, ok, info=""):
    global fails
    if not ok:
        fails += 1
        print("FAIL", name, info)

# banana
tok = [ord(c) for c in "banana"]
sa, lcp = ctx.suffix_array(tok, 200)
rsa, rlcp = R.suffix_array(tok, 200)
check("banana sa", np.array_equal(sa, rsa) and np.array_equal(lcp, rlcp), (sa, rsa, lcp, rlcp))
check("banana rep", sorted(ctx.enumerate_repeats(tok, -1, 2, 10)) == sorted(R.enumerate_repeats(tok, -1, 2, 10)))
t0 = time.time()
for trial in range(400):
    n = int(rng.integers(1, 400)); a = int(rng.integers(1, 7))
    s = rng.integers(0, a, n).astype(np.int32)
    if trial % 3 == 0:
        per = rng.integers(0, a, int(rng.integers(1, 9)))
        s = np.tile(per, n // len(per) + 1)[:n].astype(np.int32)
    sa, lcp = ctx.suffix_array(s, a)
    rsa, rlcp = R.suffix_array(s, a)
    check(f"sa {trial}", np.array_equal(sa, rsa) and np.array_equal(lcp, rlcp), (s.tolist()[:50],))
    mc = int(rng.integers(2, 5)); ml = int(rng.integers(1, 15))
    check(f"rep {trial}", sorted(ctx.enumerate_repeats(s, -1, mc, ml)) == sorted(R.enumerate_repeats(s, -1, mc, ml)))
    it = int(rng.integers(2, 9))
    if n >= 2:
        def run(f):
            try: return f()
            except (cuda.IttError, CheckerError) as e: return ("E", e.kind, str(e))
        g = run(lambda: ctx.mine_patterns(s, a, [(it, 1)]))
        r = run(lambda: R.mine_patterns(s, a, [(it, 1)]))
        check(f"mine {trial}", g == r, (g, r))
    p = s[int(rng.integers(0, n)):][:int(rng.integers(1, 8))]
    k0 = int(rng.integers(0, 3))
    g = ctx.approx_match(s, p, k0); r = R.approx_match(s, p, k0)
    check(f"match {trial}", np.array_equal(g, r), (g, r))
print("random sweep", time.time() - t0, "s; fails", fails)

for name, kw in [("C1", {}), ("C1n", dict(noise_frac=0.05, shuffle_window=64, seed=11)),
                 ("dev", dict(minority_frac=0.1, seed=12, iterations=50)),
                 ("ins", dict(body_inserts=2, insert_prob=0.3, seed=13))]:
    recs, info = synth.generate_config("C1", **kw)
    t0 = time.time()
    try:
        g = ctx.analyze_raw(recs, [recs_i := (50 if name == "dev" else 100)])
    except Exception as e:
        traceback.print_exc(); fails += 1; continue
    gt = time.time() - t0
    r = R.analyze(recs, [recs_i])
    check(name + " streams", g["streams"] == r["streams"], (g["streams"], r["streams"]))
    check(name + " main", g["main_stream"] == r["main_stream"])
    L, RL = g["loops"][0], r["loops"][0]
    for k in ("pattern_length", "pattern_count", "epsilon_used", "first_token", "k0_used"):
        check(name + " " + k, L[k] == RL[k], (L[k], RL[k]))
    rows = L["rows"]
    check(name + " n_iter", len(rows) == len(RL["iters"]), (len(rows), len(RL["iters"])))
    bad = 0
    for i, (gr, rr) in enumerate(zip(rows, RL["iters"])):
        # ref_iter: index,start,end,extra,t_start,t_end,interval,htod,has_int,has_ov,ov,gap
        if (gr[0], gr[1], gr[2], gr[3], gr[4], gr[7]) != (rr[1], rr[2], rr[3], rr[4], rr[5], rr[7]): bad += 1; continue
        if gr[10] != rr[8] or (gr[10] and gr[5] != rr[6]): bad += 1; continue
        ov = (gr[6] / gr[5]) if (gr[10] and gr[5] > 0) else None
        if (ov is None) != (not rr[9]) or (ov is not None and ov != rr[10]): bad += 1; continue
        gm = gr[8] / gr[9] if gr[9] > 0 else 0.0
        if gm != rr[11]: bad += 1
    check(name + " rows", bad == 0, bad)
    print(name, info, "gpu analyze %.3fs" % gt, "ref %.3fs" % (r["times"]["total_ms"] / 1000 if r["times"]["total_ms"] else 0))
print("TOTAL FAILS", fails)
