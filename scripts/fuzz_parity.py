"""Long randomized parity sweep against the live reference (not part of the test suite: minutes).

* traces: the TF-like generator over a wide config space (noise, shuffles, inserts, minority
  devices, extra kernel streams, multiple loops, k0 / epsilon0 / main-stream overrides), GPU
  analyze_trace vs the reference's analyze_trace: summary JSON + details CSV (or error kind +
  message) byte for byte;
* CSVs: the reference generator's CSV through the GPU parser + GPU analyze vs the reference CLI
  path;
* token strings: SA + LCP, enumerate_repeats, mining (incl. errors) vs the reference.
Usage: python scripts/fuzz_parity.py [seconds]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from oracle.bindings import CheckerError, ref
from paper_1707_03750_b200 import cuda, itertrace, synth

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 240.0
ctx = cuda.Context(0)
R = ref()
rng = np.random.default_rng(int(time.time()) & 0xFFFF)
t_end = time.time() + budget
counts = {"trace": 0, "csv": 0, "tokens": 0}
fails = []


def trace_case():
    iters = int(rng.integers(2, 300))
    kw = dict(seed=int(rng.integers(1, 1 << 30)), iterations=iters, body_len=int(rng.integers(1, 150)),
              vocab=int(rng.integers(1, 120)), init_ops=int(rng.integers(0, 20)),
              noise_frac=float(rng.choice([0.0, 0.02, 0.1])), shuffle_window=int(rng.choice([0, 0, 8, 64])),
              body_inserts=int(rng.integers(0, 4)), insert_prob=float(rng.random() * 0.4),
              minority_frac=float(rng.choice([0.0, 0.0, 0.05])), extra_stream_frac=float(rng.choice([0.0, 0.0, 0.1])))
    recs, _ = synth.generate(**kw)
    loops = [iters]
    if rng.random() < 0.15:
        loops.append(int(rng.integers(2, 50)))
    opts = dict(epsilon0=int(rng.choice([1, 1, 2, 3])), k0=None if rng.random() < 0.8 else int(rng.integers(0, 10)),
                main_stream=None if rng.random() < 0.9 else int(rng.choice([7, 13, 14, 21])))
    try:
        r = itertrace.analyze_trace(ctx, recs, loops, **opts)
        got = (r.summary_json(), r.details_csv(0))
    except itertrace.AnalyzeError as e:
        got = (e.kind, str(e))
    try:
        w = R.analyze(recs, loops, epsilon0=opts["epsilon0"], k0=-1 if opts["k0"] is None else opts["k0"],
                      main_stream=-1 if opts["main_stream"] is None else opts["main_stream"])
        want = (w["summary_json"], w["details_csv"])
    except CheckerError as e:
        want = (e.kind, str(e))
    return got == want, (kw, loops, opts)


def csv_case():
    iters = int(rng.integers(2, 120))
    plen = int(rng.integers(1, 30))
    try:
        text = R.synth_csv(seed=int(rng.integers(1, 1 << 30)), pattern_len=plen, iterations=iters,
                           vocab_size=plen + int(rng.integers(0, 20)), insert_prob=float(rng.random() * 0.3),
                           max_inserts=int(rng.integers(0, 3)), inside_pattern=bool(rng.random() < 0.3),
                           pathology=int(rng.integers(0, 3)))
    except ValueError:  # a config the reference generator itself rejects: nothing to compare
        return None, None
    want = R.analyze_csv(text, [iters], label="f.csv")
    try:
        r = itertrace.analyze_csv(ctx, text, [iters], trace_label="f.csv")
        got = (0, r.summary_json(), r.details_csv(0))
    except itertrace.AnalyzeError as e:
        got = ("err", str(e))
    w = (0, want["summary_json"], want["details_csv"]) if want["status"] == 0 else ("err", want["error"])
    return got == w, iters


def token_case():
    n = int(rng.integers(1, 3000))
    if rng.random() < 0.5:  # periodic with noise
        p = int(rng.integers(1, 60))
        body = rng.integers(0, int(rng.integers(1, 30)), p)
        tok = np.tile(body, n // p + 1)[:n].astype(np.int32)
        flip = rng.random(n) < rng.random() * 0.05
        tok[flip] = rng.integers(0, 40, int(flip.sum()))
    else:
        tok = rng.integers(0, int(rng.integers(1, 50)), n).astype(np.int32)
    term = int(tok.max()) + 1 + int(rng.integers(0, 3))
    sa, lcp = ctx.suffix_array(tok, term)
    wsa, wlcp = R.suffix_array(tok, term)
    ok = np.array_equal(sa, wsa) and np.array_equal(lcp, wlcp)
    iters = int(rng.integers(2, 40))
    loops = [(iters, int(rng.choice([1, 1, 2])))]
    try:
        g = ctx.mine_patterns(tok, term, loops)
    except cuda.IttError as e:
        g = (e.status, str(e))
    try:
        w = R.mine_patterns(tok, term, loops)
    except CheckerError as e:
        w = (e.status, str(e))
    return ok and g == w, (n, term, loops)


kinds = [("trace", trace_case), ("csv", csv_case), ("tokens", token_case)]
while time.time() < t_end:
    name, fn = kinds[int(rng.integers(0, 3))]
    try:
        ok, info = fn()
    except Exception as e:  # noqa: BLE001
        ok, info = False, repr(e)
    if ok is None:
        continue
    counts[name] += 1
    if not ok:
        fails.append((name, info))
        print("MISMATCH", name, info, flush=True)
print("fuzz:", counts, "mismatches:", len(fails), flush=True)
sys.exit(1 if fails else 0)
