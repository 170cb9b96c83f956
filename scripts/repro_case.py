"""Repro a fuzz mismatch: prints the GPU vs reference outputs' first differences."""
import difflib, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.bindings import CheckerError, ref
from paper_1707_03750_b200 import cuda, itertrace, synth
ctx = cuda.Context(0)
R = ref()
cases = [
    ({'seed': 824344830, 'iterations': 167, 'body_len': 116, 'vocab': 93, 'init_ops': 16, 'noise_frac': 0.0, 'shuffle_window': 0, 'body_inserts': 0, 'insert_prob': 0.26079195147949064, 'minority_frac': 0.0, 'extra_stream_frac': 0.0}, [167], {'epsilon0': 2, 'k0': None, 'main_stream': None}),
    ({'seed': 781422210, 'iterations': 159, 'body_len': 10, 'vocab': 6, 'init_ops': 0, 'noise_frac': 0.1, 'shuffle_window': 64, 'body_inserts': 3, 'insert_prob': 0.16670136963472088, 'minority_frac': 0.0, 'extra_stream_frac': 0.0}, [159], {'epsilon0': 1, 'k0': None, 'main_stream': None}),
    ({'seed': 99822296, 'iterations': 211, 'body_len': 46, 'vocab': 105, 'init_ops': 0, 'noise_frac': 0.0, 'shuffle_window': 0, 'body_inserts': 3, 'insert_prob': 0.17847418421144595, 'minority_frac': 0.0, 'extra_stream_frac': 0.1}, [211], {'epsilon0': 2, 'k0': None, 'main_stream': None}),
]
for kw, loops, opts in cases:
    recs, _ = synth.generate(**kw)
    try:
        r = itertrace.analyze_trace(ctx, recs, loops, **opts)
        got = (r.summary_json(), r.details_csv(0))
    except itertrace.AnalyzeError as e:
        got = ("ERR " + e.kind, str(e))
    try:
        w = R.analyze(recs, loops, epsilon0=opts["epsilon0"], k0=-1 if opts["k0"] is None else opts["k0"],
                      main_stream=-1 if opts["main_stream"] is None else opts["main_stream"])
        want = (w["summary_json"], w["details_csv"])
    except CheckerError as e:
        want = ("ERR " + e.kind, str(e))
    print("=== case seed", kw["seed"])
    for g, wv, name in zip(got, want, ("summary", "details")):
        if g != wv:
            d = list(difflib.unified_diff(wv.splitlines(), g.splitlines(), "ref", "gpu", n=1, lineterm=""))
            print(name, "DIFF:\n" + "\n".join(d[:30]))
    raw = ctx.analyze_raw(recs, loops, opts["epsilon0"], -1 if opts["k0"] is None else opts["k0"], -1)
    print("gpu pattern len/count/first/eps:", [(L["pattern_length"], L["pattern_count"], L["first_token"], L["epsilon_used"], L["rows"].shape[0]) for L in raw["loops"]])
