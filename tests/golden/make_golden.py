#!/usr/bin/env python3
"""Generate tests/golden/*.json from the REFERENCE itself (oracle/_ref, compiled in place from
/root/reference/proj/include by oracle/Makefile).  Run in the CPU container:

    make -C oracle && python tests/golden/make_golden.py

The fixtures travel to the GPU box (the reference sources do not); the GPU parity tests and the
oracle pinning tests compare against them.  Doubles are stored as float.hex() for bit-exactness.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.bindings import CheckerError, ref  # noqa: E402
from paper_1707_03750_b200 import synth  # noqa: E402


def tok_of(s):
    return [ord(c) for c in s]


def with_init(init_len, body):  # test_mine.cpp:36-41
    return [1000 + i for i in range(init_len)] + list(body)


def repeat(unit, times):  # test_mine.cpp:43-46
    return list(unit) * times


def mine_case(R, tokens, loops, multi):
    n_names = max(tokens) + 1 if tokens else 0  # seq_of: names 0..max_token (test_mine.cpp:14-26)
    try:
        res = R.mine_patterns(tokens, n_names, loops, multi=multi)
        return {"ok": res}
    except CheckerError as e:
        return {"error": e.kind, "message": str(e)}


def token_cases(R):
    rng = np.random.default_rng(20261018)
    cases = []
    # reference known answers (test_suffix_tree.cpp, test_mine.cpp, test_match.cpp)
    fixed = [
        ("banana", tok_of("banana"), -1),
        ("banana_term_max", tok_of("banana"), 200),
        ("single", [7], -1),
        ("run12", [3] * 12, -1),
        ("init_body", [900, 901, 1, 2, 3, 1, 2, 3, 1, 2, 3], 902),
        ("tandem", [1, 2, 1, 2, 1, 2], 3),
        ("eps_doubling", with_init(30, repeat([1, 2, 3], 7)), 1030),
        ("distinct", [1, 2, 3, 4, 5, 6], 7),
        ("multi_loop", repeat([10, 11], 50) + repeat([20, 21, 22], 20), 23),
        ("ambiguous", with_init(40, repeat([1, 2, 3], 10)), 1040),
        ("match_golden", [1, 2, 3, 1, 2, 9, 3, 1, 2, 3], 10),
    ]
    for t in range(40):
        n = int(rng.integers(1, 260))
        a = int(rng.integers(1, 7))
        s = rng.integers(0, a, n)
        if t % 3 == 0:
            per = rng.integers(0, a, int(rng.integers(1, 9)))
            s = np.tile(per, n // len(per) + 1)[:n]
        fixed.append((f"random{t}", [int(x) for x in s], a))
    for name, tokens, term in fixed:
        sa, lcp = R.suffix_array(tokens, term)
        c = {"name": name, "tokens": tokens, "term": term, "sa": sa.tolist(), "lcp": lcp.tolist(), "repeats": [],
             "mine": [], "match": []}
        for mc, ml in [(2, 10), (2, 2), (3, 5), (99, 10)]:
            c["repeats"].append({"min_count": mc, "max_len": ml,
                                 "out": sorted(R.enumerate_repeats(tokens, term, mc, ml))})
        for iters in (2, 3, 5, 7, 10):
            c["mine"].append({"loops": [[iters, 1]], "multi": False, **mine_case(R, tokens, [(iters, 1)], False)})
        c["mine"].append({"loops": [[50, 1], [20, 1]], "multi": True, **mine_case(R, tokens, [(50, 1), (20, 1)], True)})
        c["mine"].append({"loops": [[10, 1], [11, 1]], "multi": True, **mine_case(R, tokens, [(10, 1), (11, 1)], True)})
        c["mine"].append({"loops": [[10, 1], [10, 1]], "multi": True, **mine_case(R, tokens, [(10, 1), (10, 1)], True)})
        c["mine"].append({"loops": [[4, 3]], "multi": False, **mine_case(R, tokens, [(4, 3)], False)})
        for plen, k0 in [(1, 0), (3, 1), (4, 2), (2, 0)]:
            p = tokens[:plen] if len(tokens) >= plen else tokens
            c["match"].append({"pattern": p, "k0": k0, "spans": R.approx_match(tokens, p, k0).tolist()})
        if name == "match_golden":
            c["match"].append({"pattern": [1, 2, 3], "k0": 1, "spans": R.approx_match(tokens, [1, 2, 3], 1).tolist()})
        cases.append(c)
    return cases


TRACE_CASES = [
    ("C1", dict(), [100], {}),
    ("C1_noise_shuffled", dict(noise_frac=0.05, shuffle_window=64, seed=11), [100], {}),
    ("C1_minority_device", dict(minority_frac=0.1, seed=12, iterations=50), [50], {}),
    ("C1_body_inserts", dict(body_inserts=2, insert_prob=0.3, seed=13), [100], {}),
    ("C1_k0_override", dict(body_inserts=2, insert_prob=0.3, seed=14), [100], {"k0": 0}),
    ("C1_eps_doubling", dict(seed=15, iterations=60), [64], {}),
    ("C1_small_body", dict(seed=16, iterations=300, body_len=7, vocab=5), [300], {}),
    ("C1_not_iterative", dict(seed=17, iterations=40), [1000], {}),
    ("C1_invalid_iters", dict(seed=18, iterations=40), [1], {}),
    ("C1_main_override_copy", dict(seed=19, iterations=30), [30], {"main_stream": 14}),
    ("C1_main_override_absent", dict(seed=19, iterations=30), [30], {"main_stream": 99}),
    ("C1_overlapping_kernels", dict(seed=20, intra_lo=-300, intra_hi=400), [100], {}),
    ("C1_negative_intervals", dict(seed=21, inter_lo=-6000, inter_hi=3000), [100], {}),
    ("C1_two_kernel_streams", dict(seed=22, extra_stream_frac=0.02), [100], {}),
    ("C1_multi_loop", dict(seed=23, iterations=40), [40, 20], {}),
    ("C1_multi_loop_dup", dict(seed=23, iterations=40), [40, 40], {}),
    ("C1_eps0_4", dict(seed=24, iterations=50), [64], {"epsilon0": 4}),
]


def trace_cases(R):
    out = []
    for name, gen, loops, opts in TRACE_CASES:
        kw = dict(synth.CONFIGS["C1"])
        kw.update(gen)
        recs, info = synth.generate(**kw)
        case = {"name": name, "generator": kw, "loops": loops, "opts": opts, "info": info}
        try:
            r = R.analyze(recs, loops, epsilon0=opts.get("epsilon0", 1), k0=opts.get("k0", -1),
                          main_stream=opts.get("main_stream", -1))
            case["streams"] = [list(s[:2]) + [list(s[2])] + list(s[3:]) for s in r["streams"]]
            case["main_stream"] = r["main_stream"]
            case["warnings"] = r["warnings"]
            case["summary_json"] = r["summary_json"]
            case["details_csv"] = r["details_csv"]
            case["loops_out"] = []
            for L in r["loops"]:
                iters = [[it[0], it[1], it[2], it[3], it[4], it[5], it[6], it[7], it[8], it[9], float(it[10]).hex(),
                          float(it[11]).hex()] for it in L["iters"]]
                case["loops_out"].append({k: L[k] for k in ("iterations_declared", "pattern_length", "pattern_count",
                                                            "epsilon_used", "first_token", "k0_used")}
                                         | {"iters": iters,
                                            "avg": [float(L[k]).hex() for k in ("avg_interval_ns", "avg_overlap",
                                                                                 "avg_operation_ns", "avg_size_bytes")],
                                            "max_interval_ns": L["max_interval_ns"],
                                            "insufficient_intervals": L["insufficient_intervals"],
                                            "diagnosis": L["diagnosis"]})
        except CheckerError as e:
            case["error"] = e.kind
            case["message"] = str(e)
        # token-level reference outputs on the same trace
        tok, ri, names = R.build_token_sequence(recs, 13)
        case["tokens_sha"] = int(np.bitwise_xor.reduce(tok.astype(np.uint64) * np.arange(1, tok.size + 1,
                                                                                        dtype=np.uint64)))
        case["n_tokens"] = int(tok.size)
        case["n_names"] = int(names.size)
        out.append(case)
    return out


def reference_render_goldens():
    """The reference's own rendering goldens (tests/golden/*, report.hpp byte format), kept as
    fixtures so the CPU suite can pin the host renderer without the reference sources."""
    src = "/root/reference/proj/tests/golden"
    for name in ("summary_golden.json", "details_golden.csv"):
        p = os.path.join(src, name)
        if os.path.exists(p):
            with open(p, "rb") as f, open(os.path.join(HERE, "reference_" + name), "wb") as g:
                g.write(f.read())


def main():
    reference_render_goldens()
    R = ref()
    with open(os.path.join(HERE, "token_cases.json"), "w") as f:
        json.dump(token_cases(R), f, separators=(",", ":"))
    with open(os.path.join(HERE, "trace_cases.json"), "w") as f:
        json.dump(trace_cases(R), f, indent=0)
    print("wrote", os.listdir(HERE))


if __name__ == "__main__":
    main()
