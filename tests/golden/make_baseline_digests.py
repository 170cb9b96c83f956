#!/usr/bin/env python3
"""Reference digests at BASELINE scale -> tests/golden/baseline_digests.json (TEST INFRASTRUCTURE).

Runs oracle/_ref/ref_digest (the unmodified reference compiled in place, oracle/Makefile) on the
full C2 (10.6M events) and C3 (100M events) traces of the repo's generator and records SHA-256
digests of what the reference produces:

* ``analyze``: the stock ``analyze_trace`` (pipeline.hpp:34-134): summary JSON exactly as the CLI
  writes it (report.hpp:304), details CSV (report.hpp:191-220), and the mined pattern's integers;
* ``sa``: the main-stream token ids (streams.hpp:147-169), the suffix array read off
  ``SuffixTree(tokens, V)`` (DFS in child-key order) and Kasai's LCP over it.

The GPU tests (tests/test_gpu_baseline.py) regenerate the same traces on the box (the generator
is deterministic, libitt_synth.so), run the device path and compare digests: full-size,
bit-exact parity without shipping gigabytes of fixtures.  The reference does not exist on the
GPU box; this script runs here, once, and its output is committed.

    python tests/golden/make_baseline_digests.py [C2] [C3]      (C3 needs ~50 GB of RAM, ~10 min)
"""
from __future__ import annotations

import hashlib
import json
import os
import subprocess
import sys
import tempfile
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
TOOL = os.path.join(ROOT, "oracle", "_ref", "ref_digest")
OUT = os.path.join(HERE, "baseline_digests.json")


def cfg_args(name):
    from paper_1707_03750_b200 import synth
    c = dict(noise_frac=0.0, shuffle_window=0)
    c.update(synth.CONFIGS[name])
    return [str(c["seed"]), str(c["iterations"]), str(c["body_len"]), str(c["vocab"]), repr(c["noise_frac"]),
            str(c["shuffle_window"])], c


def sha(path, chunk=1 << 24):
    h = hashlib.sha256()
    with open(path, "rb") as f:
        while True:
            b = f.read(chunk)
            if not b:
                break
            h.update(b)
    return h.hexdigest()


def kv(path):
    d = {}
    for ln in open(path):
        k, v = ln.split()
        d[k] = float(v) if "." in v or "e" in v else int(v)
    return d


def run(name):
    args, c = cfg_args(name)
    rec = {"generator": c}
    with tempfile.TemporaryDirectory() as td:
        for mode in ("analyze", "sa"):
            t0 = time.time()
            subprocess.run([TOOL, mode, td] + args, check=True)
            print(f"{name} {mode}: {time.time() - t0:.0f} s", flush=True)
        a = kv(os.path.join(td, "pattern.txt"))
        s = kv(os.path.join(td, "sa.txt"))
        rec["analyze"] = {"summary_json_sha256": sha(os.path.join(td, "summary.json")),
                          "details_csv_sha256": sha(os.path.join(td, "details.csv")),
                          "details_csv_bytes": os.path.getsize(os.path.join(td, "details.csv")),
                          **{k: a[k] for k in ("events", "pattern_length", "pattern_count", "epsilon_used",
                                               "first_token", "k0_used", "iterations_found", "main_stream")},
                          "reference_seconds": round(a["analyze_s"], 1)}
        with open(os.path.join(td, "summary.json")) as f:
            rec["analyze"]["summary_json"] = f.read()  # a few KB: readable diff on mismatch
        rec["sa"] = {"tokens": s["tokens"], "terminator": s["terminator"], "main_stream": s["main_stream"],
                     "tokens_i32_sha256": sha(os.path.join(td, "tokens.i32")),
                     "sa_u32_sha256": sha(os.path.join(td, "sa.u32")),
                     "lcp_u32_sha256": sha(os.path.join(td, "lcp.u32")),
                     "reference_tree_seconds": round(s["tree_s"], 1)}
    return rec


def main():
    names = sys.argv[1:] or ["C2", "C3"]
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    data["_about"] = ("SHA-256 of the reference's own outputs (oracle/_ref/ref_digest: stock analyze_trace, "
                      "SuffixTree leaf order + Kasai) on the full BASELINE traces; made by "
                      "tests/golden/make_baseline_digests.py")
    for n in names:
        data[n] = run(n)
        with open(OUT, "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)
            f.write("\n")
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
