"""The CLI mirror (paper_1707_03750_b200/cli.py) against the reference tool's contract
(tools/itertrace_main.cpp; cases restated from tests/test_cli.cpp): exit codes, the lines the
reference tests grep, byte-stable output, and — beyond the reference's own tests — summary JSON
and details CSV byte-identical to the reference's analyze on the same CSV, and the console text
rebuilt from the reference's report.  Argument errors are checked on CPU (they exit before a
device is touched); runs that analyze need the GPU."""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

from conftest import ROOT


def run(args, cwd=None):
    r = subprocess.run([sys.executable, "-m", "paper_1707_03750_b200.cli"] + args, cwd=cwd or ROOT,
                       stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True, timeout=600)
    return r.returncode, r.stdout


def test_argument_errors_exit_4(tmp_path):
    t = str(tmp_path / "x.csv")
    assert run(["analyze", "--trace", t])[0] == 4                                   # neither --iterations nor --loops
    assert run(["analyze", "--trace", t, "--iterations", "5", "--loops", "5"])[0] == 4
    assert run(["analyze", "--trace", t, "--iterations", "5", "--out-summary", "a", "--out-details", "a"])[0] == 4
    assert run(["analyze", "--trace", t, "--iterations", "5", "--bogus-flag"])[0] == 4
    assert run(["analyze", "--trace", t, "--iterations", "five"])[0] == 4
    assert run([])[0] == 4                                                         # a subcommand is required
    code, out = run(["--version"])
    assert code == 0 and out.strip() == "0.1.0"
    assert run(["analyze", "--help"])[0] == 0


@pytest.mark.gpu
def test_analyze_clean_trace(tmp_path, R):
    trace = tmp_path / "ok.csv"
    trace.write_bytes(R.synth_csv(seed=99, iterations=20, pattern_len=5))
    s, d = tmp_path / "ok_summary.json", tmp_path / "ok_details.csv"
    code, out = run(["analyze", "--trace", str(trace), "--iterations", "20", "--out-summary", str(s),
                     "--out-details", str(d)])
    assert code == 0, out
    assert "diagnosis: NONE" in out and "loop 1" in out
    want = R.analyze_csv(trace.read_bytes(), [20], label=str(trace))
    assert s.read_text() == want["summary_json"]
    assert d.read_text() == want["details_csv"]
    assert out.endswith(f"summary written: {s}\ndetails written: {d}\n")


@pytest.mark.gpu
def test_analyze_errors_and_multi_loop(tmp_path, R):
    trace = tmp_path / "t.csv"
    trace.write_bytes(R.synth_csv(seed=99, iterations=20, pattern_len=5))
    code, out = run(["analyze", "--trace", str(trace), "--iterations", "13", "--out-summary", str(tmp_path / "w.json"),
                     "--out-details", str(tmp_path / "w.csv")])
    assert code == 2 and "pattern-mining" in out
    assert run(["analyze", "--trace", "/no/such/file.csv", "--iterations", "10"])[0] == 3
    empty = tmp_path / "empty.csv"
    empty.write_bytes(b"")
    assert run(["inspect", "--trace", str(empty)])[0] == 3
    code, out = run(["analyze", "--trace", str(trace), "--loops", "20", "--out-summary", str(tmp_path / "l.json"),
                     "--out-details", str(tmp_path / "l.csv")])
    assert code == 0 and "loop 1" in out


@pytest.mark.gpu
def test_inspect_and_stable_bytes(tmp_path, R):
    trace = tmp_path / "st.csv"
    trace.write_bytes(R.synth_csv(seed=99, iterations=20, pattern_len=5, insert_prob=0.3, max_inserts=2))
    code, out = run(["inspect", "--trace", str(trace)])
    assert code == 0
    for word in ("Main", "CopyHtoD", "CopyDtoH", "Assist"):
        assert word in out
    outs = []
    for i in range(2):
        code, o = run(["analyze", "--trace", str(trace), "--iterations", "20", "--k0", "2", "--out-summary",
                       str(tmp_path / f"s{i}.json"), "--out-details", str(tmp_path / f"d{i}.csv")])
        assert code == 0, o
        outs.append(o.replace(f"s{i}.json", "S").replace(f"d{i}.csv", "D"))
    assert outs[0] == outs[1]
    assert (tmp_path / "s0.json").read_bytes() == (tmp_path / "s1.json").read_bytes()
