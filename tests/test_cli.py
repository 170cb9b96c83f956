"""The B200 CLIs against the reference tool's contract (tools/itertrace_main.cpp; cases restated
from tests/test_cli.cpp): exit codes, the lines the reference tests grep, byte-stable output, and —
beyond the reference's own tests — summary JSON and details CSV byte-identical to the reference's
analyze on the same CSV.  Two front ends run every case:
  * "cpp": paper_1707_03750_b200/itertrace, the C++ tool (tools/itertrace_cli.cpp) — the drop-in
    for the reference binary, with --config and the synth subcommand;
  * "py":  the Python mirror (paper_1707_03750_b200/cli.py; analyze / inspect only).
Argument errors and synth are checked on CPU (they exit before a device is touched); runs that
analyze need the GPU."""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

from conftest import ROOT


CPP = os.path.join(ROOT, "paper_1707_03750_b200", "itertrace")
IMPLS = ["cpp", "py"]


def run(args, cwd=None, impl="py"):
    cmd = [CPP] if impl == "cpp" else [sys.executable, "-m", "paper_1707_03750_b200.cli"]
    if impl == "cpp" and not os.path.exists(CPP):
        pytest.fail(f"{CPP} not built (build() compiles it where the reference headers exist)")
    r = subprocess.run(cmd + args, cwd=cwd or ROOT, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True,
                       timeout=600)
    return r.returncode, r.stdout


@pytest.fixture(params=IMPLS)
def impl(request):
    return request.param


def test_argument_errors_exit_4(tmp_path, impl):
    def r(args):
        return run(args, impl=impl)
    t = str(tmp_path / "x.csv")
    assert r(["analyze", "--trace", t])[0] == 4                                   # neither --iterations nor --loops
    assert r(["analyze", "--trace", t, "--iterations", "5", "--loops", "5"])[0] == 4
    assert r(["analyze", "--trace", t, "--iterations", "5", "--out-summary", "a", "--out-details", "a"])[0] == 4
    assert r(["analyze", "--trace", t, "--iterations", "5", "--bogus-flag"])[0] == 4
    assert r(["analyze", "--trace", t, "--iterations", "five"])[0] == 4
    assert r([])[0] == 4                                                         # a subcommand is required
    code, out = r(["--version"])
    assert code == 0 and out.strip() == "0.1.0"
    assert r(["analyze", "--help"])[0] == 0


def test_cpp_synth_and_config(tmp_path):
    """synth (the reference's generator behind the same options, itertrace_main.cpp:209-264) and
    --config (CLI11 set_config): CPU only, no device is touched."""
    t, g = tmp_path / "s.csv", tmp_path / "s.json"
    code, out = run(["synth", "--seed", "99", "--iterations", "20", "--pattern-len", "5", "--out-trace", str(t),
                     "--out-truth", str(g)], impl="cpp")
    assert code == 0 and f"trace written: {t}" in out
    from oracle.bindings import ref
    assert t.read_bytes() == ref().synth_csv(seed=99, iterations=20, pattern_len=5)
    assert run(["synth", "--out-trace", "/no/such/dir/t.csv", "--out-truth", "/no/such/dir/g.json"], impl="cpp")[0] == 3
    assert run(["synth", "--pattern-len", "30", "--vocab-size", "8", "--out-trace", str(tmp_path / "b.csv"),
                "--out-truth", str(tmp_path / "b.json")], impl="cpp")[0] == 4
    assert run(["synth", "--pathology", "GRAPH_growth", "--out-trace", str(tmp_path / "p.csv"), "--out-truth",
                str(tmp_path / "p.json")], impl="cpp")[0] == 0                     # enums ignore case
    assert run(["synth", "--pathology", "bogus"], impl="cpp")[0] == 4
    cfg = tmp_path / "synth.toml"
    cfg.write_text(f'# generator config\n[synth]\nseed = 99\niterations = 20\npattern-len = 5\n'
                   f'out_trace = "{tmp_path / "c.csv"}"\nout-truth = "{tmp_path / "c.json"}"\n')
    assert run(["synth", "--config", str(cfg)], impl="cpp")[0] == 0
    assert (tmp_path / "c.csv").read_bytes() == t.read_bytes()
    cfg.write_text("bogus-key = 1\n")
    assert run(["synth", "--config", str(cfg)], impl="cpp")[0] == 4
    # analyze --config: the argument checks run before any device work
    acfg = tmp_path / "a.toml"
    acfg.write_text(f'trace = "{t}"\n')
    code, out = run(["analyze", "--config", str(acfg)], impl="cpp")
    assert code == 4 and "needs --iterations or --loops" in out
    acfg.write_text(f'trace = "{t}"\niterations = 20\nloops = [20, 10]\n')
    code, out = run(["analyze", "--config", str(acfg)], impl="cpp")
    assert code == 4 and "not both" in out


@pytest.mark.gpu
def test_cpp_config_analyze_equals_flags(tmp_path, R):
    trace = tmp_path / "ok.csv"
    trace.write_bytes(R.synth_csv(seed=7, iterations=30, pattern_len=6))
    cfg = tmp_path / "a.toml"
    cfg.write_text(f'[analyze]\ntrace = "{trace}"\niterations = 30\nk0 = 2\nout-summary = "{tmp_path / "c.json"}"\n'
                   f'out-details = "{tmp_path / "c.csv"}"\n')
    code, out_c = run(["analyze", "--config", str(cfg)], impl="cpp")
    assert code == 0, out_c
    code, out_f = run(["analyze", "--trace", str(trace), "--iterations", "30", "--k0", "2", "--out-summary",
                       str(tmp_path / "f.json"), "--out-details", str(tmp_path / "f.csv")], impl="cpp")
    assert code == 0, out_f
    assert (tmp_path / "c.json").read_bytes() == (tmp_path / "f.json").read_bytes()
    assert (tmp_path / "c.csv").read_bytes() == (tmp_path / "f.csv").read_bytes()
    # the command line wins over the file
    code, out = run(["analyze", "--config", str(cfg), "--iterations", "13"], impl="cpp")
    assert code == 2 and "pattern-mining" in out


@pytest.mark.gpu
def test_console_text_identical_across_front_ends(tmp_path, R):
    trace = tmp_path / "t.csv"
    trace.write_bytes(R.synth_csv(seed=5, iterations=25, pattern_len=7, insert_prob=0.2, max_inserts=1))
    outs = {}
    for im in IMPLS:
        code, o = run(["analyze", "--trace", str(trace), "--iterations", "25", "--out-summary", str(tmp_path / "s.json"),
                       "--out-details", str(tmp_path / "d.csv")], impl=im)
        assert code == 0, o
        outs[im] = o
        code, o = run(["inspect", "--trace", str(trace)], impl=im)
        assert code == 0, o
        outs[im + "-inspect"] = o
    assert outs["cpp"] == outs["py"]
    assert outs["cpp-inspect"] == outs["py-inspect"]


@pytest.mark.gpu
def test_analyze_clean_trace(tmp_path, R, impl):
    trace = tmp_path / "ok.csv"
    trace.write_bytes(R.synth_csv(seed=99, iterations=20, pattern_len=5))
    s, d = tmp_path / "ok_summary.json", tmp_path / "ok_details.csv"
    code, out = run(["analyze", "--trace", str(trace), "--iterations", "20", "--out-summary", str(s),
                     "--out-details", str(d)], impl=impl)
    assert code == 0, out
    assert "diagnosis: NONE" in out and "loop 1" in out
    want = R.analyze_csv(trace.read_bytes(), [20], label=str(trace))
    assert s.read_text() == want["summary_json"]
    assert d.read_text() == want["details_csv"]
    assert out.endswith(f"summary written: {s}\ndetails written: {d}\n")


@pytest.mark.gpu
def test_analyze_errors_and_multi_loop(tmp_path, R, impl):
    trace = tmp_path / "t.csv"
    trace.write_bytes(R.synth_csv(seed=99, iterations=20, pattern_len=5))
    code, out = run(["analyze", "--trace", str(trace), "--iterations", "13", "--out-summary", str(tmp_path / "w.json"),
                     "--out-details", str(tmp_path / "w.csv")], impl=impl)
    assert code == 2 and "pattern-mining" in out
    assert run(["analyze", "--trace", "/no/such/file.csv", "--iterations", "10"], impl=impl)[0] == 3
    empty = tmp_path / "empty.csv"
    empty.write_bytes(b"")
    assert run(["inspect", "--trace", str(empty)], impl=impl)[0] == 3
    code, out = run(["analyze", "--trace", str(trace), "--loops", "20", "--out-summary", str(tmp_path / "l.json"),
                     "--out-details", str(tmp_path / "l.csv")], impl=impl)
    assert code == 0 and "loop 1" in out


@pytest.mark.gpu
def test_inspect_and_stable_bytes(tmp_path, R, impl):
    trace = tmp_path / "st.csv"
    trace.write_bytes(R.synth_csv(seed=99, iterations=20, pattern_len=5, insert_prob=0.3, max_inserts=2))
    code, out = run(["inspect", "--trace", str(trace)], impl=impl)
    assert code == 0
    for word in ("Main", "CopyHtoD", "CopyDtoH", "Assist"):
        assert word in out
    outs = []
    for i in range(2):
        code, o = run(["analyze", "--trace", str(trace), "--iterations", "20", "--k0", "2", "--out-summary",
                       str(tmp_path / f"s{i}.json"), "--out-details", str(tmp_path / f"d{i}.csv")], impl=impl)
        assert code == 0, o
        outs.append(o.replace(f"s{i}.json", "S").replace(f"d{i}.csv", "D"))
    assert outs[0] == outs[1]
    assert (tmp_path / "s0.json").read_bytes() == (tmp_path / "s1.json").read_bytes()
