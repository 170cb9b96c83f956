"""GPU CSV ingest: itt_parse_csv vs the reference's parse_trace_text
(ingest.hpp:154-402, compiled in oracle/_ref), record by record, plus the IngestReport, the unit
warnings and the error paths; and CSV -> GPU parse -> GPU analyze -> summary JSON against the
reference CLI path (parse_trace_text + analyze_trace)."""
from __future__ import annotations

import random

import numpy as np
import pytest

from paper_1707_03750_b200 import cuda, itertrace

pytestmark = pytest.mark.gpu

HDR = "Start,Duration,Size,Throughput,Device,Stream,Name\n"


def compare(ctx, R, text: bytes, label="t.csv"):
    want = R.parse_csv(text, label)
    try:
        got = ctx.parse_csv(text, label)
    except cuda.IttError as e:
        assert want["status"] == e.status and want["error"] == str(e), (want, e.status, str(e))
        return "error"
    try:
        assert want["status"] == 0, want
        assert (got.rows_total, got.rows_parsed, got.rows_skipped) == \
            (want["rows_total"], want["rows_parsed"], want["rows_skipped"])
        assert got.skips == want["skips"]
        assert got.column == want["column"]
        assert got.warnings == want["warnings"]
        assert got.n == want["n"]
        cols = got.columns()
        order = np.lexsort((got.line, cols["start_ns"]))  # the reference's (start, row) order
        assert np.array_equal(cols["start_ns"][order], want["start_ns"])
        assert np.array_equal(cols["duration_ns"][order], want["duration_ns"])
        assert np.array_equal(cols["flags"][order], want["flags"])
        has = (want["flags"] & 1) != 0
        assert np.array_equal(cols["size_bytes"][order][has], want["size_bytes"][has])
        assert np.array_equal(cols["stream"][order], want["stream"])
        assert np.array_equal(got.line[order], want["row"])
        off, nb = cols["name_off"], cols["name_bytes"].tobytes()
        names = [nb[int(off[r]):int(off[r + 1])] for r in order]
        assert names == want["names"]
        assert [got.device_labels[d] for d in cols["device"][order]] == want["devices"]
        assert got.device_labels == sorted(set(want["devices"]))
    finally:
        got.free()
    return "ok"


def test_reference_generator_csvs(ctx, R):
    for seed, kw in [(1, {}), (2, dict(insert_prob=0.3, max_inserts=2)), (3, dict(insert_prob=0.5, max_inserts=3,
                     inside_pattern=True)), (4, dict(pathology=1)), (5, dict(pathology=2, iterations=200))]:
        text = R.synth_csv(seed=seed, **kw)
        assert compare(ctx, R, text) == "ok"


CASES = [
    # quoting: commas and doubled quotes inside names, quotes around numbers, quotes mid-cell
    HDR + '1,2,,,d0,7,"a,b"\n2,3,,,d0,7,"say ""hi"""\n"3","4",,,d0,"7",k\n4,5,,,d0,7,ab"c,d"e\n',
    # inline units override the column units; sizes in binary units; spaces/tabs trimmed
    HDR + "us,us,B,GB/s,,,\n1.5ms,20ns,2KB,,d0,7,k1\n 0.000001s ,\t3us\t,1.5MB,5GB/s,d0, 7 ,k2\n2,1,1GB,7MB/s,d0,7,k3\n",
    # every skip reason, in the reference's check order, among enough good rows
    HDR + "".join(f"{i},1,,,d0,7,k{i % 3}\n" for i in range(60)) +
    "1,1,,,d0,7,\n" "x,1,,,d0,7,k\n" "1,-2,,,d0,7,k\n" "1,1,,,d0,7a,k\n" "1,1,1.5XB,,d0,7,k\n" "1,1,,fast,d0,7,k\n",
    # CRLF lines, comments and blank lines anywhere, no trailing newline
    "== profiler\r\n\r\n" + HDR.replace("\n", "\r\n") + "== units follow\r\n\r\nus,us,B,GB/s,,,\r\n1,2,,,d0,7,a\r\n\r\n== mid\r\n3,4,,,d0,7,b",
    # not a units row: the first content line after the header is data
    HDR + "1,2,,,d0,7,a\n3,4,,,d0,7,b\n",
    # units row with a wrong unit in one column (warning) and units for absent columns
    "Start,Duration,Stream,Name\nms,KB,,\n1,2,7,a\n2,3,7,b\n",
    "Start,Duration,Stream,Name,Size,Throughput\nus,us,,,KB/s,MB\n1,2,7,a,3,4\n",
    # decimal scaling: round half up, 18-digit limit, INT64 overflow, leading zeros, '+' sign
    HDR + "ns,ns,B,,,,\n0.5,1.5,0.5,,d0,7,a\n2.4999,0.5000000001,1,,d0,7,b\n+3,000000000000000004,5,,d0,7,c\n"
    "123456789012345678,1,1,,d0,7,d\n" + "".join(f"{i},1,,,d0,7,k\n" for i in range(20)) +
    "1234567890123456789,1,,,d0,7,e\n",
    HDR + "s,s,,,,,\n9.223372036854775807,1,,,d0,7,a\n9.223372036854775808,1,,,d0,7,b\n" +
    "".join(f"{i},1,,,d0,7,k\n" for i in range(20)),
    # Stream: leading zeros, UINT32_MAX, overflow, internal space
    HDR + "1,1,,,d0,0000000000000000000000000000000000000000000000000000000013,a\n1,1,,,d0,4294967295,b\n"
    "1,1,,,d0,4294967296,c\n1,1,,,d0,1 3,d\n" + "".join(f"{i},1,,,d0,7,k\n" for i in range(30)),
    # Throughput accepted by std::stod (only presence matters) and rejected forms
    HDR + "".join(f"1,1,,{tp},d0,7,k\n" for tp in [
        "1e5", ".5", "5.", "-0", "0x1p4", "0x1.8p3GB/s", "0x1A", "1e309", "1.7976931348623157e308",
        "1.79769313486231580793728971405303415079934132710037826936173778980444968292764750946649017977587207096330286416692887910946555547851940402630657488671505820681908902000708383676273854845817711531764475730270069855571366959622842914819860834936475292719074168444365510704342711559699508093042880177904174497792e0",
        "2.2250738585072014e-308", "2.2250738585072011e-308", "1e-400", "0e500", "e5", "1e", "0x", "nan(1)",
        "inf", "-5", "0x1p-1030", "0x1p-1080", "0x1p1024", "0x1.fffffffffffff8p1023", "12 GB/s", "3KB/s", "4b/s"]) +
    "".join(f"{i},1,,,d0,7,k\n" for i in range(200)),
    # devices: absent column -> "unknown"; empty cell -> "unknown"; several labels, ranks lexicographic
    "Start,Duration,Stream,Name\n1,2,7,a\n2,3,7,b\n",
    HDR + "1,2,,,gpu-b,7,a\n2,3,,,,7,b\n3,4,,,gpu-a,7,c\n4,5,,, gpu-b ,7,d\n5,6,,,\"gpu,c\",7,e\n",
    # errors: missing required column, no header, too many bad rows, empty text
    "Start,Duration,Name\n1,2,a\n",
    "== only comments\n\n",
    HDR + "x,1,,,d0,7,a\n1,1,,,d0,7,b\n",
    "",
    # header repeated names: the last occurrence wins; extra columns ignored; short rows
    "Name,Start,Duration,Stream,Name,Extra\nn1,1,2,7,n2,z\n3,4\n",
]


@pytest.mark.parametrize("i", range(len(CASES)))
def test_adversarial_cases(ctx, R, i):
    compare(ctx, R, CASES[i].encode())


def _random_csv(rng: random.Random, rows: int) -> bytes:
    units = ["", "us", "ms", "ns", "s"]
    out = ["== fuzz", "Start,Duration,Size,Throughput,Device,Stream,Name"]
    if rng.random() < 0.5:
        out.append(",".join([rng.choice(units[1:]), rng.choice(units[1:]), rng.choice(["B", "KB", ""]),
                             rng.choice(["GB/s", ""]), "", "", ""]))
    for i in range(rows):
        st = f"{rng.randrange(0, 10**6)}.{rng.randrange(0, 1000):03d}" + (rng.choice(units) if rng.random() < 0.1 else "")
        du = f"{rng.randrange(0, 1000)}.{rng.randrange(0, 10)}"
        sz = rng.choice(["", "", str(rng.randrange(0, 10**6)), f"{rng.randrange(1, 100)}KB"])
        tp = rng.choice(["", "", f"{rng.random() * 100:.3f}", "1e3", "0x1p3", ".5GB/s"])
        dv = rng.choice(["d0", "d0", "d1", ""])
        sm = rng.choice(["7", "13", "13", "14", " 13 "])
        nm = rng.choice(["k1", "k2", '"a,b"', '"q""x"', "memcpy HtoD", " k1 "])
        cells = [st, du, sz, tp, dv, sm, nm]
        if rng.random() < 0.03:  # bad cells, under the 10% TooManyBadRows line
            cells[rng.randrange(7)] = rng.choice(["junk", "-1", "1e", '"', "1 2", ""])
        line = ",".join(cells)
        if rng.random() < 0.05:
            line += "\r"
        out.append(line)
        if rng.random() < 0.02:
            out.append(rng.choice(["", "== note", "   "]))
    return ("\n".join(out) + ("\n" if rng.random() < 0.5 else "")).encode()


def test_random_csvs(ctx, R):
    rng = random.Random(11)
    outcomes = []
    for t in range(40):
        outcomes.append(compare(ctx, R, _random_csv(rng, rng.randrange(1, 400))))
    assert outcomes.count("ok") > 20


def test_csv_end_to_end_matches_the_reference_cli_path(ctx, R):
    for seed, iters, kw in [(7, 40, {}), (8, 60, dict(insert_prob=0.2, max_inserts=2)), (9, 50, dict(pathology=1)),
                            (10, 30, dict(pathology=2))]:
        text = R.synth_csv(seed=seed, iterations=iters, **kw)
        want = R.analyze_csv(text, [iters], label="gen.csv")
        got = itertrace.analyze_csv(ctx, text, [iters], trace_label="gen.csv")
        assert want["status"] == 0
        assert got.summary_json() == want["summary_json"]
        assert got.details_csv(0) == want["details_csv"]
