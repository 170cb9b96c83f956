"""CPU: the host-side finish of analyze_trace (summary doubles, diagnosis, warnings, rendering)
reproduces the reference byte for byte, independent of the GPU."""
from __future__ import annotations

import json
import os

from conftest import GOLDEN
from paper_1707_03750_b200 import itertrace as it


def _canned():
    # test_report.cpp:27-80 (canned_report / canned_details)
    s = it.SummaryMetrics(avg_interval_ns=1000.0, max_interval_ns=2000, avg_overlap=0.05, avg_operation_ns=200.0,
                          avg_size_bytes=4096.0, iterations_found=3, iterations_declared=3)
    loop = it.LoopReport(3, ["opA", "opB"], [0, 1], 2, 3, 1, 0, 1, 3, s, it.diagnose(s))
    streams = [(13, 0, (6, 0, 0, 0, 0, 0), 100, 9000), (14, 1, (0, 2, 0, 0, 0, 0), 50, 8000)]
    details = [it.IterationMetrics(i + 1, 2 * i, 2 * i + 1, 1000 * i + 100, 1000 * i + 600, 500 if i else None,
                                   0.05 if i else None, 4096, 200.0, 0) for i in range(3)]
    return it.AnalysisResult("fixture.csv", 1, 0.10, 10.0, None, None, streams, 13, [loop], [details], [])


def test_render_matches_reference_goldens():
    r = _canned()
    want_json = open(os.path.join(GOLDEN, "reference_summary_golden.json")).read()
    want_csv = open(os.path.join(GOLDEN, "reference_details_golden.csv")).read()
    assert r.summary_json() == want_json
    assert r.details_csv() == want_csv


def test_render_matches_reference_on_golden_traces(trace_cases):
    """Rebuild each golden run's report from its integer/double data and re-render it."""
    n = 0
    for c in trace_cases:
        if "loops_out" not in c:
            continue
        doc = json.loads(c["summary_json"])
        loops, details = [], []
        for k, L in enumerate(c["loops_out"]):
            items = [it.IterationMetrics(x[0], x[1], x[2], x[4], x[5], x[6] if x[8] else None,
                                         float.fromhex(x[10]) if x[9] else None, x[7], float.fromhex(x[11]), x[3])
                     for x in L["iters"]]
            s = it.compute_summary(items, L["iterations_declared"])
            assert [float(v).hex() for v in (s.avg_interval_ns, s.avg_overlap, s.avg_operation_ns,
                                              s.avg_size_bytes)] == L["avg"], c["name"]
            assert s.max_interval_ns == L["max_interval_ns"] and s.insufficient_intervals == L["insufficient_intervals"]
            d = it.diagnose(s)
            assert it.DIAG.index(d.code) == L["diagnosis"]
            loops.append(it.LoopReport(L["iterations_declared"], doc["loops"][k]["pattern"], [], L["pattern_length"],
                                       L["pattern_count"], L["epsilon_used"], L["first_token"], L["k0_used"],
                                       len(items), s, d))
            details.append(items)
        streams = [(s[0], s[1], tuple(s[2]), s[3], s[4]) for s in c["streams"]]
        r = it.AnalysisResult("trace.csv", c["opts"].get("epsilon0", 1), 0.10, 10.0, c["opts"].get("k0"),
                              c["opts"].get("main_stream"), streams, c["main_stream"], loops, details, c["warnings"])
        assert r.summary_json() == c["summary_json"], c["name"]
        assert r.details_csv(0) == c["details_csv"], c["name"]
        n += 1
    assert n >= 10


def test_summary_and_diagnosis_known_answers():
    # test_metrics.cpp:204-235 and test_report.cpp:92-125
    items = [it.IterationMetrics(i + 1, 0, 0, 0, 0, [None, 10, 20, 30][i], None, 0, 0.0, 0) for i in range(4)]
    s = it.compute_summary(items, 4)
    assert s.avg_interval_ns == 20.0 and s.max_interval_ns == 30 and not s.insufficient_intervals
    s1 = it.compute_summary([it.IterationMetrics(1, 0, 0, 0, 0, None, None, 0, 0.0, 0)], 5)
    assert s1.insufficient_intervals and s1.avg_interval_ns == 0.0
    try:
        it.compute_summary([], 3)
        raise AssertionError("expected NoIterations")
    except it.AnalyzeError as e:
        assert e.kind == "NoIterations"

    def sw(ai, ao, aop, n=10):
        return it.SummaryMetrics(ai, int(ai * 2), ao, aop, 4096.0, n, n)
    assert it.diagnose(sw(1000, 0.5, 10)).code == "COPY_BOUND"  # copy wins even when the gap is long
    assert it.diagnose(sw(1000, 0.01, 10)).code == "CPU_BOUND"
    assert it.diagnose(sw(100, 0.01, 10)).code == "CPU_BOUND"  # >= is inclusive
    assert it.diagnose(sw(99, 0.01, 10)).code == "NONE"
    assert it.diagnose(sw(1000, 0.10, 10)).code == "COPY_BOUND"  # theta_copy inclusive
    assert it.diagnose(sw(1000, 0.5, 10, n=1)).code == "INSUFFICIENT_DATA"
    assert it.diagnose(sw(0, 0.0, 0)).code == "NONE"


def test_json_float_format():
    f = it._json_float
    assert [f(x) for x in (0.1, 10.0, 1000.0, 0.05, 4096.0, 1e-05, 1e16, 0.0001, 2.5e-07)] == \
        ["0.1", "10.0", "1000.0", "0.05", "4096.0", "1e-05", "1e+16", "0.0001", "2.5e-07"]
    assert f(1e15) == "1e+15" and f(1234567890123456.0) == "1.234567890123456e+15"


def test_json_float_matches_the_reference_json_library():
    """jsonfloat.dump_float restates the reference JSON library's Grisu2 double printing; Python's
    shortest repr differs for ~0.1% of doubles (e.g. 4957.0239520958085), so it is pinned against
    nlohmann::json(v).dump() from the reference build itself."""
    import ctypes as C
    import math
    import random
    import struct

    from oracle.bindings import ref
    from paper_1707_03750_b200.jsonfloat import dump_float
    L = ref().lib
    L.ref_json_double.argtypes = [C.c_double, C.c_char_p, C.c_int]
    buf = C.create_string_buffer(64)
    vals = [4957.0239520958085, 0.049589542629412633, 0.0030392262455614452, 1e15, 1e16, 123456789012345.0,
            1e-5, 1e-4, 5e-324, 1.7976931348623157e308, 2.2250738585072014e-308, -0.0, 0.0, 1.0, 0.1, 1e21]
    rng = random.Random(7)
    while len(vals) < 30000:
        k = rng.random()
        if k < 0.3:
            v = struct.unpack("<d", struct.pack("<Q", rng.getrandbits(64)))[0]
        elif k < 0.7:
            v = rng.random() * 10 ** rng.randint(-8, 20)
        else:
            v = rng.randint(0, 10 ** 7) / rng.randint(1, 10 ** 5)
        if not (math.isnan(v) or math.isinf(v)):
            vals.append(v)
    for v in vals:
        L.ref_json_double(v, buf, 64)
        assert dump_float(v) == buf.value.decode(), repr(v)
