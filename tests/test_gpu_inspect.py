"""GPU: the `inspect` census path — itt_parse_csv + the device stream census,
rendered as print_stream_table (itertrace_main.cpp:61-77) — against the reference's own parse and
summarize_streams/classify_streams (oracle/_ref) on reference-generator CSVs, incl. skipped rows
and a multi-device trace."""
from __future__ import annotations

import pytest

from paper_1707_03750_b200 import itertrace

pytestmark = pytest.mark.gpu


def _records(p):
    from paper_1707_03750_b200 import abi
    return abi.Records(p["start_ns"], p["duration_ns"], p["stream"], size_bytes=p["size_bytes"], flags=p["flags"],
                       names=p["names"])


@pytest.mark.parametrize("seed,extra", [(1, b""), (7, b"garbage,row\n"), (11, b"")])
def test_inspect_matches_reference_census(ctx, R, seed, extra):
    text = R.synth_csv(seed=seed, pattern_len=7, iterations=30, vocab_size=12, insert_prob=0.1, max_inserts=2) + extra
    label = f"t{seed}.csv"
    got = itertrace.inspect_csv(ctx, text, label)
    p = R.parse_csv(text, label)
    # the reference census over the reference's own parsed records (no device filter)
    streams, _ = R.summarize_streams(_records(p), filter_device=False)
    want = ("trace: %s\nrows: %d parsed, %d skipped of %d\n" % (label, p["rows_parsed"], p["rows_skipped"], p["rows_total"])
            + itertrace.stream_table(streams))
    assert got == want
    lines = got.splitlines()
    assert lines[2].split() == ["stream", "class", "kernel", "htod", "dtoh", "dtod", "memset", "other", "first_ns", "last_ns"]
    assert any(" Main " in ln for ln in lines[3:])
