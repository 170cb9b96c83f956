"""Test configuration.

Markers: ``gpu`` tests need a B200 (they run on the GPU box via gpurun / the driver); every
other test runs on the CPU container.  The parity oracle is the reference itself
(oracle/_ref, built from the reference headers by oracle/Makefile) plus the committed golden
fixtures in tests/golden/ generated from it.
"""
from __future__ import annotations

import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 GPU (sm_100a); run with -m gpu on the GPU box")


@pytest.fixture(scope="session")
def ctx():
    from paper_1707_03750_b200 import cuda
    c = cuda.Context(0)  # raises (no CPU fallback) when there is no sm_100 device
    yield c
    c.close()


@pytest.fixture(scope="session")
def R():
    from oracle.bindings import ref
    return ref()


@pytest.fixture(scope="session")
def O():
    from oracle.bindings import oracle
    return oracle()


@pytest.fixture(scope="session")
def token_cases():
    with open(os.path.join(GOLDEN, "token_cases.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def trace_cases():
    with open(os.path.join(GOLDEN, "trace_cases.json")) as f:
        return json.load(f)


def records_from_ops(ops, device=None):
    """In-memory trace builder in the style of test_metrics.cpp:22-42 / test_streams.cpp:25-32.
    ops: list of (stream, name, start, duration[, size[, throughput]])."""
    import numpy as np
    from paper_1707_03750_b200.abi import REC_HAS_SIZE, REC_HAS_THROUGHPUT, Records
    start = [o[2] for o in ops]
    dur = [o[3] for o in ops]
    size = [o[4] if len(o) > 4 and o[4] is not None else 0 for o in ops]
    flags = [(REC_HAS_SIZE if len(o) > 4 and o[4] is not None else 0) |
             (REC_HAS_THROUGHPUT if len(o) > 5 and o[5] is not None else 0) for o in ops]
    return Records(start_ns=start, duration_ns=dur, stream=[o[0] for o in ops], names=[o[1] for o in ops],
                   size_bytes=size, flags=flags, device=np.asarray(device, np.uint16) if device is not None else None)
