"""GPU: the C++ drop-in (include/itertrace_cuda.hpp) against the reference, in C++.

oracle/_ref/dropin_test is built by oracle/Makefile from tests/cpp/dropin_test.cpp against the
reference headers (it needs them at build time only) and linked to libitertrace_cuda.so.  It
feeds the REFERENCE's own generator + CSV ingest output through itertrace::analyze_trace and
itertrace::cuda::analyze_trace (and each stage function) and requires identical bytes.
"""
from __future__ import annotations

import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
EXE = os.path.join(ROOT, "oracle", "_ref", "dropin_test")


def test_cpp_dropin_matches_reference():
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/dropin_test not built (needs the reference headers at build time)")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr[-4000:]
    assert "0 mismatches" in r.stdout
