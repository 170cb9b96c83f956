"""CPU: the C-ABI library loads, exports exactly what include/*.h declares, and the ctypes
mirror has the C layouts.  No compute calls (there is no GPU here)."""
from __future__ import annotations

import ctypes as C
import os
import re
import subprocess
import tempfile

import pytest

from conftest import ROOT
from paper_1707_03750_b200 import abi, cuda


def _exports(path):
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True, check=True).stdout
    return sorted({line.split()[-1] for line in out.splitlines() if " T " in line})


def test_library_exports_every_declared_symbol():
    declared = cuda.exported_symbols()
    assert len(declared) >= 28
    exported = [s for s in _exports(cuda.LIB_PATH) if s.startswith("itt_")]
    assert sorted(declared) == exported
    lib = cuda.lib()  # loads, ABI version matches
    for name in declared:
        assert hasattr(lib, name)


def test_product_library_is_sm100a_only_and_has_no_oracle():
    out = subprocess.run(["cuobjdump", "--list-elf", cuda.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in l for l in out.splitlines() if ".cubin" in l)
    syms = subprocess.run(["nm", "-D", cuda.LIB_PATH], capture_output=True, text=True).stdout
    assert "orc_" not in syms and "ref_" not in syms  # the checker is never linked into the product


STRUCTS = ["itt_records", "itt_kernel_stat", "itt_stream_summary", "itt_census", "itt_tokens", "itt_repeat",
           "itt_mining_cfg", "itt_pattern", "itt_span", "itt_iter_row", "itt_clamps", "itt_analyze_opts",
           "itt_loop_result", "itt_analysis", "itt_op_cell"]


def test_ctypes_layouts_match_the_header():
    src = ["#include <stdio.h>", "#include <stddef.h>", '#include "itertrace_cuda.h"', "int main(void){"]
    for s in STRUCTS:
        src.append(f'printf("{s} %zu\\n", sizeof({s}));')
        for f, _ in getattr(abi, s)._fields_:
            src.append(f'printf("{s}.{f} %zu\\n", offsetof({s}, {f}));')
    src.append("return 0;}")
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "layout.c")
        exe = os.path.join(d, "layout")
        open(c, "w").write("\n".join(src))
        subprocess.run(["gcc", "-I" + os.path.join(ROOT, "include"), "-o", exe, c], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()
    got = dict(zip(out[0::2], map(int, out[1::2])))
    for s in STRUCTS:
        t = getattr(abi, s)
        assert got[s] == C.sizeof(t), s
        for f, _ in t._fields_:
            assert got[f"{s}.{f}"] == getattr(t, f).offset, f"{s}.{f}"


def test_status_codes_mirror_error_kinds():
    hdr = open(os.path.join(ROOT, "include", "itertrace_cuda.h")).read()
    codes = dict((m.group(1), int(m.group(2))) for m in re.finditer(r"ITT_E_(\w+) = (\d+)", hdr))
    kinds = ["UNREADABLE_FILE", "MISSING_COLUMN", "TOO_MANY_BAD_ROWS", "EMPTY_TRACE", "NO_MAIN_STREAM",
             "EMPTY_MAIN_STREAM", "INVALID_ITERATION_COUNT", "NO_PATTERN_FOUND", "AMBIGUOUS_LOOPS", "NO_ITERATIONS",
             "INVALID_CONFIG", "IO_ERROR"]  # errors.hpp:8-21 order
    for i, k in enumerate(kinds):
        assert codes[k] == i + 1
    assert [e.upper() for e in abi.ERROR_KINDS] == [k.replace("_", "") for k in kinds]


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback_without_gpu():
    with pytest.raises(cuda.IttError) as e:
        cuda.Context(0)
    assert e.value.status == abi.ITT_E_CUDA


def test_headers_cite_reference_interfaces():
    hdr = open(os.path.join(ROOT, "include", "itertrace_cuda.h")).read()
    for ref in ("streams.hpp:147-169", "mine.hpp:119-122", "mine.hpp:132-165", "match.hpp:41-85", "metrics.hpp:44-164",
                "pipeline.hpp:34-134", "suffix_tree.hpp:21-190", "mine.hpp:46-60"):
        assert ref in hdr
