"""Build the in-tree native libraries (sm_100a).

* libitertrace_cuda.so — the product: hand-written CUDA kernels + the C-ABI (csrc/*.cu)
* libitt_synth.so      — host-only TF-like trace generator (test/bench infrastructure)

nvcc cross-compiles for sm_100a without a GPU, so this runs in the CPU container too.
Objects are rebuilt only when a source or header is newer (headers invalidate all objects).
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
                  "-I" + CSRC, "-I" + os.path.join(ROOT, "include"), "--expt-relaxed-constexpr"]
NVFLAGS += os.environ.get("ITT_NVCC_EXTRA", "").split()  # A/B builds of kernel variants (e.g. -DITT_HASH_MINB=5)
CUDA_SO = os.path.join(HERE, "libitertrace_cuda.so")
CLI_BIN = os.path.join(HERE, "itertrace")  # the reference tool's CLI on the B200 path (tools/itertrace_cli.cpp)
REF_INC = os.environ.get("ITT_REFERENCE_INCLUDE", "/root/reference/proj/include")
SYNTH_SO = os.path.join(HERE, "libitt_synth.so")


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {os.path.basename(cmd[-1])}")


def build(verbose: bool = False, jobs: int = 8) -> None:
    os.makedirs(OBJ, exist_ok=True)
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    objs, todo = [], []
    for src in sources:
        obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        if _newer(obj, [src] + headers):
            todo.append([NVCC] + NVFLAGS + ["-c", "-o", obj, src])
    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        for f in [ex.submit(_run, cmd) for cmd in todo]:
            f.result()
    if todo or _newer(CUDA_SO, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", CUDA_SO] + objs + ["-lcudart_static", "-lrt", "-ldl", "-lpthread"])
    synth_src = os.path.join(CSRC, "synth_tf.cpp")
    if _newer(SYNTH_SO, [synth_src, os.path.join(ROOT, "include", "itt_synth.h")]):
        _run(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-I" + os.path.join(ROOT, "include"), "-o", SYNTH_SO,
              synth_src])
    # the CLI is built against the reference's headers (the types the drop-in keeps); where they are
    # absent (the GPU box) the prebuilt binary is used
    cli_src = os.path.join(HERE, "tools", "itertrace_cli.cpp")
    shim = os.path.join(ROOT, "include", "itertrace_cuda.hpp")
    if os.path.isdir(os.path.join(REF_INC, "itertrace")) and _newer(CLI_BIN, [cli_src, shim, CUDA_SO]):
        _run(["g++", "-O2", "-std=c++20", "-I" + os.path.join(ROOT, "include"), "-I" + REF_INC, "-I" + _json_include(),
              "-o", CLI_BIN, cli_src, "-L" + HERE, "-litertrace_cuda", "-Wl,-rpath,$ORIGIN"])
    if verbose:
        print(f"built {CUDA_SO} ({len(todo)} objects recompiled)")


def _json_include() -> str:
    """nlohmann/json.hpp (the reference's renderer needs it; not vendored by the reference)."""
    import site
    for p in site.getsitepackages():
        d = os.path.join(p, "include", "cudnn_frontend", "thirdparty", "nlohmann")
        if os.path.exists(os.path.join(d, "json.hpp")):
            return d
    raise RuntimeError("nlohmann/json.hpp not found")


if __name__ == "__main__":
    build(verbose=True)
