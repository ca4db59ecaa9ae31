"""Build the in-tree native libraries (sm_100a only).

* ``libhsolve_cuda.so`` — CUDA kernels + the C ABI (include/hs_cuda.h),
  nvcc ``-gencode arch=compute_100a,code=sm_100a``.
* ``libhsolve_b200.so`` — the C++ host shim re-exposing the reference
  ``hsolve`` API (include/hsolve/*.hpp) on top of the C ABI.

Both land next to this file so they travel with the repo snapshot to the GPU
box. Rebuilds only when a source is newer than the library.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
HOST = os.path.join(PKG, "host")
INC = os.path.join(ROOT, "include")
CUDA_LIB = os.path.join(PKG, "libhsolve_cuda.so")
HOST_LIB = os.path.join(PKG, "libhsolve_b200.so")
CLI_SRC = os.path.join(ROOT, "tools", "hsolve_bench.cpp")
CLI_BIN = os.path.join(PKG, "bin", "hsolve_bench")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills",
]


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd: list[str]) -> None:
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build_cuda(force: bool = False, verbose_ptxas: bool = False) -> str:
    cus = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    deps = cus + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(
        os.path.join(CSRC, "*.cuh")) + [os.path.join(INC, "hs_cuda.h")]
    if not force and not _stale(CUDA_LIB, deps):
        return CUDA_LIB
    objdir = os.path.join(ROOT, "build", "obj")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for cu in cus:
        obj = os.path.join(objdir, os.path.basename(cu) + ".o")
        objs.append(obj)
        cmd = [NVCC, *NVCC_FLAGS, "-I", INC, "-I", CSRC, "-c", cu, "-o", obj]
        if verbose_ptxas:
            cmd += ["-Xptxas", "-v"]
        print("+", " ".join(cmd), flush=True)
        procs.append(subprocess.Popen(cmd))
    bad = [p for p in procs if p.wait() != 0]
    if bad:
        raise RuntimeError("nvcc failed")
    _run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
          "-Xcompiler", "-fPIC", *objs, "-o", CUDA_LIB, "-ldl"])
    return CUDA_LIB


def build_host(force: bool = False) -> str:
    srcs = sorted(glob.glob(os.path.join(HOST, "*.cpp")))
    if not srcs:
        return ""
    deps = srcs + glob.glob(os.path.join(HOST, "*.hpp")) + glob.glob(
        os.path.join(INC, "hsolve", "*.hpp")) + [os.path.join(INC, "hs_cuda.h"), CUDA_LIB]
    if not force and not _stale(HOST_LIB, deps):
        return HOST_LIB
    cxx = os.environ.get("CXX", "g++")
    _run([cxx, "-std=c++20", "-O2", "-fPIC", "-shared", "-I", INC, *srcs,
          "-o", HOST_LIB, "-L", PKG, "-lhsolve_cuda", "-Wl,-rpath,$ORIGIN"])
    return HOST_LIB


def build_cli(force: bool = False) -> str:
    """The reference's hsolve_bench CLI (gen / solve / sweep)."""
    if not force and not _stale(CLI_BIN, [CLI_SRC, HOST_LIB]):
        return CLI_BIN
    os.makedirs(os.path.dirname(CLI_BIN), exist_ok=True)
    cxx = os.environ.get("CXX", "g++")
    _run([cxx, "-std=c++20", "-O2", "-I", INC, CLI_SRC, "-o", CLI_BIN, "-L", PKG,
          "-lhsolve_b200", "-lhsolve_cuda", "-Wl,-rpath,$ORIGIN/.."])
    return CLI_BIN


def build(force: bool = False) -> None:
    build_cuda(force)
    build_host(force)
    build_cli(force)


def build_debug_variant(macro: str, out_name: str) -> str:
    """A diagnostic build of the CUDA library with `-D<macro>` into tools/
    (HS_SYMV_TIMING: per-launch / per-CTA SYMV timestamps for
    tools/symv_timing.py and tools/cg_timeline.py; HS_DIAG_TIMING: diag128
    phase timing for tools/diag_timing.py). Never loaded by the product."""
    objdir = os.path.join(ROOT, "build", "obj_" + macro.lower())
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for cu in sorted(glob.glob(os.path.join(CSRC, "*.cu"))):
        obj = os.path.join(objdir, os.path.basename(cu) + ".o")
        _run([NVCC, *NVCC_FLAGS, "-D" + macro, "-I", INC, "-I", CSRC, "-c", cu, "-o", obj])
        objs.append(obj)
    out = os.path.join(ROOT, "tools", out_name)
    _run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
          "-Xcompiler", "-fPIC", *objs, "-o", out, "-ldl"])
    return out


if __name__ == "__main__":
    if "--symv-timing" in sys.argv:
        build_debug_variant("HS_SYMV_TIMING", "libhsolve_cuda_symvtiming.so")
    elif "--diag-timing" in sys.argv:
        build_debug_variant("HS_DIAG_TIMING", "libhsolve_cuda_diagtiming.so")
    else:
        build(force="--force" in sys.argv)
