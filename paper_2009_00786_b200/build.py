"""In-tree build of libtsgpu.so (sm_100a) and, optionally, the oracle.

    python -m paper_2009_00786_b200.build        # library only
    python -m paper_2009_00786_b200.build --all  # + oracle/ (+ oracle/_ref when the reference is present)

The library is compiled straight with nvcc for sm_100a (-gencode
arch=compute_100a,code=sm_100a) so the .so travels with the repo snapshot to
the GPU box; nothing is JIT-compiled at import time.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libtsgpu.so")
BUILD = os.path.join(PKG, "_build")

CU_SOURCES = ["summarise.cu", "build.cu", "search.cu", "generate.cu", "exchange.cu", "audit.cu", "api.cu"]
# host C++: (file, extra flags). breakpoints.cpp must match the reference's
# x86-64 arithmetic (no -march, no FMA); tsidx_api.cpp is the C++20 drop-in API.
CPP_SOURCES = [("breakpoints.cpp", ["-std=c++17"]),
               ("tsidx_api.cpp", ["-std=c++20", "-I/usr/local/cuda/include"])]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
    "--expt-relaxed-constexpr", "-Xptxas", "-O3",
    "-I" + os.path.join(ROOT, "include"),
]
# Host C++ that must be bit-identical to the reference's x86-64 build: no -march, no FMA.
CXX_FLAGS = ["-O3", "-fPIC", "-ffp-contract=off"]


def _run(cmd):
    print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_library(force: bool = False, verbose_ptxas: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".cuh", ".h"))]
    headers.append(os.path.join(ROOT, "include", "tsgpu.h"))
    objs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _stale(o, [s, *headers]):
            extra = ["-Xptxas", "-v"] if verbose_ptxas else []
            _run([NVCC, *NVCC_FLAGS, *extra, "-c", s, "-o", o])
        objs.append(o)
    cxx = os.environ.get("CXX", "g++")
    for src, extra in CPP_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _stale(o, [s, *headers, os.path.join(ROOT, "include", "tsidx", "tsidx.hpp")]):
            _run([cxx, *CXX_FLAGS, *extra, "-c", s, "-o", o])
        objs.append(o)
    if force or _stale(LIB, objs):
        _run([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB, *objs,
              "-lcudart_static", "-lrt", "-lpthread", "-ldl"])
    return LIB


def build_oracle() -> None:
    sys.path.insert(0, ROOT)
    from oracle import oracle as orc  # test infrastructure: compiled, never linked into the library

    orc.build()


if __name__ == "__main__":
    force = "--force" in sys.argv
    build_library(force=force, verbose_ptxas="--ptxas-v" in sys.argv)
    if "--all" in sys.argv:
        build_oracle()
