"""Build the in-tree native libraries of the product path.

  libdgdiff.so  -- csrc/dgdiff.cu + csrc/operator.cpp, nvcc for sm_100a
                   (-gencode arch=compute_100a,code=sm_100a -lineinfo), static
                   cudart, NCCL dlopen'ed at run time
  librsa.so     -- csrc/rsa.c (input generation helper, gcc)
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libdgdiff.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

SOURCES = ["dgdiff.cu", "operator.cpp"]
HEADERS = ["kernels.cuh", "operator.h", "stage_imm.cuh", "stage_tb.cuh", "stage_ring.cuh"]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.exists(d) and os.path.getmtime(d) > t for d in deps)


TABLES = os.path.join(CSRC, "tables.inc")
GEN = os.path.join(HERE, "gen_tables")


def build_tables(force=False) -> str:
    """Run K0 at build time (gen_tables) to emit the compile-time operator."""
    deps = [os.path.join(CSRC, f) for f in ("gen_tables.cpp", "operator.cpp", "operator.h")]
    if force or _stale(GEN, deps):
        tmp = GEN + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-Wno-free-nonheap-object", "-o", tmp,
                               os.path.join(CSRC, "gen_tables.cpp"), os.path.join(CSRC, "operator.cpp")])
        os.replace(tmp, GEN)
    if force or _stale(TABLES, [GEN]):
        tmp = TABLES + f".tmp{os.getpid()}"
        subprocess.check_call([GEN, tmp])
        os.replace(tmp, TABLES)
    return TABLES


def build_dgdiff(force=False, verbose=False) -> str:
    build_tables(force=force)
    deps = [TABLES] + [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "dgdiff.h"), __file__]
    if not force and not _stale(LIB, deps):
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-DDGDIFF_BUILD",
           "-Xcompiler", "-fPIC,-Wno-free-nonheap-object", "-shared", "-cudart", "static",
           "-I", os.path.join(ROOT, "include"), "-I", CSRC,
           "-o", tmp] + [os.path.join(CSRC, f) for f in SOURCES] + ["-ldl"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


def build_all(force=False, verbose=False):
    from . import substrate
    substrate._rsa_lib()
    return build_dgdiff(force=force, verbose=verbose)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
