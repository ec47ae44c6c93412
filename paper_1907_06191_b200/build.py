"""Build the in-tree native libraries of the product path.

  libdgdiff.so  -- csrc/*.cu translation units + csrc/operator.cpp, compiled in
                   parallel by nvcc for sm_100a (-gencode arch=compute_100a,
                   code=sm_100a -lineinfo), static cudart, NCCL dlopen'ed at
                   run time; csrc/tables.inc is generated first by gen_tables
                   (K0 at build time)
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
# tuning build (experiments only): -DDGDIFF_TUNING makes the library read its
# DGDIFF_* tuning knobs from the environment; it goes to a separate library
# (loaded by dgdiff.py only when DGDIFF_TUNING_LIB=1) so the product library
# never does
LIB_TUNING = os.path.join(HERE, "libdgdiff_tuning.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

SOURCES = ["dgdiff.cu", "launch.cu", "stage_v12_f64.cu", "stage_v12_f32.cu", "stage_ring_p1_f64.cu",
           "stage_ring_p1_f32.cu", "stage_ring_p2_f64.cu", "stage_ring_p2_f32.cu",
           "stage_ring_p3_f64.cu", "stage_ring_p3_f32.cu", "stage_ring_q_f64.cu", "stage_ring_q_f32.cu", "step_fused_f64.cu", "step_dec_f64.cu", "step_wave.cu",
           "step_fused_f32.cu", "stage_pair.cu", "stage_ring_adj_f64.cu", "operator.cpp"]
HEADERS = ["kernels.cuh", "operator.h", "stage_imm.cuh", "stage_ring.cuh", "stage_v12.cuh", "launch.h",
           "step_fused.cuh", "step_dec.cuh", "stage_wave.cuh", "mc_walk.cuh", "stage_pair.cuh"]
OBJDIR = os.path.join(HERE, "build_obj")
OBJDIR_TUNING = os.path.join(HERE, "build_obj_tuning")


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


def _compile(src, verbose, tuning=False):
    """nvcc -c one translation unit (skipped when its object is fresh)."""
    objdir = OBJDIR_TUNING if tuning else OBJDIR
    os.makedirs(objdir, exist_ok=True)
    obj = os.path.join(objdir, os.path.basename(src) + ".o")
    deps = [src, TABLES] + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "dgdiff.h")]
    if not _stale(obj, deps):
        return obj
    tmp = obj + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC,-Wno-free-nonheap-object",
           "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-c", src, "-o", tmp]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    if tuning:
        cmd.insert(1, "-DDGDIFF_TUNING")
        for f in os.environ.get("DGDIFF_TUNING_FLAGS", "").split():   # e.g. -DDGDIFF_PAIR_W=6
            cmd.insert(1, f)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or r.returncode:
        sys.stderr.write(r.stdout + r.stderr)
    if r.returncode:
        raise subprocess.CalledProcessError(r.returncode, cmd)
    os.replace(tmp, obj)
    return obj


def build_dgdiff(force=False, verbose=False, tuning=False) -> str:
    """Compile every TU in parallel (nvcc, sm_100a) and link libdgdiff.so
    (tuning=True: libdgdiff_tuning.so, see LIB_TUNING)."""
    lib = LIB_TUNING if tuning else LIB
    objdir = OBJDIR_TUNING if tuning else OBJDIR
    from concurrent.futures import ThreadPoolExecutor
    build_tables(force=force)
    srcs = [os.path.join(CSRC, f) for f in SOURCES]
    if force:
        for f in SOURCES:
            o = os.path.join(objdir, f + ".o")
            if os.path.exists(o):
                os.remove(o)
    with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda f: _compile(f, verbose, tuning), srcs))
    if not force and not _stale(lib, objs + [__file__]):
        return lib
    tmp = lib + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp] + objs + ["-ldl"])
    os.replace(tmp, lib)
    return lib


def build_all(force=False, verbose=False):
    from . import substrate
    substrate._rsa_lib()
    return build_dgdiff(force=force, verbose=verbose)


if __name__ == "__main__":
    if "--tuning" in sys.argv:
        print(build_dgdiff(force="--force" in sys.argv, verbose="-v" in sys.argv, tuning=True))
    else:
        build_all(force="--force" in sys.argv, verbose="-v" in sys.argv)
        print(LIB)
