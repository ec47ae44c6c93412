"""Build a variant of libdgdiff.so for A/B runs: the listed translation units
are recompiled with extra -D flags, the rest come from the product objects.
  python tools/mk_variant.py NAME "stage_ring_p3_f64.cu" -DDGDIFF_P3COL_NC=7 ...
-> scratch_libs/libdgdiff_NAME.so (copy it over libdgdiff.so on the GPU box;
tools/ab_libs.sh does that)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1907_06191_b200 import build as B  # noqa: E402

name, tus, flags = sys.argv[1], sys.argv[2].split(), sys.argv[3:]
B.build_dgdiff()
out = os.path.join(ROOT, "scratch_libs", name)
os.makedirs(out, exist_ok=True)
objs = []
for f in B.SOURCES:
    if f in tus:
        o = os.path.join(out, f + ".o")
        cmd = [B.NVCC, *B.ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC,-Wno-free-nonheap-object",
               *flags, "-I", os.path.join(ROOT, "include"), "-I", B.CSRC, "-c", os.path.join(B.CSRC, f), "-o", o,
               "-Xptxas=-v"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        for line in (r.stdout + r.stderr).splitlines():
            if "registers" in line or "spill" in line or "error" in line:
                print(f, line.strip())
        if r.returncode:
            sys.exit(r.returncode)
        objs.append(o)
    else:
        objs.append(os.path.join(B.OBJDIR, f + ".o"))
lib = os.path.join(ROOT, "scratch_libs", f"libdgdiff_{name}.so")
subprocess.check_call([B.NVCC, *B.ARCH, "-shared", "-cudart", "static", "-o", lib] + objs + ["-ldl"])
print(lib)
