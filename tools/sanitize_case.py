"""Small solves for compute-sanitizer (racecheck / synccheck / memcheck) of the
pipelined kernels: K2 k_stage_ring (P1, P2; fp64, fp32; REFLECT, ABSORB;
windows) and K3c k_step_wave.  Run under the sanitizer, e.g.

    compute-sanitizer --tool racecheck python tools/sanitize_case.py ring
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_06191_b200 import configs, dgdiff as dg   # noqa: E402


def cases(which):
    rng = np.random.default_rng(5)
    m = (rng.random((40, 72)) < 0.45).astype(np.uint8)
    free = np.argwhere(m == 0)
    src = free[rng.integers(0, len(free), 70)][:, ::-1].astype(np.int32)
    c1 = configs.mask("c1")
    if which == "ring":
        yield "c1 P1 fp64", dict(mask=c1, p=1, opts={}, src=configs.sources("c1"), dt=1 / 32, n=4)
        yield "rand P1 fp64 2 groups", dict(mask=m, p=1, opts={}, src=src, dt=1 / 32, n=3)
        yield "rand P1 fp32", dict(mask=m, p=1, opts=dict(precision=32), src=src, dt=1 / 32, n=3)
        yield "rand P2 fp64", dict(mask=m, p=2, opts={}, src=src, dt=1 / 128, n=2)
        yield "rand P1 ABSORB", dict(mask=m, p=1, opts=dict(outer_bc=1), src=src, dt=1 / 32, n=2)
        yield "rand P1 windows", dict(mask=m, p=1, opts=dict(windows=1), src=src, dt=1 / 32, n=3)
    elif which == "wave":
        yield "rand P1 fp64 K3c", dict(mask=m, p=1, opts=dict(temporal_steps=4), src=src, dt=1 / 32, n=2)
        yield "rand P2 fp64 K3c", dict(mask=m, p=2, opts=dict(temporal_steps=4), src=src, dt=1 / 128, n=2)
    elif which == "fused":
        yield "rand P1 fp64 K3", dict(mask=m, p=1, opts=dict(temporal_steps=5), src=src, dt=1 / 32, n=2)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "ring"
    for name, c in cases(which):
        with dg.Solver(c["mask"], 1.0, 1.0, c["p"], **c["opts"]) as s:
            s.solve(c["src"], c["dt"], c["n"])
            S, _ = s.covariance()
        print(f"{name}: Sigma {S.ravel().tolist()}", flush=True)
