"""Small driver for ncu / timing of the stage kernel on the c4 substrate.

  python tools/prof_stage.py [--precision 64] [--kernel 0] [--sources 256] [--nsteps 2] [--reps 2]
Runs `reps` solves (the first is warm-up) and prints per-launch stage time
and achieved algorithmic GB/s from the library's CUDA-event timing.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--precision", type=int, default=64)
    ap.add_argument("--kernel", type=int, default=0)
    ap.add_argument("--degree", type=int, default=1)
    ap.add_argument("--sources", type=int, default=256)
    ap.add_argument("--nsteps", type=int, default=2)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--tb", type=int, default=0)
    ap.add_argument("--windows", type=int, default=0)
    ap.add_argument("--element", type=int, default=0)
    a = ap.parse_args()
    import torch
    torch.cuda.set_device(0)
    from paper_1907_06191_b200 import configs
    from paper_1907_06191_b200 import dgdiff as dg
    m = configs.mask(a.config)
    src = configs.sources(a.config)[:a.sources] if a.config != "c1" else configs.sources("c1")
    dt = ({1: 1 / 16, 2: 1 / 64} if a.element else {1: 1 / 32, 2: 1 / 128, 3: 1 / 256})[a.degree]
    s = dg.Solver(m, 1.0, 1.0, a.degree, precision=a.precision, kernel=a.kernel, temporal_steps=a.tb,
                  max_chunk=max(a.sources, 64), windows=a.windows, element=a.element)
    out = []
    for r in range(a.reps):
        dg.dgdiff_reset_stats(s.handle)
        dg.dgdiff_set_timing(s.handle, 1)
        t0 = time.perf_counter()
        s.solve(src, dt, a.nsteps)
        S, mu = s.covariance()
        wall = (time.perf_counter() - t0) * 1e3
        st = s.stats()
        ms = st["stage_ms"] / max(1, st["stage_launches"])
        gbs = st["stage_bytes"] / max(1, st["stage_launches"]) / (ms * 1e-3) / 1e9 if ms else 0
        out.append(dict(rep=r, wall_ms=wall, stage_ms=ms, gbs=gbs, launches=st["launches"], chunk=st["chunk"],
                        sigma=[S[0, 0], S[0, 1], S[1, 1]]))
    print(json.dumps(dict(args=vars(a), runs=out)))


if __name__ == "__main__":
    main()
