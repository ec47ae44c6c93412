"""N3: DG vs Monte-Carlo under mesh refinement.

The same staircase geometry (the c3 Gamma mask, each pixel split into f x f
pixels of side h/f) and the same physical source points (the centres of 64
c3 source pixels) are solved by DG at h = 1, 1/2, 1/4 (dt = h^2/32 for P1,
h^2/128 for P2, Delta = 8); the Monte-Carlo reference runs once on the coarse
mask (identical geometry).  If the DG-MC gap is the O(h) wall error of the
paper's u+ = 0 wall flux (reading R6), it halves per refinement.
  python tools/dg_mc_refine.py [--factors 1,2,4] [--degrees 1,2] > profiles/r02_dg_mc_refine.jsonl
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
    ap.add_argument("--config", default="c3")
    ap.add_argument("--sources", type=int, default=64)
    ap.add_argument("--delta", type=float, default=8.0)
    ap.add_argument("--factors", default="1,2,4")
    ap.add_argument("--degrees", default="1,2")
    ap.add_argument("--walkers", type=int, default=20000)
    ap.add_argument("--T", type=int, default=8192)
    a = ap.parse_args()
    import numpy as np
    import torch
    torch.cuda.set_device(0)
    from paper_1907_06191_b200 import configs
    from paper_1907_06191_b200 import dgdiff as dg
    m = configs.mask(a.config)
    src = configs.sources(a.config, a.sources)
    pts = (src.astype(np.float64) + 0.5)                      # physical points (h = 1 units)
    with dg.Solver(m, 1.0, 1.0, 1) as s:
        t0 = time.time()
        Sm, mum, se = s.mc_covariance(src, a.walkers, a.T, a.delta, seed=2024)
        print(json.dumps(dict(kind="mc", config=a.config, sources=a.sources, delta=a.delta, walkers=a.walkers,
                              T=a.T, sigma=[Sm[0, 0], Sm[0, 1], Sm[1, 1]], se=list(se), seconds=time.time() - t0)),
              flush=True)
    for p in [int(x) for x in a.degrees.split(",")]:
        for f in [int(x) for x in a.factors.split(",")]:
            h = 1.0 / f
            mf = np.kron(m, np.ones((f, f), np.uint8))          # same geometry, pixels of side h
            dt = h * h / (32 if p == 1 else 128)
            nsteps = int(round(a.delta / dt))
            t0 = time.time()
            with dg.Solver(mf, h, 1.0, p, windows=1) as s:
                s.solve_points(pts, dt, nsteps)
                S, mu = s.covariance()
            gap = [(S[0, 0] - Sm[0, 0]) / Sm[0, 0], (S[1, 1] - Sm[1, 1]) / Sm[1, 1]]
            print(json.dumps(dict(kind="dg", degree=p, refine=f, h=h, grid=list(mf.shape), dt=dt, nsteps=nsteps,
                                  sigma=[S[0, 0], S[0, 1], S[1, 1]], rel_gap_vs_mc=gap,
                                  mean_abs_gap=float(np.mean(np.abs(gap))), seconds=time.time() - t0)), flush=True)


if __name__ == "__main__":
    main()
