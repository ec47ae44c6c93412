"""DG vs Monte-Carlo covariance on a Gamma substrate (N3 cross-check).
  python tools/dg_vs_mc.py [--config c3] [--sources 64] [--nsteps 256] [--walkers 20000] [--T 2000]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--sources", type=int, default=64)
    ap.add_argument("--nsteps", type=int, default=256)
    ap.add_argument("--walkers", type=int, default=20000)
    ap.add_argument("--T", type=int, default=2000)
    ap.add_argument("--degree", type=int, default=1)
    a = ap.parse_args()
    import numpy as np
    import torch
    torch.cuda.set_device(0)
    from paper_1907_06191_b200 import configs
    from paper_1907_06191_b200 import dgdiff as dg
    m = configs.mask(a.config)
    src = configs.sources(a.config, a.sources)
    dt = 1 / 32 if a.degree == 1 else 1 / 128
    delta = a.nsteps * dt
    out = {}
    with dg.Solver(m, 1.0, 1.0, a.degree) as s:
        s.solve(src, dt, a.nsteps)
        S, mu = s.covariance()
        Sm, mum, se = s.mc_covariance(src, a.walkers, a.T, delta, seed=2024)
    out = dict(config=a.config, sources=a.sources, delta=delta, degree=a.degree, dg=[S[0, 0], S[0, 1], S[1, 1]],
               mc=[Sm[0, 0], Sm[0, 1], Sm[1, 1]], mc_se=list(se), free=2 * delta,
               rel_diff=[(Sm[0, 0] - S[0, 0]) / S[0, 0], (Sm[1, 1] - S[1, 1]) / S[1, 1]],
               dg_mu=list(mu), mc_mu=list(mum), walkers=a.walkers * a.sources, T=a.T)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
