"""K3b (temporal_steps = 3) vs K2: parity on small cases and c4 timing."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1907_06191_b200 import configs, dgdiff as dg  # noqa: E402

cases = [("c1", configs.mask("c1"), configs.sources("c1"), 200)]
rng = np.random.default_rng(3)
m = (rng.random((37, 41)) < 0.4).astype(np.uint8)
free = np.argwhere(m == 0)
pick = free[rng.integers(0, len(free), 45)]
cases.append(("rand", m, np.stack([pick[:, 1], pick[:, 0]], 1).astype(np.int32), 50))
cases.append(("c3", configs.mask("c3"), configs.sources("c3")[:64], 20))
for name, mk, src, nst in cases:
    out = {}
    for ts in (0, 3):
        with dg.Solver(mk, 1.0, 1.0, 1, temporal_steps=ts, keep_density=1, max_chunk=32) as s:
            s.solve(src, 1 / 32, nst)
            out[ts] = (s.moments(), s.density(len(src) - 1))
    dm = np.abs(out[3][0] - out[0][0]).max() / np.abs(out[0][0]).max()
    dd = np.linalg.norm(out[3][1] - out[0][1]) / np.linalg.norm(out[0][1])
    print(name, "moment diff", dm, "density diff", dd, flush=True)
m = configs.mask("c4")
src = configs.sources("c4", 256)
for ts in (0, 2, 3):
    with dg.Solver(m, 1.0, 1.0, 1, temporal_steps=ts, max_chunk=256) as s:
        s.solve(src, 1 / 32, 2)
        s.covariance()
        t0 = time.perf_counter()
        s.solve(src, 1 / 32, 8)
        s.covariance()
        print("c4 ts", ts, "ms per step", (time.perf_counter() - t0) * 1e3 / 8, flush=True)
