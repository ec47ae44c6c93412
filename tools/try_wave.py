"""K3c (temporal_steps = 4, wavefront step) vs K2: bitwise parity on small
cases and c4 timing.  DGDIFF_WAVE_BAND sets the band height."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1907_06191_b200 import configs, dgdiff as dg  # noqa: E402

if os.environ.get("WAVE_PARITY", "1") == "1":
    cases = [("c1", configs.mask("c1"), configs.sources("c1"), 200)]
    rng = np.random.default_rng(3)
    m = (rng.random((37, 41)) < 0.4).astype(np.uint8)
    free = np.argwhere(m == 0)
    pick = free[rng.integers(0, len(free), 45)]
    cases.append(("rand", m, np.stack([pick[:, 1], pick[:, 0]], 1).astype(np.int32), 50))
    cases.append(("c3", configs.mask("c3"), configs.sources("c3")[:70], 9))
    for name, mk, src, nst in cases:
        for deg in (1, 2):
            for prec in (64, 32):
                dt = 1 / 32 if deg == 1 else 1 / 128
                out = {}
                for ts in (0, 4):
                    with dg.Solver(mk, 1.0, 1.0, deg, precision=prec, temporal_steps=ts, keep_density=1,
                                   max_chunk=64) as s:
                        s.solve(src, dt, nst)
                        out[ts] = (s.moments(), s.density(len(src) - 1))
                same = np.array_equal(out[4][0], out[0][0]) and np.array_equal(out[4][1], out[0][1])
                dm = np.abs(out[4][0] - out[0][0]).max() / np.abs(out[0][0]).max()
                print(name, "P%d" % deg, "fp%d" % prec, "bitwise" if same else "DIFF %.3e" % dm, flush=True)
m = configs.mask("c4")
src = configs.sources("c4", 256)
for ts in [int(x) for x in os.environ.get("WAVE_TS", "0,4").split(",")]:
    with dg.Solver(m, 1.0, 1.0, 1, temporal_steps=ts, max_chunk=256) as s:
        s.solve(src, 1 / 32, 2)
        s.covariance()
        t0 = time.perf_counter()
        s.solve(src, 1 / 32, 8)
        sig = s.covariance()
        print("c4 ts", ts, "band", os.environ.get("DGDIFF_WAVE_BAND", "4"), "ms per step",
              (time.perf_counter() - t0) * 1e3 / 8, "sigma", np.asarray(sig[0]).ravel()[:2], flush=True)
