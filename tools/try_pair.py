"""K3d (temporal_steps = 5, fused stages 2 + 3) vs K2: device time per step on
the c4 bench chunk (256 sources fp64 P1, 128 fp32), c5 P2 and c3, from the
library's CUDA-event stage timing; Sigma compared bitwise.

    python tools/try_pair.py [ts,ts,...]      (default 0,5)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1907_06191_b200 import configs, dgdiff as dg  # noqa: E402

tss = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "0,5").split(",")]
cases = [("c4", 1, 64, 256, 1 / 32, 8), ("c4", 1, 32, 256, 1 / 32, 8), ("c5", 2, 64, 64, 1 / 128, 40),
         ("c3", 1, 64, 1024, 1 / 32, 16)]
only = os.environ.get("PAIR_CASES")
if only:
    cases = [c for c in cases if f"{c[0]}_p{c[1]}_fp{c[2]}" in only.split(",")]
for name, deg, prec, n, dt, nsteps in cases:
    m = configs.mask(name)
    src = configs.sources(name, n)
    ref = None
    for ts in tss:
        with dg.Solver(m, 1.0, 1.0, deg, precision=prec, temporal_steps=ts) as s:
            s.solve(src, dt, 2)
            s.covariance()
            dg.dgdiff_set_timing(s.handle, 1)
            dg.dgdiff_reset_stats(s.handle)
            s.solve(src, dt, nsteps)
            S, _ = s.covariance()
            st = s.stats()
        ms = st["stage_ms"] / nsteps
        gbs = st["stage_bytes"] / (st["stage_ms"] * 1e-3) / 1e9
        same = "" if ref is None else ("bitwise" if np.array_equal(S, ref) else "DIFF %.2e" % np.abs(S - ref).max())
        ref = S if ref is None else ref
        print(f"{name} P{deg} fp{prec} n={n} ts={ts}: {ms:.3f} ms/step  (algorithmic {gbs:.0f} GB/s, "
              f"{st['stage_bytes'] / nsteps / 1e9:.1f} GB/step)  Sigma {S[0, 0]:.12g} {same}", flush=True)
