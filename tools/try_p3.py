"""P3 (N4) stage timing on the c5 substrate (64 sources fp64 / 64 fp32), K2 ring kernel."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1907_06191_b200 import configs, dgdiff as dg  # noqa: E402

m = configs.mask("c5")
for prec in (64, 32):
    src = configs.sources("c5", 64)
    with dg.Solver(m, 1.0, 1.0, 3, precision=prec) as s:
        s.solve(src, 1 / 512, 2)
        s.covariance()
        dg.dgdiff_set_timing(s.handle, 1)
        dg.dgdiff_reset_stats(s.handle)
        s.solve(src, 1 / 512, 10)
        S, _ = s.covariance()
        st = s.stats()
    print(f"c5 P3 fp{prec} n=64: {st['stage_ms'] / 10:.3f} ms/step ({st['stage_ms'] / 30:.3f} ms/stage), "
          f"{st['stage_flops'] / (st['stage_ms'] * 1e-3) / 1e12:.2f} TFLOP/s algorithmic, Sigma {S[0, 0]:.12g}", flush=True)
