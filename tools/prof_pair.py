"""One c4 chunk (256 sources fp64 P1) for 2 steps with K3d (temporal_steps 5):
the ncu target of the stage-pair kernel."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1907_06191_b200 import configs, dgdiff as dg  # noqa: E402

ts = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cfg = sys.argv[2] if len(sys.argv) > 2 else "c4"
n = 256 if cfg == "c4" else 64
with dg.Solver(configs.mask(cfg), 1.0, 1.0, configs.CONFIGS[cfg].degree, temporal_steps=ts) as s:
    s.solve(configs.sources(cfg, n), configs.CONFIGS[cfg].dt, 2)
    print(s.covariance()[0])
