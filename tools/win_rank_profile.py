"""One windowed c4 solve of logical rank r of R (all 65 536 sources, 32 steps):
the launch list under ncu shows where a rank's non-stage time goes.
  python tools/win_rank_profile.py R r"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_1907_06191_b200 import configs  # noqa: E402
from paper_1907_06191_b200 import dgdiff as dg  # noqa: E402

R, r = int(sys.argv[1]), int(sys.argv[2])
torch.cuda.set_device(0)
m = configs.mask("c4")
src = configs.sources("c4")
with dg.Solver(m, 1.0, 1.0, 1, windows=1, rank=r, nranks=R) as s:
    s.solve(src, 1 / 32, 32)
    s.moments()
