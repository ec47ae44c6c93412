"""Cost of the N2 mixture grid on the bench workload: c4, 256 sources x 32
steps, with and without mixture_radius (ms per solve, CUDA events)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_1907_06191_b200 import configs  # noqa: E402
from paper_1907_06191_b200 import dgdiff as dg  # noqa: E402

torch.cuda.set_device(0)
m = configs.mask("c4")
src = configs.sources("c4")[:256]
st = torch.cuda.current_stream()
for R in (0, 16, 64):
    with dg.Solver(m, 1.0, 1.0, 1, mixture_radius=R, stream=st.cuda_stream) as s:
        s.solve(src, 1 / 32, 1)
        for rep in range(2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(st)
            s.solve(src, 1 / 32, 32)
            s.covariance()
            if R:
                s.mixture()
            e1.record(st)
            torch.cuda.synchronize()
        print(f"mixture_radius={R}: {e0.elapsed_time(e1):.1f} ms per solve+covariance(+mixture)", flush=True)
