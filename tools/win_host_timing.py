"""Host vs device time of one windowed c4 solve per logical rank (R, r):
  python tools/win_host_timing.py R r
prints the host time of the solve call (enqueue + host set-up + syncs inside
the library), the device interval (CUDA events) and the stage-kernel time."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_1907_06191_b200 import configs  # noqa: E402
from paper_1907_06191_b200 import dgdiff as dg  # noqa: E402

R, r = int(sys.argv[1]), int(sys.argv[2])
NST = int(sys.argv[3]) if len(sys.argv) > 3 else 32
torch.cuda.set_device(0)
m = configs.mask("c4")
src = configs.sources("c4")
st = torch.cuda.current_stream()
with dg.Solver(m, 1.0, 1.0, 1, windows=1, rank=r, nranks=R, stream=st.cuda_stream) as s:
    s.solve(src, 1 / 32, 1)
    dg.dgdiff_set_timing(s.handle, 1)
    for rep in range(2):
        dg.dgdiff_reset_stats(s.handle)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        t0 = time.perf_counter()
        s.solve(src, 1 / 32, NST)
        t1 = time.perf_counter()
        s.moments()
        e1.record(st)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        stt = s.stats()
        print(f"R={R} r={r} nsteps={NST}: host solve call {1e3*(t1-t0):.0f} ms, wall to sync {1e3*(t2-t0):.0f} ms, "
              f"device {e0.elapsed_time(e1):.0f} ms, stage kernels {stt['stage_ms']:.0f} ms, launches {stt['launches']}")
