"""Config c5 at full length: 1024^2 Gamma substrate (seed 7), P2, 64 sources
(seed 8), dt = 1/128, 1e5 SSP-RK3 steps (Delta = 781.25, sigma ~ 40 px).
Prints one JSON line: device time, element-dof updates/s, Sigma, mass.
  python tools/run_c5.py [--nsteps 100000] [--precision 64]
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
    ap.add_argument("--nsteps", type=int, default=100000)
    ap.add_argument("--precision", type=int, default=64)
    ap.add_argument("--element", type=int, default=0, help="1 = quadrilateral Q2 (N4)")
    a = ap.parse_args()
    import numpy as np
    import torch
    torch.cuda.set_device(0)
    from paper_1907_06191_b200 import configs
    from paper_1907_06191_b200 import dgdiff as dg
    m = configs.mask("c5")
    src = configs.sources("c5")
    st = torch.cuda.current_stream()
    s = dg.Solver(m, 1.0, 1.0, 2, precision=a.precision, stream=st.cuda_stream, element=a.element)
    dt = 1 / 128
    s.solve(src, dt, 10)                       # warm-up
    s.covariance()
    dg.dgdiff_reset_stats(s.handle)
    dg.dgdiff_set_timing(s.handle, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.time()
    e0.record(st)
    s.solve(src, dt, a.nsteps)
    S, mu = s.covariance()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    stt = s.stats()
    mom = s.moments()
    ny, nx = m.shape
    dofs = nx * ny * (9 if a.element else 12)
    delta = a.nsteps * dt
    out = dict(config="c5", grid=[nx, ny], degree=2, element="Q2" if a.element else "P2", precision=a.precision, sources=len(src), nsteps=a.nsteps,
               dt=dt, delta=delta, device_ms=ms, wall_s=time.time() - w0,
               element_dof_updates_per_s=len(src) * dofs * a.nsteps / (ms * 1e-3),
               stage_gbs=stt["stage_bytes"] / (stt["stage_ms"] * 1e-3) / 1e9,
               stage_tflops=stt["stage_flops"] / (stt["stage_ms"] * 1e-3) / 1e12,
               sigma=[S[0, 0], S[0, 1], S[1, 1]], mu=list(mu), sigma_over_2DDelta=[S[0, 0] / (2 * delta), S[1, 1] / (2 * delta)],
               mass_err_max=float(np.abs(mom[:, 0] - 1).max()), launches=stt["launches"])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
