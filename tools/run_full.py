"""A whole configuration at full size on one GPU: every source of the config's
source set (c3: 4096 sources x 256 steps; c4: 65536 sources x 32 steps), in
device-memory-sized chunks, then Sigma.  Prints one JSON line.
  python tools/run_full.py --config c4 [--windows 0|1] [--precision 64] [--max-sources N]
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
    ap.add_argument("--config", default="c4")
    ap.add_argument("--windows", type=int, default=0)
    ap.add_argument("--precision", type=int, default=64)
    ap.add_argument("--max-sources", type=int, default=0)
    a = ap.parse_args()
    import numpy as np
    import torch
    torch.cuda.set_device(0)
    from paper_1907_06191_b200 import configs
    from paper_1907_06191_b200 import dgdiff as dg
    c = configs.CONFIGS[a.config]
    m = configs.mask(a.config)
    src = configs.sources(a.config)
    if a.max_sources:
        src = src[:a.max_sources]
    nsteps = {"c3": 256, "c4": 32}.get(a.config, c.nsteps)
    st = torch.cuda.current_stream()
    s = dg.Solver(m, 1.0, 1.0, 1, precision=a.precision, stream=st.cuda_stream, windows=a.windows)
    s.solve(src[:256], c.dt, 2)                # warm-up (allocations, module load)
    s.covariance()
    dg.dgdiff_reset_stats(s.handle)
    dg.dgdiff_set_timing(s.handle, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.time()
    e0.record(st)
    s.solve(src, c.dt, nsteps)
    S, mu = s.covariance()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    stt = s.stats()
    mom = s.moments()
    ny, nx = m.shape
    dofs = 2 * nx * ny * 3
    out = dict(config=a.config, grid=[nx, ny], degree=1, precision=a.precision, windows=a.windows,
               sources=len(src), nsteps=nsteps, dt=c.dt, delta=nsteps * c.dt, chunk=stt["chunk"],
               device_ms=ms, wall_s=time.time() - w0,
               element_dof_updates_per_s=len(src) * dofs * nsteps / (ms * 1e-3),
               stage_gbs=stt["stage_bytes"] / (stt["stage_ms"] * 1e-3) / 1e9 if stt["stage_ms"] else None,
               stage_share=stt["stage_ms"] / ms,
               sigma=[S[0, 0], S[0, 1], S[1, 1]], mu=list(mu),
               eig=list(np.linalg.eigvalsh(S)), mass_err_max=float(np.abs(mom[:, 0] - 1).max()),
               launches=stt["launches"])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
