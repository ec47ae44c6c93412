"""Adjoint moments (opts.adjoint) on the full c4 job: all 65 536 sources x 32
steps, fp64 P1.  Times one adjoint solve + covariance (CUDA events) against
the per-source solves (N1 exact windows: the fastest forward path; and the
bench's whole-grid rate), and checks the moments against the stored O1
answers of tests/golden/c4_o1.npz and against the per-source GPU solve.
  python tools/adjoint_bench.py [--forward-windows 1]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--nsteps", type=int, default=32)
    ap.add_argument("--degree", type=int, default=1)
    ap.add_argument("--forward-windows", type=int, default=1)
    a = ap.parse_args()
    import numpy as np
    import torch
    torch.cuda.set_device(0)
    from paper_1907_06191_b200 import configs
    from paper_1907_06191_b200 import dgdiff as dg
    m = configs.mask(a.config)
    src = configs.sources(a.config)
    dt = 1 / 32 if a.degree == 1 else 1 / 128
    st = torch.cuda.current_stream()

    def timed(solver):
        solver.solve(src[:64], dt, 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        solver.solve(src, dt, a.nsteps)
        S, mu = solver.covariance()
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1), S, solver.moments()

    with dg.Solver(m, 1.0, 1.0, a.degree, adjoint=1, stream=st.cuda_stream) as s:
        t_adj, S_adj, M_adj = timed(s)
    with dg.Solver(m, 1.0, 1.0, a.degree, windows=a.forward_windows, stream=st.cuda_stream) as s:
        t_fwd, S_fwd, M_fwd = timed(s)
    scale = np.maximum(np.abs(M_fwd[:, 3:4]) + np.abs(M_fwd[:, 5:6]), 1e-300)
    out = {"config": a.config, "degree": a.degree, "sources": int(len(src)), "nsteps": a.nsteps,
           "adjoint_ms": t_adj, "forward_ms": t_fwd, "forward_windows": a.forward_windows,
           "speedup": t_fwd / t_adj, "sigma_adjoint": S_adj.tolist(), "sigma_forward": S_fwd.tolist(),
           "sigma_rel_diff": float(np.abs(S_adj - S_fwd).max() / max(S_fwd[0, 0], S_fwd[1, 1])),
           "m00_max_diff": float(np.abs(M_adj[:, 0] - M_fwd[:, 0]).max()),
           "second_moment_rel_diff_max": float((np.abs(M_adj[:, 3:] - M_fwd[:, 3:]) / scale).max())}
    gp = os.path.join(ROOT, "tests", "golden", f"{a.config}_o1.npz")
    if os.path.exists(gp) and a.degree == 1 and a.nsteps == 32:
        z = np.load(gp)
        idx = z["idx"]
        r = z["mom"]
        sc = np.maximum(np.abs(r[:, 3:4]) + np.abs(r[:, 5:6]), 1e-300)
        out["vs_oracle_second_moment_rel_max"] = float((np.abs(M_adj[idx, 3:] - r[:, 3:]) / sc).max())
        out["vs_oracle_m00_max"] = float(np.abs(M_adj[idx, 0] - r[:, 0]).max())
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
