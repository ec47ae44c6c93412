"""Projected multi-GPU scaling from logical ranks on ONE B200 (no 8-GPU node
is available to this build).  For R in {1, 2, 4, 8}, each logical rank r
(nranks = R, no communicator) solves its contiguous source shard of the job
exactly as rank r of an R-GPU run would; its device time (CUDA events on its
stream, minimum over --reps solves) is measured alone.  An R-GPU run takes max_r T_r plus one all-reduce
of the zero-padded [n][6] moment table (n*48 bytes; reported, not measured
here), so the projected speedup is T(R=1) / max_r T_r.  The host sum of the R
tables must reproduce the one-rank moments and Sigma bit for bit.
  python tools/logical_scaling.py [--config c4] [--sources 2048] [--nsteps 32] [--windows 0]
Prints one JSON line per R."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--sources", type=int, default=2048)
    ap.add_argument("--nsteps", type=int, default=32)
    ap.add_argument("--windows", type=int, default=0)
    ap.add_argument("--precision", type=int, default=64)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--diag", type=int, default=0, help="1: per-rank stage-kernel time / bytes / launches")
    a = ap.parse_args()
    import numpy as np
    import torch
    torch.cuda.set_device(0)
    from paper_1907_06191_b200 import configs
    from paper_1907_06191_b200 import dgdiff as dg
    m = configs.mask(a.config)
    src = configs.sources(a.config)[:a.sources]
    dt = 1 / 32
    st = torch.cuda.current_stream()
    diag_rows = []

    def run(r, R):
        with dg.Solver(m, 1.0, 1.0, 1, precision=a.precision, windows=a.windows, rank=r, nranks=R,
                       stream=st.cuda_stream) as s:
            s.solve(src, dt, 1)        # warm-up: kernels, tables and the full chunk buffers (allocated by solve)
            if a.diag:                 # per-launch events: stage-kernel device time and bytes
                dg.dgdiff_set_timing(s.handle, 1)
            best = None
            for _ in range(a.reps):    # min over repetitions (clock / power transients)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                dg.dgdiff_reset_stats(s.handle)
                torch.cuda.synchronize()
                e0.record(st)
                s.solve(src, dt, a.nsteps)
                mom = s.moments()
                e1.record(st)
                torch.cuda.synchronize()
                t = e0.elapsed_time(e1)
                if best is None or t < best:
                    best = t
                    if a.diag:
                        stt = s.stats()
                        drow = {"stage_ms": stt["stage_ms"], "stage_launches": stt["stage_launches"],
                                "stage_gb": stt["stage_bytes"] / 1e9, "launches": stt["launches"], "chunk": stt["chunk"]}
            if a.diag:
                diag_rows.append(drow)
            return best, mom, s

    t1, M1, _ = run(0, 1)
    with dg.Solver(m, 1.0, 1.0, 1, precision=a.precision, windows=a.windows) as s:
        S1, mu1 = s.covariance_table(M1)
    d1 = diag_rows[-1:] if a.diag else []
    for R in (1, 2, 4, 8):
        diag_rows.clear()
        times, tab = [], np.zeros_like(M1)
        for r in range(R):
            t, Mr, _ = run(r, R) if R > 1 else (t1, M1, None)
            times.append(t)
            tab += Mr
        with dg.Solver(m, 1.0, 1.0, 1, precision=a.precision, windows=a.windows) as s:
            SR, muR = s.covariance_table(tab)
        print(json.dumps({"config": a.config, "sources": int(len(src)), "nsteps": a.nsteps, "windows": a.windows,
                          "precision": a.precision, "ranks": R, "rank_ms": times, "max_rank_ms": max(times),
                          "sum_rank_ms": sum(times), "projected_speedup": t1 / max(times),
                          "allreduce_bytes": int(len(src)) * 48,
                          **({"diag": (d1 if R == 1 else list(diag_rows))} if a.diag else {}),
                          "bitwise_equal_to_one_rank": bool(np.array_equal(tab, M1) and np.array_equal(SR, S1)
                                                            and np.array_equal(muR, mu1))}), flush=True)


if __name__ == "__main__":
    main()
