#!/usr/bin/env python
"""Benchmark of the hot path on B200.

One bench step = one pass of the whole hot path over one batch: Dirac data
(K1), 32 SSP-RK3 steps (3 x K2 each), moments (K4), the moment all-reduce
(N > 1) and Sigma (K5), through the C-ABI (dgdiff_solve_batch +
dgdiff_covariance).  Workload: the c4 substrate (2048^2 Gamma axons, f = 0.60,
seed 5), 256 sources per GPU per step drawn in order from the c4 source set
(seed 6), P1, fp64 by default, dt = 1/32 (grid units h = D = 1).

Metric (BASELINE.json): element-dof updates/s = sources x 2 nx ny d x nsteps
/ time, whole job, all dofs (axon pixels included, as the paper's whole-domain
solve counts them); the active-dof rate, Sigma solves/s and the stage
kernel's HBM roofline fraction are reported beside it.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--precision 64|32]
  python bench.py --impl reference ...   # the CPU oracle, bounded sample
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NX = NY = 2048
NSTEPS = 32
DT = 1.0 / 32
SRC_PER_GPU = 256
DEFAULT_TS = 0      # the bench's kernel path (see --temporal-steps)
METRIC = "element-dof updates/s and \u03a3 solves/s at 1/2/4/8 B200; % of HBM roofline"
UNIT = "element-dof updates/s"


def step_dt(degree):
    """dt of the bench step: 1/32 (P1) and 1/128 (P2, the P2 stability limit is ~1/77)."""
    return DT if degree == 1 else DT / 4


TS_NAMES = {0: "K2 per-stage ring kernel (3 launches per SSP-RK3 step)",
            5: "K3d: stage 1 on K2 + stages 2-3 fused in one launch (2 launches per step)"}


def workload_cfg(args, n_gpus):
    dt = step_dt(args.degree)
    return {
        "workload": f"c4: {NX}x{NY} Gamma-axon substrate (f=0.60, seed 5), {SRC_PER_GPU} point sources per GPU per "
                    f"step from the c4 source set (seed 6), P{args.degree}, dt=1/{round(1 / dt)}, {NSTEPS} SSP-RK3 "
                    f"steps, moments + Sigma",
        "kernel_path": TS_NAMES.get(args.temporal_steps, f"temporal_steps={args.temporal_steps}"),
        "grid": [NX, NY],
        "degree": args.degree,
        "sources_per_step": SRC_PER_GPU * n_gpus,
        "nsteps": NSTEPS,
        "precision": args.precision,
        "l2": "inputs larger than L2: the per-GPU state is ~62 GB (fp64) vs 126 MB L2",
        "parallelism": f"dp{n_gpus} (sources sharded, one NCCL all-reduce of the moment table per step)",
        **({"windows": "N1 exact active windows: Morton-sorted source groups, every stage clipped to the group's "
                       "source box grown by one pixel per stage (bitwise equal to the whole-grid solve); value "
                       "still counts every element of the grid"} if getattr(args, "windows", 0) == 1 else {}),
        **({"windows": "N1 windows clipped at K sigma (K = 20 for P1; moments within 1e-12 of the whole-grid "
                       "solve); value still counts every element of the grid"}
           if getattr(args, "windows", 0) == 2 else {}),
    }


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.rows = []
        if self.p is None:
            return
        self.p.terminate()
        try:
            out, _ = self.p.communicate(timeout=5)
        except Exception:
            self.p.kill()
            out = ""
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                self.rows.append(f)

    def summary(self):
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[5 + k].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ----------------------------------------------------------------------------- CPU oracle legs
def oracle_sample(mask, sources, degree, nthreads, nsteps, dt=DT):
    """Time the oracle (as it stands) on `len(sources)` sources x nsteps."""
    from oracle import oracle as O
    O.build()
    t0 = time.perf_counter()
    O.solve(degree, 1.0, 1.0, mask, sources, dt, nsteps, nthreads=nthreads)
    return time.perf_counter() - t0


def oracle_threads():
    """All host threads this process may use (no cap)."""
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except Exception:
        return max(1, os.cpu_count() or 1)


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_baseline(mask, sources, degree):
    """O1 as it stands (test infrastructure) on the host: one source x two
    steps on one core, and nproc sources x two steps on all cores (one OpenMP
    thread per source); ~12 s on the c4 substrate."""
    th = oracle_threads()
    d = (degree + 1) * (degree + 2) // 2
    per = 2 * NX * NY * d                                   # element-dofs per source-step
    t1 = oracle_sample(mask, sources[:1], degree, 1, 2)
    ta = oracle_sample(mask, sources[:th], degree, th, 2)
    one, allc = 2 * per / t1, 2 * th * per / ta
    return {"value": allc, "unit": UNIT, "cores": th, "kind": "oracle",
            "one_core": one, "all_cores": allc, "nproc": os.cpu_count(), "cpu_model": cpu_model(),
            "sample": f"same {NX}x{NY} c4 substrate, O1 fp64: 1 source x 2 SSP-RK3 steps on 1 core ({t1:.1f} s) and "
                      f"{th} sources x 2 steps on {th} threads ({ta:.1f} s)"}


def run_reference(args):
    world, rank, local = dist_env()
    if rank != 0:
        return 0
    from paper_1907_06191_b200 import configs
    mask = configs.mask("c4")
    sources = configs.sources("c4")
    th = oracle_threads()
    d = (args.degree + 1) * (args.degree + 2) // 2
    nsteps = 1
    dt = step_dt(args.degree)
    times = []
    for k in range(args.warmup + args.steps):
        src = sources[k * th:(k + 1) * th]
        t = oracle_sample(mask, src, args.degree, th, nsteps, dt)
        if k >= args.warmup:
            times.append(t)
    work = th * 2 * NX * NY * d * nsteps
    value = work * len(times) / sum(times)
    sample = (f"per step: {th} sources x {nsteps} SSP-RK3 step on the {NX}x{NY} c4 substrate (O1 fp64, "
              f"{th} OpenMP threads); the GPU arm's step is {SRC_PER_GPU} sources x {NSTEPS} steps")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_cfg(args, world) | {"note": "bounded oracle sample"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": th, "kind": "oracle",
                             "nproc": os.cpu_count(), "cpu_model": cpu_model(), "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU arm
def measure_k3d(args, dg, mask, batch, dt, nsteps, per_step, dofs, dist, stream, rank, world, local, nccl_id, peak):
    """K3d (temporal_steps = 5: stage 1 on K2, stages 2 + 3 fused; bitwise equal
    to K2) on the bench workload: 1 warm-up + k3d_steps timed steps."""
    import torch
    s = dg.Solver(mask, 1.0, 1.0, args.degree, precision=args.precision, rank=rank, nranks=world, nccl_id=nccl_id,
                  stream=stream.cuda_stream, device=local, max_chunk=SRC_PER_GPU, temporal_steps=5)
    try:
        s.solve(batch(0), dt, nsteps)
        S0, _ = s.covariance()
        torch.cuda.synchronize()
        dg.dgdiff_reset_stats(s.handle)
        dg.dgdiff_set_timing(s.handle, 1)
        if dist:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for k in range(args.k3d_steps):
            s.solve(batch(args.warmup + k), dt, nsteps)
            s.covariance()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if dist:
            t = torch.tensor([ms], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = t.item()
        st = s.stats()
        pl_b = st["dom_bytes"] / max(1, st["dom_launches"])
        pl_ms = st["dom_ms"] / max(1, st["dom_launches"])
        ach = pl_b / (pl_ms * 1e-3) / 1e9 if pl_ms > 0 else None
        return {"value": per_step * args.k3d_steps * dofs * nsteps / (ms * 1e-3), "unit": UNIT,
                "ms_per_step": ms / args.k3d_steps, "steps": args.k3d_steps,
                "sigma_first_batch": [S0[0, 0], S0[0, 1], S0[1, 1]],
                "pair_kernel": {"achieved_gbs": ach, "frac_of_hbm": ach / peak if ach else None,
                                "avg_launch_ms": pl_ms, "algorithmic_bytes_per_launch": pl_b,
                                "share_of_step": st["dom_ms"] / ms if ms > 0 else None},
                "note": "stage 1 on K2 + k_stage_pair (SSP-RK3 stages 2-3 fused, U2 in shared memory); "
                        "5 state passes per step instead of 8; bitwise equal to K2"}
    finally:
        s.close()


def measure_adjoint(args, dg, mask, all_src, dt, nsteps, stream, rank, world, local, peak_unused=None):
    """Adjoint moments (opts.adjoint = 1) for the WHOLE source set of the
    configuration (c4: all 65 536 sources) x nsteps: one solve + covariance,
    timed with CUDA events after a warm-up; logical ranks take their shard
    (no communicator here: this is a side measurement, Sigma from rank 0's
    table when world == 1)."""
    import torch
    s = dg.Solver(mask, 1.0, 1.0, args.degree, adjoint=1, stream=stream.cuda_stream, device=local)
    try:
        s.solve(all_src[:64], dt, 1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s.solve(all_src, dt, nsteps)
        S, _ = s.covariance()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        return {"sources": int(len(all_src)), "nsteps": nsteps, "ms": ms, "sigma_solves_per_s": 1e3 / ms,
                "sigma": [S[0, 0], S[0, 1], S[1, 1]],
                "note": "moments of every source from a few source groups of weight fields stepped with the "
                        "transposed operator (ring kernel, the sources' domain of dependence) and read at each "
                        "source pixel; the same Sigma as the per-source solves of the whole job up to rounding "
                        "(DESIGN 9b, N5)"}
    finally:
        s.close()


def run_ours(args):
    import torch
    world, rank, local = dist_env()
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1907_06191_b200 import configs
    from paper_1907_06191_b200 import dgdiff as dg
    mask = configs.mask("c4")
    all_src = configs.sources("c4")
    d = (args.degree + 1) * (args.degree + 2) // 2
    nccl_id = None
    if world > 1:
        obj = [torch.cuda.nccl.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    stream = torch.cuda.current_stream()
    solver = dg.Solver(mask, 1.0, 1.0, args.degree, precision=args.precision, rank=rank, nranks=world,
                       nccl_id=nccl_id, stream=stream.cuda_stream, device=local, max_chunk=SRC_PER_GPU,
                       windows=args.windows, temporal_steps=args.temporal_steps)
    per_step = SRC_PER_GPU * world
    dt = step_dt(args.degree)
    nsteps = NSTEPS

    # the step's sources live in pinned host memory (the e2e leg copies them
    # host -> device inside the timed region; covariance() synchronises each
    # step, so the buffer is free again before the next step refills it)
    pinned = torch.empty((per_step, 2), dtype=torch.int32).pin_memory()
    pinned_np = pinned.numpy()

    def batch(k):
        off = (k * per_step) % (len(all_src) - per_step + 1)
        pinned_np[:] = all_src[off:off + per_step]
        return pinned_np

    def step(k):
        solver.solve(batch(k), dt, nsteps)
        return solver.covariance()

    for k in range(args.warmup):
        step(k)
    torch.cuda.synchronize()
    dg.dgdiff_reset_stats(solver.handle)
    dg.dgdiff_set_timing(solver.handle, 1)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        w0 = time.perf_counter()
        ev0.record(stream)
        for k in range(args.steps):
            S, mu = step(args.warmup + k)
        ev1.record(stream)
        torch.cuda.synchronize()
        w1 = time.perf_counter()
    if dist:
        dist.barrier()
    dev_ms = ev0.elapsed_time(ev1)
    wall_ms = (w1 - w0) * 1e3
    st = dg.dgdiff_get_stats(solver.handle)
    if dist:
        t = torch.tensor([dev_ms, wall_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms, wall_ms = t.tolist()
    total_src = per_step * args.steps
    dofs = 2 * NX * NY * d
    value = total_src * dofs * nsteps / (dev_ms * 1e-3)
    e2e = total_src * dofs * nsteps / (wall_ms * 1e-3)
    n_act = st["n_active"]
    active = total_src * n_act * 2 * d * nsteps / (dev_ms * 1e-3)
    peak, peak_src = peaks()
    # the dominant kernel: K2's stage kernel, or K3d's stage-pair kernel
    per_launch_bytes = st["dom_bytes"] / max(1, st["dom_launches"])
    per_launch_ms = st["dom_ms"] / max(1, st["dom_launches"])
    achieved = per_launch_bytes / (per_launch_ms * 1e-3) / 1e9 if per_launch_ms > 0 else None
    kname = "k_stage_pair (K3d: SSP-RK3 stages 2+3 fused)" if args.temporal_steps == 5 else \
        "k_stage_ring (K2: one SSP-RK3 stage)"
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "stage_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tj = json.load(f)
        key = f"{'pair' if args.temporal_steps == 5 else 'ring'}_p{args.degree}_fp{args.precision}"
        if key in tj and not args.windows:
            traffic, traffic_src = tj[key], tj.get("_source")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64" if args.precision == 64 else "f32", "data": "synthetic",
        "config": workload_cfg(args, world),
        "active_dof_updates_per_s": active,
        "sigma_solves_per_s": args.steps / (dev_ms * 1e-3),
        "sigma_last": [S[0, 0], S[0, 1], S[1, 1]],
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "traffic_source": traffic_src,
                     "kernel": kname, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": per_launch_bytes,
                     "avg_launch_ms": per_launch_ms,
                     "share_of_step": st["dom_ms"] / dev_ms if dev_ms > 0 else None,
                     "stepping_share_of_step": st["stage_ms"] / dev_ms if dev_ms > 0 else None},
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": st["h2d_bytes"],
                "d2h_bytes_per_step": st["d2h_bytes"],
                "note": "wall clock around dgdiff_solve_batch(sources in pinned host memory) + "
                        "dgdiff_covariance(Sigma to host)"},
        "gpu_launches": st["launches"],
        "clocks": clk.summary(),
        "library": {"env_overrides": st["env_overrides"], "tuning_build": st["tuning_build"],
                    "temporal_steps": args.temporal_steps},
    }
    solver.close()
    # the temporal-blocked path (K3d) on the same workload, beside the default
    # K2 line: a short extra measurement (device time, same step definition)
    if args.temporal_steps == 0 and args.degree == 1 and not args.windows and args.k3d_steps > 0:
        line["k3d"] = measure_k3d(args, dg, mask, batch, dt, nsteps, per_step, dofs, dist, stream, rank, world,
                                  local, nccl_id, peak)
    if rank == 0 and world == 1 and args.precision == 64 and not args.windows and args.adjoint_job:
        line["adjoint_full_job"] = measure_adjoint(args, dg, mask, all_src, dt, nsteps, stream, rank, world, local)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(mask, all_src, args.degree)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", type=int, default=64, choices=[64, 32])
    ap.add_argument("--degree", type=int, default=1, choices=[1, 2])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--adjoint-job", type=int, default=1,
                    help="1: also time the adjoint-moment solve of the whole source set (Sigma of the full job)")
    ap.add_argument("--k3d-steps", type=int, default=3,
                    help="extra K3d steps timed beside the default K2 line (0 = skip)")
    ap.add_argument("--temporal-steps", type=int, default=DEFAULT_TS, choices=[0, 5],
                    help="0: K2, one launch per SSP-RK3 stage; 5: K3d, stages 2+3 fused (bitwise equal)")
    ap.add_argument("--windows", type=int, default=0, choices=[0, 1, 2],
                    help="N1 active windows: 1 exact (bitwise), 2 also clipped at K sigma; not the default "
                         "(the headline is the whole-grid solve)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("note: warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
