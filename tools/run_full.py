"""A whole configuration at full size: every source of the config's source set
(c3: 4096 sources x 256 steps; c4: 65536 sources x 32 steps), in
device-memory-sized chunks, then Sigma.  Prints one JSON line (rank 0).

One GPU:
  python tools/run_full.py --config c4 [--windows 0|1|2] [--precision 64] [--temporal-steps 0|5]
The north star's strong-scaling curve (all c4 sources over 1..8 GPUs of one
node, one process per GPU, sources sharded by the library, one NCCL
all-reduce of the moment table) is one command per N:
  python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \\
         --master-port 29511 tools/run_full.py --config c4
Device time is taken on every rank with CUDA events and reduced as the max
over ranks; Sigma is bitwise the same for every N (fixed-order reduction of
the zero-padded table).
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
    ap.add_argument("--temporal-steps", type=int, default=0)
    ap.add_argument("--max-sources", type=int, default=0)
    a = ap.parse_args()
    import numpy as np
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    nccl_id = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [torch.cuda.nccl.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    from paper_1907_06191_b200 import configs
    from paper_1907_06191_b200 import dgdiff as dg
    c = configs.CONFIGS[a.config]
    m = configs.mask(a.config)
    src = configs.sources(a.config)
    if a.max_sources:
        src = src[:a.max_sources]
    nsteps = {"c3": 256, "c4": 32}.get(a.config, c.nsteps)
    st = torch.cuda.current_stream()
    # warm-up on a private one-rank handle (allocations, module load)
    with dg.Solver(m, 1.0, 1.0, c.degree, precision=a.precision, stream=st.cuda_stream, windows=a.windows,
                   temporal_steps=a.temporal_steps, device=local) as w:
        w.solve(src[:256], c.dt, 2)
        w.covariance()
    s = dg.Solver(m, 1.0, 1.0, c.degree, precision=a.precision, stream=st.cuda_stream, windows=a.windows,
                  temporal_steps=a.temporal_steps, device=local, rank=rank, nranks=world, nccl_id=nccl_id)
    dg.dgdiff_set_timing(s.handle, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    w0 = time.time()
    e0.record(st)
    s.solve(src, c.dt, nsteps)
    S, mu = s.covariance()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    wall = time.time() - w0
    if dist:
        t = torch.tensor([ms, wall], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, wall = t.tolist()
    stt = s.stats()
    mom = s.moments()
    ny, nx = m.shape
    d = (c.degree + 1) * (c.degree + 2) // 2
    dofs = 2 * nx * ny * d
    out = dict(config=a.config, grid=[nx, ny], degree=c.degree, precision=a.precision, windows=a.windows,
               temporal_steps=a.temporal_steps, n_gpus=world, scaling="strong", sources=len(src),
               nsteps=nsteps, dt=c.dt, delta=nsteps * c.dt, chunk=stt["chunk"],
               device_ms_max_over_ranks=ms, wall_s=wall,
               element_dof_updates_per_s=len(src) * dofs * nsteps / (ms * 1e-3),
               stage_gbs_rank0=stt["stage_bytes"] / (stt["stage_ms"] * 1e-3) / 1e9 if stt["stage_ms"] else None,
               sigma=[S[0, 0], S[0, 1], S[1, 1]], mu=list(mu),
               eig=list(np.linalg.eigvalsh(S)), mass_err_max=float(np.abs(mom[:, 0] - 1).max()),
               launches_rank0=stt["launches"])
    if rank == 0:
        print(json.dumps(out), flush=True)
    s.close()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
