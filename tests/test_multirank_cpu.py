"""N > 1 host logic on CPU with gloo (world size 2): every rank shards the
full source list with dgdiff_shard, computes its rows of the moment table
(here with the oracle, standing in for the GPU kernels), zero-pads the rest,
and all-reduces with SUM -- the exact collective dgdiff_covariance issues with
NCCL.  Disjoint rows plus zeros make the sum exact, so the table and Sigma
must be bitwise identical to the single-rank run."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case():
    rng = np.random.default_rng(77)
    mask = (rng.random((14, 15)) < 0.35).astype(np.uint8)
    free = np.argwhere(mask == 0)
    pick = free[rng.integers(0, len(free), 9)]          # odd count: uneven shards
    return mask, np.stack([pick[:, 1], pick[:, 0]], 1).astype(np.int32)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    from oracle import oracle as O
    from paper_1907_06191_b200 import dgdiff as dg
    mask, src = _case()
    n = len(src)
    b, e = dg.dgdiff_shard(n, rank, world)
    table = np.zeros((n, 6))
    if e > b:
        table[b:e] = O.solve(1, 1.0, 1.0, mask, src[b:e], 1 / 32, 30, nthreads=1)
    t = torch.from_numpy(table)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    S, mu = O.sigma(t.numpy())
    out[rank] = (t.numpy().copy(), S, mu, (b, e))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_moment_table_is_exact(world):
    from oracle import oracle as O
    O.build()
    from paper_1907_06191_b200 import build
    build.build_all()
    mask, src = _case()
    full = O.solve(1, 1.0, 1.0, mask, src, 1 / 32, 30, nthreads=1)
    S_ref, mu_ref = O.sigma(full)
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, out), nprocs=world, join=True, start_method="spawn")
    spans = sorted(out[r][3] for r in range(world))
    assert spans[0][0] == 0 and spans[-1][1] == len(src)
    assert all(spans[k][1] == spans[k + 1][0] for k in range(world - 1))
    for r in range(world):
        table, S, mu, _ = out[r]
        assert np.array_equal(table, full)          # bitwise: disjoint rows + zeros
        assert np.array_equal(S, S_ref)
        assert np.array_equal(mu, mu_ref)
