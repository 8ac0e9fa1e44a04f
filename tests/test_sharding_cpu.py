"""Multi-rank host logic on CPU (gloo, world_size 2): member sharding and the
allreduce of the barycenter objective/gradient reproduce the single-process
objective (barycenter.hpp:60-86); pair sharding covers every pair once."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_17206_b200.sharding import shard_range, sharded_barycenter_objective


@pytest.mark.parametrize("n,world", [(1024, 8), (1024, 3), (7, 4), (3, 8), (0, 2)])
def test_shard_range_partition(n, world):
    seen = []
    for r in range(world):
        lo, hi = shard_range(n, world, r)
        assert 0 <= lo <= hi <= n
        assert hi - lo in (n // world, n // world + 1)
        seen.extend(range(lo, hi))
    assert seen == list(range(n))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, z, members, weights, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    orc = oracle.OracleC()

    def objective(zz, mm, ww):
        return orc.barycenter_objective(zz, mm, 1.0, 0, ww)

    def allreduce(v, g):
        t = torch.from_numpy(np.concatenate([[v], g.ravel()]))
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        a = t.numpy()
        return float(a[0]), a[1:].reshape(g.shape)

    v, g = sharded_barycenter_objective(objective, allreduce, z, members, weights, world, rank)
    out[rank] = (v, g)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("weighted", [False, True])
def test_sharded_barycenter_matches_single_process(weighted):
    import oracle
    rng = np.random.default_rng(5)
    members = rng.standard_normal((5, 17, 3))
    z = rng.standard_normal((13, 3))
    weights = rng.uniform(0.2, 1.0, 5) if weighted else None
    v_ref, g_ref = oracle.OracleC().barycenter_objective(z, members, 1.0, 0, weights)
    world = 2
    with mp.Manager() as man:
        out = man.dict()
        mp.spawn(_worker, args=(world, _free_port(), z, members, weights, out), nprocs=world, join=True)
        res = dict(out)
    for r in range(world):
        v, g = res[r]
        assert abs(v - v_ref) <= 1e-12 * max(1.0, abs(v_ref))
        np.testing.assert_allclose(g, g_ref, rtol=1e-12, atol=1e-12)
