"""Multi-GPU host logic: how the hot path is split over ranks.

* Soft-DTW batches (sdtw_with_gradients): pairs are independent problems
  (backward.hpp:276-304 loops over the batch), so every rank owns whole
  pairs and there is no collective on the data path (weak scaling in
  bench.py).
* Barycenter (barycenter.hpp:60-86): the objective is a weighted SUM over
  members, so members are sharded contiguously and the per-rank partial
  objective and grad_z are summed by one allreduce (the engine's NCCL
  allreduce over NVLink on GPUs, sdtw_allreduce_grad_f32), after which every
  rank applies the identical Adam step (barycenter.hpp:181-191).

The functions here are backend-agnostic (``objective`` and ``allreduce``
are callables) so the same code runs with the CUDA engine + NCCL in
bench.py and with the CPU oracle + gloo in tests/test_sharding_cpu.py.
"""
from __future__ import annotations


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [lo, hi) share of n items for `rank` of `world` (sizes
    differ by at most one; every item owned exactly once)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return rank * n // world, (rank + 1) * n // world


def sharded_barycenter_objective(objective, allreduce, z, members, weights, world, rank):
    """Partial objective over this rank's members, summed across ranks.

    objective(z, members_shard, weights_shard) -> (value, grad)
    allreduce(value, grad) -> (value_sum, grad_sum)
    """
    lo, hi = shard_range(len(members), world, rank)
    w = None if weights is None else weights[lo:hi]
    value, grad = objective(z, members[lo:hi], w)
    if world > 1:
        value, grad = allreduce(value, grad)
    return value, grad
