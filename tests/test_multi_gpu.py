"""Multi-GPU paths of SURVEY.md §8(e), exercised on the one GPU a test box
has: several engine contexts on device 0 stand in for the per-device
contexts of a multi-GPU host (pairs are independent, so shards never wait on
one another), and the NCCL path runs as a one-rank communicator
(ncclCommInitAll over the contexts' distinct devices).

* sharded fwd+bwd (sdtw_fwd_bwd_multi_*) == one context, bit for bit,
  fp32 / fp64, both cost modes, ragged shards (B not a multiple of G);
* the barycenter over G devices (member shards + NCCL allreduce of grad_z
  and the objective) on G = 1 equals the single-context objective bit for
  bit and executes the NCCL allreduce.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def engines3():
    from paper_2602_17206_b200 import Engine
    engs = [Engine(0) for _ in range(3)]
    yield engs
    for e in engs:
        e.close()


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_sharded_equals_single_bitwise(engine, engines3, fused, dtype):
    from paper_2602_17206_b200.capi import sdtw_with_gradients_multi
    rng = np.random.default_rng(12)
    B, N, M, D = 7, 150, 137, 64
    x = rng.standard_normal((B, N, D)).astype(dtype)
    y = rng.standard_normal((B, M, D)).astype(dtype)
    x[3] *= 40.0  # a pair of its own scale: shards must not share operand scales
    one = engine.sdtw_with_gradients(x, y, 0.1, fused=fused, dtype=dtype)
    for G in (2, 3):
        many = sdtw_with_gradients_multi(engines3[:G], x, y, 0.1, fused=fused, dtype=dtype)
        for u, v in zip(one, many):
            assert np.array_equal(u, v), G


def test_sharded_more_shards_than_pairs(engines3):
    from paper_2602_17206_b200.capi import sdtw_with_gradients_multi
    rng = np.random.default_rng(4)
    x = rng.standard_normal((2, 40, 8)).astype(np.float32)
    y = rng.standard_normal((2, 33, 8)).astype(np.float32)
    a = sdtw_with_gradients_multi(engines3[:1], x, y, 1.0)
    b = sdtw_with_gradients_multi(engines3, x, y, 1.0)  # one shard is empty
    for u, v in zip(a, b):
        assert np.array_equal(u, v)


def test_sharded_validation(engines3):
    from paper_2602_17206_b200 import ValidationError
    from paper_2602_17206_b200.capi import sdtw_with_gradients_multi
    x = np.zeros((2, 4, 2), np.float32)
    with pytest.raises(ValidationError):
        sdtw_with_gradients_multi(engines3[:2], x, x, 0.0)


def test_barycenter_multi_nccl_one_rank(engine):
    """NCCL path (ncclCommInitAll + grouped ncclAllReduce) with one rank:
    the allreduce is the identity, so the result equals the single-context
    objective bit for bit."""
    from paper_2602_17206_b200 import Engine
    from paper_2602_17206_b200.capi import barycenter_objective_multi, nccl_init_all
    rng = np.random.default_rng(8)
    members = rng.standard_normal((16, 96, 8)).astype(np.float32)
    z = members.mean(axis=0).astype(np.float32)
    w = rng.uniform(0.5, 2.0, 16)
    e = Engine(0)
    try:
        nccl_init_all([e])
        v1, g1 = engine.barycenter_objective(z, members, 1.0, weights=w)
        vm, gm = barycenter_objective_multi([e], z, members, 1.0, weights=w)
        assert vm == v1
        assert np.array_equal(gm, g1)
    finally:
        e.close()


def test_nccl_init_all_rejects_duplicate_devices(engines3):
    from paper_2602_17206_b200 import SdtwError
    from paper_2602_17206_b200.capi import nccl_init_all
    with pytest.raises(SdtwError):
        nccl_init_all(engines3[:2])  # both on device 0


def test_sharded_fused_band_cache(engine, engines3):
    """Fused shards at a length where the band cache is on (each context keeps
    its own band and band counters): bitwise equal to one context."""
    from paper_2602_17206_b200.capi import sdtw_with_gradients_multi
    rng = np.random.default_rng(21)
    t = np.linspace(0, 6, 1100)[None, :, None]
    x = (np.sin(t * np.arange(1, 33)) + 0.2 * rng.standard_normal((5, 1100, 32))).astype(np.float32)
    y = (np.cos(t * np.arange(1, 33)) + 0.2 * rng.standard_normal((5, 1100, 32))).astype(np.float32)
    one = engine.sdtw_with_gradients(x, y, 0.05, fused=True)
    b0 = [e.band_stats()[0] for e in engines3[:2]]
    many = sdtw_with_gradients_multi(engines3[:2], x, y, 0.05, fused=True)
    assert all(e.band_stats()[0] > c for e, c in zip(engines3[:2], b0))
    for u, v in zip(one, many):
        assert np.array_equal(u, v)
