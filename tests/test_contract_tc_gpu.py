"""The input-gradient contraction on tcgen05 (sdtw_grad_tc.cuh) against the
ordered FMA kernel (sdtw_grad.cuh) and the fp64 oracle: dX and dY buckets
(strip slots, chunk lists), ragged shapes, features not a multiple of 8 or of
128, N != M, band, the capped tile store (fixed-point overflow path), and
D > 128 (several feature blocks).  SDTW_CONTRACT_SIMT=0 / =1 force either
kernel (backward() reads it per call)."""
import os

import numpy as np
import pytest

from tests.tolerances import F64_LOSS, rel_err

pytestmark = pytest.mark.gpu


def _with(env, fn):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("B,N,M,D,gamma,bw", [(3, 300, 257, 128, 0.1, 0), (2, 190, 230, 100, 1.0, 0),
                                             (2, 128, 160, 37, 0.5, 0), (2, 200, 200, 96, 0.3, 40),
                                             (1, 96, 64, 300, 1.0, 0)])
def test_tc_matches_fma_and_oracle(engine, oracle_c, B, N, M, D, gamma, bw):
    rng = np.random.default_rng(N * 7 + D)
    x = rng.standard_normal((B, N, D)).astype(np.float32)
    y = rng.standard_normal((B, M, D)).astype(np.float32)
    for fused in (False, True):
        tc = _with({"SDTW_CONTRACT_SIMT": "0"},
                   lambda: engine.sdtw_with_gradients(x, y, gamma, bandwidth=bw, fused=fused))
        fma = _with({"SDTW_CONTRACT_SIMT": "1"},
                    lambda: engine.sdtw_with_gradients(x, y, gamma, bandwidth=bw, fused=fused))
        assert np.array_equal(tc[0], fma[0])  # the loss does not go through the contraction
        for a, r in zip(tc[1:], fma[1:]):
            assert rel_err(a, r).max() <= 1e-5, (fused, rel_err(a, r).max())
    rc, rl, rgx, rgy = oracle_c.sdtw_with_gradients(x.astype(np.float64), y.astype(np.float64), gamma, bw)
    assert rc == 0
    assert rel_err(tc[0], rl).max() <= 1e-5
    # the DP's own fp32 parity is pinned elsewhere (test_parity_*); here the
    # gradients only have to stay the engine's: p99 at the fp32 bar, max
    # within the near-tie allowance of N(0,1) data at small gamma (measured
    # 1.2e-3 at gamma = 0.1 with the FMA kernel as well)
    for a, r in ((tc[1], rgx), (tc[2], rgy)):
        e = rel_err(a, r)
        assert e.max() <= 5e-3 and np.quantile(e, 0.99) <= 5e-5


def test_tc_overflow_store(engine):
    """A capped tile store: tiles past the quota go to the backward's
    fixed-point path and are added after the tensor-core contraction."""
    rng = np.random.default_rng(11)
    x = rng.standard_normal((2, 256, 128)).astype(np.float32)
    y = rng.standard_normal((2, 256, 128)).astype(np.float32)
    full = _with({"SDTW_CONTRACT_SIMT": "0"}, lambda: engine.sdtw_with_gradients(x, y, 1.0))
    capped = _with({"SDTW_CONTRACT_SIMT": "0", "SDTW_DEBUG_TILE_QUOTA": "1"},
                   lambda: engine.sdtw_with_gradients(x, y, 1.0))
    for a, r in zip(capped[1:], full[1:]):
        assert rel_err(a, r).max() <= 1e-5


def test_tc_deterministic_and_batch_independent(engine):
    rng = np.random.default_rng(5)
    x = rng.standard_normal((4, 333, 128)).astype(np.float32) * np.array([1, 50, 1e-2, 3], np.float32)[:, None, None]
    y = rng.standard_normal((4, 301, 128)).astype(np.float32) * np.array([1, 50, 1e-2, 3], np.float32)[:, None, None]
    a = engine.sdtw_with_gradients(x, y, 0.2)
    b = engine.sdtw_with_gradients(x, y, 0.2)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)
    for k in range(4):
        one = engine.sdtw_with_gradients(x[k:k + 1], y[k:k + 1], 0.2)
        assert np.array_equal(one[1][0], a[1][k]) and np.array_equal(one[2][0], a[2][k])
