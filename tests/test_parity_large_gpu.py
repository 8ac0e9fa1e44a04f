"""GPU parity at the sizes BASELINE.json names (VERDICT r1 "next" item 1).

* C3 (B=32, L=4096, D=128, gamma=0.01, the "log-space backward stability"
  config): the full batch runs on the engine in both cost modes; pairs are
  independent (forward.hpp:72-79), so two pairs sliced out of the full-B
  reference-generator tensors are checked against the reference's T=double
  path, and the sliced pairs' results must equal the full-batch results bit
  for bit (per-pair operand scales: a pair's result never depends on its
  batch-mates).
* gamma = 1e-3 at L = 4096.
* The fp32 stability witness (test_backward.cpp:286-321,
  acceptance.cpp:96-134) with its gradients against fp64, and the
  witness's linear half on the engine's standalone fp32 table path.
* A K=64, L=512, D=64 fp32 barycenter objective with its gradient.
"""
import os

import numpy as np
import pytest

from tests.tolerances import (F32_GRAD_MAX, F32_GRAD_P99, F32_LOSS, F64_GRAD, F64_LOSS, f32_grad_max,
                              f64_grad_tol,
                              grad_stats, rel_err)

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _check(loss, gx, gy, rl, rgx, rgy, tag, gamma=1.0):
    lr = rel_err(loss, rl).max()
    st = [grad_stats(a, r) for a, r in ((gx, rgx), (gy, rgy))]
    print(f"[parity] {tag}: loss {lr:.2e} grad max/p99 {st}")
    assert lr <= F32_LOSS, (tag, loss, rl)
    for mx, p99 in st:
        assert mx <= f32_grad_max(gamma) and p99 <= F32_GRAD_P99, (tag, mx, p99)


@pytest.fixture(scope="module")
def c3_inputs(reference):
    # the reference bench generator (bench.hpp:61-66): all of x, then all of y
    return reference.bench_inputs(32, 4096, 128)


@pytest.mark.parametrize("fused", [False, True])
def test_c3_vs_reference(engine, reference, c3_inputs, fused):
    x, y = c3_inputs
    loss, gx, gy = engine.sdtw_with_gradients(x, y, 0.01, fused=fused)
    assert np.isfinite(loss).all() and np.isfinite(gx).all() and np.isfinite(gy).all()
    pairs = [0, 31]
    xs, ys = np.ascontiguousarray(x[pairs]), np.ascontiguousarray(y[pairs])
    rc, rl, rgx, rgy = reference.sdtw_with_gradients(xs.astype(np.float64), ys.astype(np.float64), 0.01)
    assert rc == 0
    _check(loss[pairs], gx[pairs], gy[pairs], rl, rgx, rgy, f"c3 fused={fused}", 0.01)
    # batch independence: the 2-pair call reproduces the full batch's bits
    l2, gx2, gy2 = engine.sdtw_with_gradients(xs, ys, 0.01, fused=fused)
    assert np.array_equal(l2, loss[pairs])
    assert np.array_equal(gx2, gx[pairs]) and np.array_equal(gy2, gy[pairs])


def test_c3_fused_equals_unfused(engine, c3_inputs):
    x, y = c3_inputs
    x, y = np.ascontiguousarray(x[:4]), np.ascontiguousarray(y[:4])
    a = engine.sdtw_with_gradients(x, y, 0.01)
    b = engine.sdtw_with_gradients(x, y, 0.01, fused=True)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)


@pytest.mark.parametrize("fused", [False, True])
def test_gamma_1e3_L4096(engine, reference, fused):
    rng = np.random.default_rng(4096)
    x = rng.standard_normal((1, 4096, 64)).astype(np.float32)
    y = rng.standard_normal((1, 4096, 64)).astype(np.float32)
    rc, rl, rgx, rgy = reference.sdtw_with_gradients(x.astype(np.float64), y.astype(np.float64), 1e-3)
    assert rc == 0
    loss, gx, gy = engine.sdtw_with_gradients(x, y, 1e-3, fused=fused)
    _check(loss, gx, gy, rl, rgx, rgy, f"gamma=1e-3 L=4096 fused={fused}", 1e-3)


@pytest.fixture(scope="module")
def witness():
    return dict(np.load(os.path.join(ROOT, "tests", "golden", "witness.npz")))


@pytest.mark.parametrize("fused", [False, True])
def test_witness_gradients(engine, witness, fused):
    """The witness through the log-space engine: loss and gradients against
    the reference's T=double result (the fp32 reference itself is off by
    ~100% here), E(1,1) against fp64."""
    w = witness
    loss, gx, gy = engine.sdtw_with_gradients(w["x"], w["y"], float(w["gamma"]), fused=fused)
    _check(loss, gx, gy, w["loss"], w["grad_x"], w["grad_y"], f"witness fused={fused}", float(w["gamma"]))
    _, E = engine.forward_backward_E(w["x"], w["y"], float(w["gamma"]), fused=fused)
    assert np.isfinite(E).all()
    assert abs(E[0, 1, 1] - float(w["E11"])) <= 1e-5
    assert np.abs(E[0, 1:-1, 1:-1].sum(axis=1) - w["E_rowsum"]).max() <= 1e-3


def test_witness_f64(engine, witness):
    w = witness
    loss, gx, gy = engine.sdtw_with_gradients(w["x"].astype(np.float64), w["y"].astype(np.float64),
                                              float(w["gamma"]), dtype=np.float64)
    assert rel_err(loss, w["loss"]).max() <= F64_LOSS
    tol = f64_grad_tol(float(w["loss"][0]), float(w["gamma"]))
    assert rel_err(gx, w["grad_x"]).max() <= tol
    assert rel_err(gy, w["grad_y"]).max() <= tol


def test_witness_linear_half_fp32_tables(engine, witness):
    """test_backward.cpp:305-320: on the fp32 R table, backward_linear
    overflows (>= 1 non-finite cell) while backward_log stays finite."""
    w = witness
    g = float(w["gamma"])
    loss, R, d, _ = engine.forward(w["x"], w["y"], g, table=True, costs=True, dtype=np.float32)
    El = engine.backward_table(R, g, costs=d, linear=True, dtype=np.float32)
    Eg = engine.backward_table(R, g, costs=d, dtype=np.float32)
    inner = (slice(None), slice(1, -1), slice(1, -1))
    assert (~np.isfinite(El[inner])).sum() > 0
    assert np.isfinite(Eg[inner]).all()


def test_barycenter_k64_f32(engine, reference):
    """barycenter_objective (barycenter.hpp:60-86), K=64 members, L=512,
    D=64, gamma=1: value and gradient of the fp32 engine vs the reference's
    T=double objective."""
    rng = np.random.default_rng(64)
    members = rng.standard_normal((64, 512, 64)).astype(np.float32)
    z = members.mean(axis=0).astype(np.float32)
    rc, rv, rg = reference.barycenter_objective(z.astype(np.float64), members.astype(np.float64), 1.0)
    assert rc == 0
    v, g = engine.barycenter_objective(z, members, 1.0)
    assert abs(v - rv) <= F32_LOSS * max(1.0, abs(rv)), (v, rv)
    mx, p99 = grad_stats(g, rg)
    assert mx <= F32_GRAD_MAX and p99 <= F32_GRAD_P99, (mx, p99)


@pytest.mark.parametrize("fused", [False, True])
def test_batch_independence_bitwise(engine, fused):
    """Pairs of very different magnitudes in one batch: every pair's fp32
    result equals the result of calling it alone, bit for bit."""
    rng = np.random.default_rng(5)
    B, L, D = 5, 300, 128
    x = rng.standard_normal((B, L, D)).astype(np.float32)
    y = rng.standard_normal((B, L, D)).astype(np.float32)
    scale = np.array([1.0, 300.0, 1e-3, 7.0, 0.5], np.float32)[:, None, None]
    x *= scale
    y *= scale
    loss, gx, gy = engine.sdtw_with_gradients(x, y, 0.1, fused=fused)
    for b in range(B):
        l1, gx1, gy1 = engine.sdtw_with_gradients(x[b:b + 1], y[b:b + 1], 0.1, fused=fused)
        assert l1[0] == loss[b], b
        assert np.array_equal(gx1[0], gx[b]) and np.array_equal(gy1[0], gy[b]), b


def test_arena_shape_sequence_f64(engine, oracle_c):
    """The tagged-halo arena is shared by calls of different shapes and
    dtypes on one context: big -> small -> medium fp64 calls interleaved
    with fp32 ones still match the oracle (stale status / fp32 words must
    never pass for the current call's fp64 tags)."""
    rng = np.random.default_rng(9)
    shapes = [(4, 300, 280), (1, 40, 33), (2, 130, 150), (3, 64, 64), (2, 200, 190)]
    for k, (B, N, M) in enumerate(shapes):
        x = rng.uniform(-1, 1, (B, N, 3)); y = rng.uniform(-1, 1, (B, M, 3))
        rc, rl, rgx, rgy = oracle_c.sdtw_with_gradients(x, y, 0.3)
        assert rc == 0
        loss, gx, gy = engine.sdtw_with_gradients(x, y, 0.3, dtype=np.float64)
        assert rel_err(loss, rl).max() <= F64_LOSS, k
        assert rel_err(gx, rgx).max() <= F64_GRAD and rel_err(gy, rgy).max() <= F64_GRAD, k
        engine.sdtw_with_gradients(x.astype(np.float32), y.astype(np.float32), 0.3)
