"""GPU parity: the CUDA engine (through the C-ABI) against the reference.

Inputs are fp32-representable; the reference runs in T=double (SURVEY.md
§8(c)).  Tolerances live in tests/tolerances.py and are stated per check.
"""
import numpy as np
import pytest

from tests.tolerances import (F32_E_ABS, F32_GRAD_MAX, F32_GRAD_P99, F32_LOSS, F64_E_ABS,
                              F64_GRAD, F64_LOSS, grad_stats, rel_err)

pytestmark = pytest.mark.gpu


def _f32(a):
    return np.ascontiguousarray(a, np.float32)


@pytest.mark.parametrize("fused", [False, True])
def test_golden_f32(engine, golden, fused):
    for c in golden:
        loss, gx, gy = engine.sdtw_with_gradients(_f32(c["x"]), _f32(c["y"]), c["gamma"],
                                                  c["bandwidth"], fused=fused)
        assert rel_err(loss, c["loss"]).max() <= F32_LOSS, (c["x"].shape, loss, c["loss"])
        mx, p99 = grad_stats(gx, c["grad_x"])
        assert mx <= F32_GRAD_MAX and p99 <= F32_GRAD_P99, (c["x"].shape, mx, p99)
        mx, p99 = grad_stats(gy, c["grad_y"])
        assert mx <= F32_GRAD_MAX and p99 <= F32_GRAD_P99, (c["y"].shape, mx, p99)


@pytest.mark.parametrize("fused", [False, True])
def test_golden_f64(engine, golden, fused):
    for c in golden:
        loss, gx, gy = engine.sdtw_with_gradients(c["x"], c["y"], c["gamma"], c["bandwidth"],
                                                  fused=fused, dtype=np.float64)
        assert rel_err(loss, c["loss"]).max() <= F64_LOSS, (c["x"].shape, loss - c["loss"])
        assert rel_err(gx, c["grad_x"]).max() <= F64_GRAD
        assert rel_err(gy, c["grad_y"]).max() <= F64_GRAD


@pytest.mark.parametrize("dtype,tol", [(np.float32, F32_E_ABS), (np.float64, F64_E_ABS)])
def test_golden_E_table(engine, golden, dtype, tol):
    for c in golden:
        loss, E = engine.forward_backward_E(c["x"].astype(dtype), c["y"].astype(dtype), c["gamma"],
                                            c["bandwidth"], dtype=dtype)
        assert E.shape == c["E"].shape
        assert np.abs(E - c["E"]).max() <= tol, (c["x"].shape, np.abs(E - c["E"]).max())


def test_kats(engine):
    # forward 1x1 -> 9 (test_forward.cpp:33-41); backward 1x1: E=1, grads -6/+6
    x = np.array([[[2.0]]]); y = np.array([[[5.0]]])
    loss, gx, gy = engine.sdtw_with_gradients(x, y, 1.0, dtype=np.float64)
    assert loss[0] == 9.0 and abs(gx[0, 0, 0] + 6) < 1e-12 and abs(gy[0, 0, 0] - 6) < 1e-12
    loss, E = engine.forward_backward_E(x, y, 1.0, dtype=np.float64)
    assert E[0, 1, 1] == 1.0
    # worked example (test_forward.cpp:43-57)
    x = np.array([[[0.0], [1.0]]])
    loss, _, _ = engine.sdtw_with_gradients(x, x, 1.0, dtype=np.float64, grads=False)
    assert abs(loss[0] + np.log(1.0 + 2.0 * np.exp(-1.0))) < 1e-12


def _bench_like(B, L, D, seed=42):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((B, L, D)).astype(np.float32),
            rng.standard_normal((B, L, D)).astype(np.float32))


@pytest.mark.parametrize("L,D,gamma", [(256, 128, 1.0), (256, 128, 0.01), (256, 128, 1e-3),
                                       (300, 16, 0.1), (256, 1024, 1.0)])
@pytest.mark.parametrize("fused", [False, True])
def test_vs_reference_f32(engine, reference, L, D, gamma, fused):
    B = 2
    x, y = _bench_like(B, L, D)
    rc, rl, rgx, rgy = reference.sdtw_with_gradients(x.astype(np.float64), y.astype(np.float64), gamma)
    assert rc == 0
    loss, gx, gy = engine.sdtw_with_gradients(x, y, gamma, fused=fused)
    assert rel_err(loss, rl).max() <= F32_LOSS
    for a, r in ((gx, rgx), (gy, rgy)):
        mx, p99 = grad_stats(a, r)
        assert mx <= F32_GRAD_MAX and p99 <= F32_GRAD_P99, (mx, p99)


@pytest.mark.slow
def test_c2_slice_vs_reference(engine, reference):
    """C2 shape (L=1024, D=128, gamma=0.1) on a pair slice (pairs are
    independent)."""
    x, y = _bench_like(1, 1024, 128, seed=7)
    rc, rl, rgx, rgy = reference.sdtw_with_gradients(x.astype(np.float64), y.astype(np.float64), 0.1)
    assert rc == 0
    for fused in (False, True):
        loss, gx, gy = engine.sdtw_with_gradients(x, y, 0.1, fused=fused)
        assert rel_err(loss, rl).max() <= F32_LOSS
        for a, r in ((gx, rgx), (gy, rgy)):
            mx, p99 = grad_stats(a, r)
            assert mx <= F32_GRAD_MAX and p99 <= F32_GRAD_P99, (mx, p99)


@pytest.mark.parametrize("N,M,bw", [(1, 1, 0), (1, 37, 0), (45, 1, 0), (33, 64, 0), (64, 33, 0),
                                    (31, 97, 0), (100, 100, 5), (70, 90, 25), (129, 130, 1),
                                    (257, 200, 60)])
def test_ragged_and_band_f64(engine, oracle_c, N, M, bw):
    rng = np.random.default_rng(N * 1000 + M)
    x = rng.uniform(-1, 1, (2, N, 3)); y = rng.uniform(-1, 1, (2, M, 3))
    rc, rl, rgx, rgy = oracle_c.sdtw_with_gradients(x, y, 0.7, bw)
    assert rc == 0
    for fused in (False, True):
        loss, gx, gy = engine.sdtw_with_gradients(x, y, 0.7, bw, fused=fused, dtype=np.float64)
        assert rel_err(loss, rl).max() <= F64_LOSS
        assert rel_err(gx, rgx).max() <= F64_GRAD
        assert rel_err(gy, rgy).max() <= F64_GRAD


def test_fused_equals_unfused_bitwise(engine):
    """test_backward.cpp:225-241 / test_forward.cpp:82-101: one cost routine
    for both modes (fp64 path)."""
    x, y = _bench_like(3, 75, 9, seed=3)
    x, y = x.astype(np.float64), y.astype(np.float64)
    a = engine.sdtw_with_gradients(x, y, 0.3, dtype=np.float64)
    b = engine.sdtw_with_gradients(x, y, 0.3, fused=True, dtype=np.float64)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)


@pytest.mark.parametrize("B,N,M,D,gamma,bw", [
    (3, 75, 75, 16, 0.3, 0),      # ragged strips and chunks, D padded to 64
    (2, 300, 170, 128, 0.1, 0),   # N > M tail, 3 super-strips, partial last one
    (2, 130, 333, 100, 1.0, 0),   # M > N tail, D not a multiple of 16
    (4, 256, 256, 64, 0.05, 40),  # Sakoe-Chiba band
    (1, 33, 1, 8, 1.0, 0),        # single column
    (1, 1, 40, 8, 1.0, 0),        # single row
])
def test_fused_tc_equals_unfused_bitwise_f32(engine, B, N, M, D, gamma, bw):
    """fp32 fused mode (tcgen05 costs inside the DP kernels) reproduces the
    unfused mode (tcgen05 cost tensor) bit for bit: same operand split, same
    MMA sequence, same epilogue (test_backward.cpp:225-241 analogue)."""
    rng = np.random.default_rng(B * 1000 + N + M + D)
    x = rng.standard_normal((B, N, D)).astype(np.float32)
    y = rng.standard_normal((B, M, D)).astype(np.float32)
    a = engine.sdtw_with_gradients(x, y, gamma, bandwidth=bw)
    b = engine.sdtw_with_gradients(x, y, gamma, bandwidth=bw, fused=True)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)


def test_deterministic(engine):
    """acceptance.cpp:348-377 analogue: repeated runs are bit-identical."""
    x, y = _bench_like(4, 130, 16, seed=5)
    a = engine.sdtw_with_gradients(x, y, 0.5)
    for _ in range(3):
        b = engine.sdtw_with_gradients(x, y, 0.5)
        for u, v in zip(a, b):
            assert np.array_equal(u, v)


def test_E_properties_small_gamma(engine):
    """E in [0,1], E(1,1)=1, E(N,M)=1 at gamma = 1e-3, L = 512 (the fp32
    reference's own E(1,1) collapses here)."""
    x, y = _bench_like(2, 512, 32, seed=11)
    loss, E = engine.forward_backward_E(x, y, 1e-3)
    inner = E[:, 1:-1, 1:-1]
    assert np.isfinite(inner).all()
    assert (inner >= 0).all() and (inner <= 1).all()
    assert np.allclose(E[:, 1, 1], 1.0, atol=1e-5)
    assert (E[:, -2, -2] == 1.0).all()


def test_stability_witness_log(engine):
    """acceptance.cpp:96-134 witness (L=2048, D=2, gamma=1e-3): the log-space
    route is finite AND correct (E(1,1) = 1), unlike the fp32 reference."""
    rng = np.random.default_rng(1)
    L = 2048
    x = (2.0 * rng.uniform(0, 1, (1, L, 2))).astype(np.float32)
    y = (7.0 - 2.0 * rng.uniform(0, 1, (1, L, 2))).astype(np.float32)
    loss, E = engine.forward_backward_E(x, y, 1e-3)
    assert np.isfinite(E).all()
    assert abs(E[0, 1, 1] - 1.0) < 1e-5


def test_validation_errors(engine):
    from paper_2602_17206_b200 import ValidationError
    x = np.zeros((1, 4, 2), np.float32)
    with pytest.raises(ValidationError):
        engine.sdtw_with_gradients(x, x, 0.0)
    with pytest.raises(ValidationError):
        engine.sdtw_with_gradients(x, np.zeros((1, 9, 2), np.float32), 1.0, bandwidth=2)
    with pytest.raises(ValidationError):
        engine.sdtw_with_gradients(x, np.zeros((1, 4, 3), np.float32), 1.0)


def test_mem_limit_oom(engine):
    from paper_2602_17206_b200 import OutOfMemoryError
    x, y = _bench_like(1, 64, 4)
    engine.set_mem_limit(1024)
    try:
        with pytest.raises(OutOfMemoryError) as ei:
            engine.sdtw_with_gradients(x, y, 1.0)
        assert ei.value.requested_bytes > 0
    finally:
        engine.set_mem_limit(0)
    engine.sdtw_with_gradients(x, y, 1.0)


@pytest.mark.parametrize("B,L,D", [(32, 512, 64), (8, 512, 256), (4, 384, 1024)])
def test_fused_uses_less_memory(engine, B, L, D):
    """acceptance criterion 6 analogue: fused peak below unfused by at least
    the B x N x M cost tensor, at every D (D > 128: SIMT costs in the DP
    kernels, still no cost tensor)."""
    x, y = _bench_like(B, L, D)
    engine.trim()
    peaks = {}
    for fused in (False, True):
        engine.reset_peak()
        engine.sdtw_with_gradients(x, y, 1.0, fused=fused)
        peaks[fused] = engine.mem_stats()[1]
    assert peaks[False] - peaks[True] >= 4 * B * L * L, (peaks, 4 * B * L * L)


def test_barycenter_objective_golden(engine, bary_golden):
    b = bary_golden
    v, g = engine.barycenter_objective(b["z"], b["members"], 1.0, dtype=np.float64)
    assert abs(v - float(b["value"])) <= 1e-10 * max(1.0, abs(float(b["value"])))
    assert rel_err(g, b["grad"]).max() <= F64_GRAD
    v, g = engine.barycenter_objective(b["z"], b["members"], 1.0, weights=b["weights"],
                                       dtype=np.float64)
    assert abs(v - float(b["value_w"])) <= 1e-10 * max(1.0, abs(float(b["value_w"])))
    assert rel_err(g, b["grad_w"]).max() <= F64_GRAD
    v32, g32 = engine.barycenter_objective(b["z"].astype(np.float32),
                                           b["members"].astype(np.float32), 1.0)
    assert abs(v32 - float(b["value"])) <= 1e-5 * max(1.0, abs(float(b["value"])))
    mx, p99 = grad_stats(g32, b["grad"])
    assert mx <= F32_GRAD_MAX and p99 <= F32_GRAD_P99, (mx, p99)


def test_adam_matches_oracle(engine):
    import oracle
    rng = np.random.default_rng(3)
    n = 1000
    z = rng.standard_normal(n); g = rng.standard_normal(n)
    m1 = np.zeros(n); m2 = np.zeros(n)
    zr, m1r, m2r = z.copy(), m1.copy(), m2.copy()
    o = oracle.OracleC()
    for t in (1, 2, 3):
        engine.adam_step(z, g, m1, m2, t, dtype=np.float64)
        o.lib.oracle_adam_step(zr.ctypes.data, g.ctypes.data, m1r.ctypes.data, m2r.ctypes.data, n, t,
                               0.01, 0.9, 0.999, 1e-8)
    assert np.allclose(z, zr, rtol=0, atol=1e-14)


def test_table_api_matches_reference(engine, golden):
    """forward -> padded R table -> backward_log / backward_linear on that
    table (CS3), in fp64."""
    for c in golden:
        loss, R, d, _ = engine.forward(c["x"], c["y"], c["gamma"], c["bandwidth"], table=True,
                                       costs=True)
        assert np.abs(d - c["costs"]).max() <= 1e-12
        fin = np.isfinite(c["R"])
        assert (np.isfinite(R) == fin).all()
        assert rel_err(R[fin], c["R"][fin]).max() <= 1e-12
        E = engine.backward_table(c["R"], c["gamma"], c["bandwidth"], costs=c["costs"])
        assert np.abs(E - c["E"]).max() <= 1e-12
        El = engine.backward_table(c["R"], c["gamma"], c["bandwidth"], costs=c["costs"], linear=True)
        assert np.abs(El - c["E_linear"]).max() <= 1e-12
        gx, gy = engine.input_gradients(c["E"], c["x"], c["y"])
        assert rel_err(gx, c["grad_x"]).max() <= 1e-12
        assert rel_err(gy, c["grad_y"]).max() <= 1e-12


def test_tile_store_overflow_path(engine, oracle_c, monkeypatch):
    """A tile quota of 1 per strip sends the other non-zero tiles
    through the backward's in-warp fixed-point contraction; gradients still
    match the fp64 oracle and are deterministic."""
    x, y = _bench_like(2, 200, 24, seed=21)
    _, rl, rgx, rgy = oracle_c.sdtw_with_gradients(x.astype(np.float64), y.astype(np.float64), 1.0)
    ref = (rl, rgx, rgy)
    monkeypatch.setenv("SDTW_DEBUG_TILE_QUOTA", "1")
    a = engine.sdtw_with_gradients(x, y, 1.0)
    b = engine.sdtw_with_gradients(x, y, 1.0)
    monkeypatch.delenv("SDTW_DEBUG_TILE_QUOTA")
    for u, v in zip(a, b):
        assert np.array_equal(u, v)
    assert rel_err(a[0], ref[0]).max() <= F32_LOSS
    for g, r in zip(a[1:], ref[1:]):
        assert grad_stats(g, r)[0] <= F32_GRAD_MAX


@pytest.mark.parametrize("fused", [False, True])
def test_forward_normalized(engine, oracle_c, fused):
    """forward_normalized (forward.hpp:85-102): sdtw(x,y) - (sdtw(x,x) + sdtw(y,y)) / 2,
    exactly 0 when x == y."""
    rng = np.random.default_rng(77)
    x = rng.uniform(-1, 1, (3, 40, 5)); y = rng.uniform(-1, 1, (3, 40, 5))
    ref = []
    for a_, b_ in ((x, y), (x, x), (y, y)):
        ref.append(oracle_c.sdtw_with_gradients(a_, b_, 0.5)[1])
    want = ref[0] - (ref[1] + ref[2]) / 2
    got = engine.forward(x, y, 0.5, fused=fused, dtype=np.float64, normalized=True)[0]
    assert rel_err(got, want).max() <= F64_LOSS
    same = engine.forward(x, x, 0.5, fused=fused, dtype=np.float64, normalized=True)[0]
    assert np.abs(same).max() <= 1e-9
    with pytest.raises(Exception):
        engine.forward(x, y[:, :30], 0.5, dtype=np.float64, normalized=True)


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_host_call_pair_chunks(engine, oracle_c, monkeypatch, fused, dtype):
    """Host-pointer calls split the pairs over sub-context streams so copies
    overlap compute (sdtw_capi.cu e2e_chunks): the chunked call (ragged
    chunks: 5 pairs over 3 streams) matches the one-stream call and the fp64
    oracle, and repeated chunked calls are bit-identical."""
    x, y = _bench_like(5, 150, 24, seed=33)
    x, y = np.ascontiguousarray(x[:, :137], dtype), np.ascontiguousarray(y, dtype)
    _, rl, rgx, rgy = oracle_c.sdtw_with_gradients(x.astype(np.float64), y.astype(np.float64), 0.1)
    monkeypatch.setenv("SDTW_E2E_CHUNKS", "1")
    one = engine.sdtw_with_gradients(x, y, 0.1, fused=fused, dtype=dtype)
    monkeypatch.setenv("SDTW_E2E_CHUNKS", "3")
    a = engine.sdtw_with_gradients(x, y, 0.1, fused=fused, dtype=dtype)
    b = engine.sdtw_with_gradients(x, y, 0.1, fused=fused, dtype=dtype)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)
    lt, gt = (F32_LOSS, F32_GRAD_MAX) if dtype == np.float32 else (F64_LOSS, F64_GRAD)
    # per-pair operand scales: a chunk of pairs computes exactly what the
    # whole batch computes for those pairs
    for u, v in zip(a, one):
        assert np.array_equal(u, v)
    assert rel_err(a[0], rl).max() <= lt
    for g, r in zip(a[1:], (rgx, rgy)):
        assert grad_stats(g, r)[0] <= gt
