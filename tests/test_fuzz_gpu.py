"""Randomised shapes against the fp64 oracle (oracle/sdtw_oracle.c): N, M
from 1 to 140 (single rows and columns, ragged last strips and chunks,
N != M both ways), D from 1 to 9, gamma from 1e-2 to 10, Sakoe-Chiba bands
at and above |N - M|, both cost modes, fp64 (1e-11 / 1e-9) and fp32 (the
parity tolerances), and fused == unfused bit for bit in fp32 (tensor-core
costs in both)."""
import numpy as np
import pytest

from tests.tolerances import F32_LOSS, F64_GRAD, F64_LOSS, f32_grad_max, rel_err

pytestmark = pytest.mark.gpu


def _cases(n, seed):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        B = int(rng.integers(1, 4))
        N = int(rng.choice([1, 2, 31, 32, 33, int(rng.integers(1, 141))]))
        M = int(rng.choice([1, 2, 31, 32, 33, int(rng.integers(1, 141))]))
        D = int(rng.integers(1, 10))
        gamma = float(10 ** rng.uniform(-2, 1))
        bw = 0
        if rng.random() < 0.3 and min(N, M) > 1:
            bw = abs(N - M) + int(rng.integers(0, 12))
        out.append((B, N, M, D, gamma, bw, int(rng.integers(1 << 30))))
    return out


@pytest.mark.parametrize("case", _cases(80, 2026))
def test_fuzz_vs_oracle(engine, oracle_c, case):
    B, N, M, D, gamma, bw, seed = case
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1, 1, (B, N, D))
    y = rng.uniform(-1, 1, (B, M, D))
    rc, rl, rgx, rgy = oracle_c.sdtw_with_gradients(x, y, gamma, bw)
    assert rc == 0
    for fused in (False, True):
        l, gx, gy = engine.sdtw_with_gradients(x, y, gamma, bandwidth=bw, fused=fused, dtype=np.float64)
        assert rel_err(l, rl).max() <= F64_LOSS, (case, fused)
        assert rel_err(gx, rgx).max() <= F64_GRAD and rel_err(gy, rgy).max() <= F64_GRAD, (case, fused)
    xf, yf = x.astype(np.float32), y.astype(np.float32)
    u = engine.sdtw_with_gradients(xf, yf, gamma, bandwidth=bw)
    f = engine.sdtw_with_gradients(xf, yf, gamma, bandwidth=bw, fused=True)
    for a, b in zip(u, f):
        assert np.array_equal(a, b), case
    assert rel_err(u[0], rl).max() <= F32_LOSS, case
    gm = max(rel_err(u[1], rgx).max(), rel_err(u[2], rgy).max())
    assert gm <= f32_grad_max(gamma), (case, gm)
