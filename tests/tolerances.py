"""Parity tolerances, metric rel = |a - r| / max(1, |r|)
(acceptance.cpp:45-48, gradcheck.hpp:110-111), against the reference's
T=double path on identical (fp32-representable) inputs."""
import numpy as np

# fp32 engine
F32_LOSS = 1e-5
F32_GRAD_MAX = 1e-3
F32_GRAD_P99 = 5e-5       # fp32 cost rounding at gamma=1: 1.4e-5 measured
F32_E_ABS = 1e-4          # alignment-gradient table entries, absolute


def f64_grad_tol(loss: float, gamma: float) -> float:
    """fp64 gradient bound: the reference's own log-space backward evaluates
    (R_s - R_self - d) / gamma on R ~ |loss|, so its weights carry ~eps64 |R|
    / gamma of rounding (the witness: |R| = 1e5, gamma = 1e-3 -> 2e-8); the
    engine's edge-difference form does not, and the two differ by that
    much.  Bound: max(F64_GRAD, 10 eps64 |loss| / gamma)."""
    return max(F64_GRAD, 10 * 2.220446049250313e-16 * abs(loss) / gamma)


def f32_grad_max(gamma: float) -> float:
    """Max-element gradient bound for the fp32 engine at small gamma.

    The DP's edge differences and costs are O(cost) ~ 2 D and carry fp32
    rounding of ~ulp(2 D) ~ 3e-5 absolute; the softmin weights see it divided
    by gamma.  Where two alignment branches nearly tie, that shifts
    probability mass between them and moves the gradient of the few rows /
    columns at the tie by ~ulp/gamma relative (measured at C3, gamma = 0.01:
    5e-3 on 2 rows of 8192, p99 1.4e-7).  The bound is therefore
    max(1e-3, 6e-5 / gamma); the p99 bound (F32_GRAD_P99) does not scale."""
    return max(F32_GRAD_MAX, 6e-5 / gamma)
# fp64 engine (the reference's unit tests use 1e-10..1e-12)
F64_LOSS = 1e-11
F64_GRAD = 1e-9
F64_E_ABS = 1e-10


def rel_err(a, r):
    a = np.asarray(a, np.float64)
    r = np.asarray(r, np.float64)
    return np.abs(a - r) / np.maximum(1.0, np.abs(r))


def grad_stats(a, r):
    e = rel_err(a, r).ravel()
    if e.size == 0:
        return 0.0, 0.0
    return float(e.max()), float(np.quantile(e, 0.99))
