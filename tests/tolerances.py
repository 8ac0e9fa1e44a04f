"""Parity tolerances, metric rel = |a - r| / max(1, |r|)
(acceptance.cpp:45-48, gradcheck.hpp:110-111), against the reference's
T=double path on identical (fp32-representable) inputs."""
import numpy as np

# fp32 engine
F32_LOSS = 1e-5
F32_GRAD_MAX = 1e-3
F32_GRAD_P99 = 5e-5       # fp32 cost rounding at gamma=1: 1.4e-5 measured
F32_E_ABS = 1e-4          # alignment-gradient table entries, absolute
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
