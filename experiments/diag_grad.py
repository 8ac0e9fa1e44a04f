import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_2602_17206_b200 import Engine
from tests.tolerances import rel_err, grad_stats

eng = Engine(0)
ref = oracle.Reference()
L, D, g = 256, 128, 1.0
rng = np.random.default_rng(42)
x = rng.standard_normal((2, L, D)).astype(np.float32)
y = rng.standard_normal((2, L, D)).astype(np.float32)
x64, y64 = x.astype(np.float64), y.astype(np.float64)
rc, rl, R, d, E = ref.tables(x64, y64, g)
rc, rl2, rgx, rgy = ref.sdtw_with_gradients(x64, y64, g)
loss, E32 = eng.forward_backward_E(x, y, g)
err = np.abs(E32.astype(np.float64) - E)
relE = err / np.maximum(E, 1e-30)
print("E abs max", err.max(), "E rel (E>1e-6) max", relE[E > 1e-6].max(), "median", np.median(relE[E > 1e-6]))
print("rowsum ref", E.sum(axis=2).max(), "mass per antidiag check")
# gradient from the reference E in f32 via our contraction
gx, gy = eng.input_gradients(E.astype(np.float32), x, y, dtype=np.float32)
print("contraction-only f32 gx", grad_stats(gx, rgx), "gy", grad_stats(gy, rgy))
gx, gy = eng.input_gradients(E32, x, y, dtype=np.float32)
print("engine E f32 gx", grad_stats(gx, rgx))
gx, gy = eng.input_gradients(E32.astype(np.float64), x64, y64, dtype=np.float64)
print("engine E, f64 contraction gx", grad_stats(gx, rgx))
l, gx, gy = eng.sdtw_with_gradients(x, y, g)
print("e2e f32", grad_stats(gx, rgx), grad_stats(gy, rgy))
l, gx, gy = eng.sdtw_with_gradients(x64, y64, g, dtype=np.float64)
print("e2e f64", grad_stats(gx, rgx), grad_stats(gy, rgy))
# numpy f32 contraction in a different formulation: sum_j E_ij (x_i - y_j)
E32n = E.astype(np.float32)[:, 1:-1, 1:-1]
gx2 = 2 * np.einsum('bij,bijk->bik', E32n, (x[:, :, None, :] - y[:, None, :, :]))
print("numpy f32 (x-y) form", grad_stats(gx2, rgx))
print("grad magnitude max", np.abs(rgx).max(), "rowsum max", E32n.sum(2).max())
