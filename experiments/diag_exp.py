import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_2602_17206_b200 import capi
from tests.tolerances import grad_stats
variant = sys.argv[1]
path = {"0": capi.LIB_PATH, "1": "experiments/libsdtw_exp1.so", "2": "experiments/libsdtw_exp2.so"}[variant]
capi.load_library(path)
eng = capi.Engine(0)
ref = oracle.Reference()
for (L, D, g) in [(256, 128, 1.0), (256, 128, 0.01), (1024, 128, 0.1)]:
    B = 2 if L < 1000 else 1
    rng = np.random.default_rng(42)
    x = rng.standard_normal((B, L, D)).astype(np.float32)
    y = rng.standard_normal((B, L, D)).astype(np.float32)
    rc, rl, rgx, rgy = ref.sdtw_with_gradients(x.astype(np.float64), y.astype(np.float64), g)
    l, gx, gy = eng.sdtw_with_gradients(x, y, g)
    print(variant, L, D, g, "gx", grad_stats(gx, rgx), "gy", grad_stats(gy, rgy))
