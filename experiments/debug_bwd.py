import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_2602_17206_b200 import Engine
eng = Engine(0); o = oracle.OracleC()
for (N, M, g) in [(64, 64, 1.0), (33, 64, 1.0), (64, 33, 1.0), (64, 70, 0.05), (65, 70, 0.05), (96, 64, 1.0), (64, 96, 1.0), (40, 100, 1.0)]:
    rng = np.random.default_rng(N * 7 + M)
    x = rng.uniform(-1, 1, (1, N, 3)); y = rng.uniform(-1, 1, (1, M, 3))
    rc, loss, R = o.forward(x, y, g)
    rc, Eref = o.backward(R, o.costs(x, y), g)
    l2, E = eng.forward_backward_E(x, y, g, dtype=np.float64)
    err = np.abs(E - Eref)[0, 1:-1, 1:-1]
    bad = np.argwhere(err > 1e-9)
    print(N, M, g, "maxerr", err.max(), "nbad", len(bad), "first bad (i,j 0-based)", bad[:3].tolist(), "tiles", sorted(set((int(a)//32, int(b)//32) for a, b in bad))[:10])
