import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from tests.conftest import ROOT
from tests.tolerances import rel_err, grad_stats
from paper_2602_17206_b200 import Engine
d = np.load(os.path.join(ROOT, "tests", "golden", "sdtw_small.npz"))
eng = Engine(0)
for k in range(int(d["n_cases"])):
    x, y = d[f"c{k}_x"], d[f"c{k}_y"]; g = float(d[f"c{k}_gamma"]); bw = int(d[f"c{k}_bandwidth"])
    for dt in (np.float32, np.float64):
        loss, gx, gy = eng.sdtw_with_gradients(x.astype(dt), y.astype(dt), g, bw, dtype=dt)
        l2, E = eng.forward_backward_E(x.astype(dt), y.astype(dt), g, bw, dtype=dt)
        eerr = np.abs(E - d[f"c{k}_E"]).max()
        print(k, x.shape, y.shape, g, bw, dt.__name__, "loss", rel_err(loss, d[f"c{k}_loss"]).max(), "gx", grad_stats(gx, d[f"c{k}_grad_x"])[0], "gy", grad_stats(gy, d[f"c{k}_grad_y"])[0], "E", eerr)
