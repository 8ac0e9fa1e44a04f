import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2602_17206_b200 import Engine
eng = Engine(0)
dt = np.float64 if (len(sys.argv) > 1 and sys.argv[1] == "f64") else np.float32
rng = np.random.default_rng(1)
x = rng.uniform(-1, 1, (1, 64, 3)).astype(dt); y = rng.uniform(-1, 1, (1, 64, 3)).astype(dt)
loss, E = eng.forward_backward_E(x, y, 1.0, dtype=dt)
print("ok", loss)
