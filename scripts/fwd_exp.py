# Forward phase time of the current build (SDTW_LIB selects a variant).
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import CONFIGS
from paper_2602_17206_b200 import Engine
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
eng = Engine(0)
torch.manual_seed(0)
B, L, D = cfg["B"], cfg["L"], cfg["D"]
x = torch.randn((B, L, D), device="cuda"); y = torch.randn((B, L, D), device="cuda")
eng.enable_timing(True)
ts = []
for it in range(4):
    eng.forward_backward_E(x, y, cfg["gamma"]) if False else eng.sdtw_with_gradients(x, y, cfg["gamma"])
    torch.cuda.synchronize()
    ts.append(eng.phase_times()["forward"])
print(os.environ.get("SDTW_LIB", "main"), sys.argv[1], "forward ms", [round(v, 3) for v in ts[1:]])
