# Phase times of the current build (SDTW_LIB selects a variant).
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import CONFIGS
from paper_2602_17206_b200 import Engine
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
fused = len(sys.argv) > 2 and sys.argv[2] == "fused"
eng = Engine(0)
torch.manual_seed(0)
B, L, D = cfg["B"], cfg["L"], cfg["D"]
x = torch.randn((B, L, D), device="cuda"); y = torch.randn((B, L, D), device="cuda")
eng.enable_timing(True)
acc = {}
for it in range(5):
    eng.sdtw_with_gradients(x, y, cfg["gamma"], fused=fused)
    torch.cuda.synchronize()
    if it >= 1:
        for k, v in eng.phase_times().items():
            acc[k] = acc.get(k, 0.0) + v / 4
print(os.path.basename(os.environ.get("SDTW_LIB", "main")), sys.argv[1], "fused" if fused else "unfused",
      {k: round(v, 3) for k, v in acc.items()}, "total", round(sum(acc.values()), 3))
