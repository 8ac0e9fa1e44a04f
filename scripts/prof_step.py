"""One engine step for profiling: python experiments/prof_step.py c2 unfused [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import CONFIGS  # noqa: E402
from paper_2602_17206_b200 import Engine  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
fused = (sys.argv[2] if len(sys.argv) > 2 else "unfused") == "fused"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
eng = Engine(0)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
eng.set_stream(s.cuda_stream)
B, L, D = cfg["B"], cfg["L"], cfg["D"]
g = torch.Generator(device="cuda").manual_seed(42)
x = torch.randn((B, L, D), generator=g, device="cuda")
y = torch.randn((B, L, D), generator=g, device="cuda")
outs = (torch.empty(B, device="cuda"), torch.empty((B, L, D), device="cuda"), torch.empty((B, L, D), device="cuda"))
eng.enable_timing(True)
for _ in range(reps):
    eng.sdtw_with_gradients(x, y, cfg["gamma"], fused=fused, out=outs)
    print(eng.phase_times())
torch.cuda.synchronize()
