# One long strip through the fused forward (for ncu): B=1, N, M from argv.
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_17206_b200 import Engine
N = int(sys.argv[1]) if len(sys.argv) > 1 else 32
M = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
eng = Engine(0)
x = torch.randn((B, N, 128), device="cuda"); y = torch.randn((B, M, 128), device="cuda")
for _ in range(2):
    eng.sdtw_with_gradients(x, y, 0.1, fused=True)
torch.cuda.synchronize()
print("ok")
