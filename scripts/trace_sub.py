# Sub-group timeline of pair 0's first strips in forward6 (trace mode).
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import CONFIGS
from paper_2602_17206_b200 import Engine
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
B, L, D = cfg["B"], cfg["L"], cfg["D"]
S = (L + 31) // 32
eng = Engine(0)
x = torch.randn((B, L, D), device="cuda"); y = torch.randn((B, L, D), device="cuda")
n = max(140 * B * S, 4 * B * S + 2 * 16384 + 16)
tr = torch.zeros(n, dtype=torch.int64, device="cuda")
eng.lib.sdtw_debug_set_trace(eng.ctx, tr.data_ptr())
for _ in range(2):
    tr.zero_()
    eng.sdtw_with_gradients(x, y, cfg["gamma"])
o = 4 * B * S
st = tr[o:o + 16384].cpu().numpy().reshape(16, 1024).astype(np.float64)
ca = tr[o + 16384:o + 32768].cpu().numpy().reshape(16, 1024).astype(np.float64)
t0 = st[0, 0]
ng = (L + 31 + 31) // 32 * 4
for s in range(4):
    a = (st[s, :ng] - t0) / 1e3; c = (ca[s, :ng] - t0) / 1e3
    dur = np.diff(a)
    wait = c - a
    print(f"strip {s}: start {a[0]:.2f} us, sub-group period median {np.median(dur)*1e3:.0f} ns, halo wait median {np.median(wait)*1e3:.0f} ns mean {wait.mean()*1e3:.0f} ns")
for s in range(1, 4):
    # lag in sub-groups: when strip s starts sub-group j vs when strip s-1 started sub-group j
    lag = (st[s, :ng] - st[s - 1, :ng]) / 1e3
    print(f"strip {s} lag behind strip {s-1}: median {np.median(lag):.2f} us, at j=10 {lag[10]:.2f}, j=60 {lag[60]:.2f}, j=120 {lag[min(120, ng-1)]:.2f}")
print("timeline strip0/strip1 sub-groups 40..48 (us):")
print(np.round((st[0, 40:48] - t0) / 1e3, 2)); print(np.round((st[1, 40:48] - t0) / 1e3, 2)); print(np.round((ca[1, 40:48] - t0) / 1e3, 2))
