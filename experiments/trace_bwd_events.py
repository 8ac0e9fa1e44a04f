# Backward event log (trace mode): per strip (time, chunk, kind) records.
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import CONFIGS
from paper_2602_17206_b200 import Engine
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
fused = len(sys.argv) > 2 and sys.argv[2] == "fused"
B, L, D = cfg["B"], cfg["L"], cfg["D"]
S = (L + 31) // 32
eng = Engine(0)
from bench import bench_inputs
xh, yh = bench_inputs(B, L, D, 42)
x, y = torch.from_numpy(xh).cuda(), torch.from_numpy(yh).cuda()
tr = torch.zeros(140 * B * S, dtype=torch.int64, device="cuda")
for it in range(2):
    eng.lib.sdtw_debug_set_trace(eng.ctx, tr.data_ptr() if it == 1 else None)
    tr.zero_()
    eng.sdtw_with_gradients(x, y, cfg["gamma"], fused=fused)
    torch.cuda.synchronize()
eng.lib.sdtw_debug_set_trace(eng.ctx, None)
t = tr.cpu().numpy()
evs = t[40 * B * S:88 * B * S].reshape(B, S, 16, 3)
t0 = evs[..., 0][evs[..., 0] > 0].min()
names = {1: "R+", 2: "R-", 3: "E+", 4: "E-", 5: "X", 6: "S", 7: "V"}
b = 0
mid = int(sys.argv[3]) if len(sys.argv) > 3 else S - 1
for s in range(mid, max(-1, mid - 8), -1):
    line = []
    for k in range(16):
        tm, ch, kd = evs[b, s, k]
        if tm == 0:
            break
        line.append(f"{names[int(kd)]}{int(ch)}@{(tm - t0) / 1e3:.1f}")
    print(f"strip {s:3d}: " + " ".join(line))
    hl = []
    hev = t[88 * B * S:136 * B * S].reshape(B, S, 16, 3)
    for k in range(16):
        tm, ch, kd = hev[b, s, k]
        if tm == 0:
            break
        hl.append(f"{names[int(kd)]}{int(ch)}@{(tm - t0) / 1e3:.1f}")
    print(f"   helper: " + " ".join(hl))
