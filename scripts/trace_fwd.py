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
tr = torch.zeros(140 * B * S, dtype=torch.int64, device="cuda")
eng.lib.sdtw_debug_set_trace(eng.ctx, tr.data_ptr())
for _ in range(2):
    tr.zero_()
    eng.sdtw_with_gradients(x, y, cfg["gamma"])
t = tr[:2 * B * S].cpu().numpy().reshape(B, S, 2).astype(np.float64)
t0 = t[:, :, 0][t[:, :, 0] > 0].min()
st = (t[:, :, 0] - t0) / 1e3; en = (t[:, :, 1] - t0) / 1e3
dur = en - st
print("strip durations us: min %.1f median %.1f max %.1f" % (dur.min(), np.median(dur), dur.max()))
print("pair 0 starts:", np.round(st[0, :8], 1), "... ends:", np.round(en[0, -4:], 1))
print("start gap between consecutive strips (pair 0) median %.2f us" % np.median(np.diff(st[0])))
print("end gap between consecutive strips (pair 0) median %.2f us" % np.median(np.diff(en[0])))
print("total span us %.1f" % en.max())
steps = L + 31
print("strip0 us/step %.3f" % (dur[:, 0].mean() / steps))
