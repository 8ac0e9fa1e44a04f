# Per-strip start/end trace of the slot forward (sdtw_forward5 / forward_tc):
# slot_strip_forward writes [16 B S + 4 (b S + s) + e], e = 0 start, 3 end.
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
x = torch.randn((B, L, D), device="cuda"); y = torch.randn((B, L, D), device="cuda")
tr = torch.zeros(140 * B * S, dtype=torch.int64, device="cuda")
eng.lib.sdtw_debug_set_trace(eng.ctx, tr.data_ptr())
for _ in range(2):
    tr.zero_()
    eng.sdtw_with_gradients(x, y, cfg["gamma"], fused=fused)
t = tr[16 * B * S:20 * B * S].cpu().numpy().reshape(B, S, 4).astype(np.float64)
t0 = t[:, :, 0][t[:, :, 0] > 0].min()
st = (t[:, :, 0] - t0) / 1e3; en = (t[:, :, 3] - t0) / 1e3
dur = en - st
print("strip durations us: min %.1f median %.1f max %.1f" % (dur.min(), np.median(dur), dur.max()))
eg = np.diff(en, axis=1)
print("end gap between consecutive strips: median %.2f us, mean %.2f us" % (np.median(eg), eg.mean()))
W = int(os.environ.get("SDTW_FWD5_W", "8")) if not fused else 4
if S > W:
    intra = eg[:, [i for i in range(S - 1) if (i + 1) % W != 0]]
    inter = eg[:, [i for i in range(S - 1) if (i + 1) % W == 0]]
    print("  intra-slot hop median %.2f us, inter-slot (L2) hop median %.2f us" % (np.median(intra), np.median(inter)))
print("total span us %.1f" % en.max())
print("strip0 us/step %.4f" % (dur[:, 0].mean() / (L + 31)))
cy = tr[24 * B * S:32 * B * S].cpu().numpy().reshape(B, S, 8)[:, :, :5].astype(np.float64) / (L + 31)
names = ["cost wait", "epilogue", "halo wait", "back-pressure", "steps"]
print("cycles/step, mean over strips:", {n: round(v, 1) for n, v in zip(names, cy.reshape(-1, 5).mean(0))})
print("cycles/step, strip 0:", {n: round(v, 1) for n, v in zip(names, cy[:, 0].mean(0))})
for w in range(min(S, 8)):
    print("  strip", w, {n: round(v, 1) for n, v in zip(names, cy[:, w].mean(0))})
