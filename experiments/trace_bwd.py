import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import CONFIGS
from paper_2602_17206_b200 import Engine
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
B, L, D = cfg["B"], cfg["L"], cfg["D"]
S = (L + 31) // 32
eng = Engine(0)
g = torch.Generator(device="cuda").manual_seed(42)
x = torch.randn((B, L, D), device="cuda", generator=g); y = torch.randn((B, L, D), device="cuda", generator=g)
tr = torch.zeros(40 * B * S, dtype=torch.int64, device="cuda")
eng.lib.sdtw_debug_set_trace(eng.ctx, tr.data_ptr())
for _ in range(2):
    tr.zero_()
    eng.sdtw_with_gradients(x, y, cfg["gamma"])
t = tr.cpu().numpy().astype(np.float64)
fw = t[:2 * B * S].reshape(B, S, 2); bw = t[2 * B * S:4 * B * S].reshape(B, S, 2); nt = t[4 * B * S:5 * B * S].reshape(B, S)
t0 = bw[:, :, 0][bw[:, :, 0] > 0].min()
st = (bw[:, :, 0] - t0) / 1e3; en = (bw[:, :, 1] - t0) / 1e3
print("bwd span us %.1f" % en.max())
print("strip durations us: min %.1f median %.1f max %.1f" % ((en - st).min(), np.median(en - st), (en - st).max()))
print("pair0 strip start (bottom first):", np.round(st[0, ::-1][:8], 1))
print("pair0 strip end (bottom first):", np.round(en[0, ::-1][:8], 1), "...", np.round(en[0, ::-1][-4:], 1))
print("live tiles per strip (pair 0, bottom first):", nt[0, ::-1][:16].astype(int))
print("mean live tiles per strip", nt.mean())
evs = t[5 * B * S:13 * B * S].reshape(B, S, 8)
def rel(e):
    v = evs[:, :, e]
    return np.where(v > 0, (v - bw[:, :, 0]) / 1e3, np.nan)
names = ["hint_seen", "specR_done", "final_seen", "tile1_start", "tile1_Rdone", "tile2_start", "tile2_Rdone"]
for e, nm in enumerate(names):
    r = rel(e)
    print("%-12s median since strip start: %8.1f us (n=%d)" % (nm, np.nanmedian(r), np.sum(~np.isnan(r))))
print("strip duration median %.1f" % np.median((bw[:, :, 1] - bw[:, :, 0]) / 1e3))
