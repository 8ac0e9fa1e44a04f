# Cycle accounting of the backward DP warps (trace mode).
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
xh, yh = bench_inputs(B, L, D, 42)  # the reference generator (bench.py's inputs)
x, y = torch.from_numpy(xh).cuda(), torch.from_numpy(yh).cuda()
tr = torch.zeros(40 * B * S, dtype=torch.int64, device="cuda")
eng.enable_timing(True)
for it in range(3):
    if it == 2:
        eng.lib.sdtw_debug_set_trace(eng.ctx, tr.data_ptr())
    tr.zero_()
    eng.sdtw_with_gradients(x, y, cfg["gamma"], fused=fused)
    torch.cuda.synchronize()
    if it == 1:
        ph = eng.phase_times()
eng.lib.sdtw_debug_set_trace(eng.ctx, None)
t = tr.cpu().numpy().astype(np.float64)
cy = t[32 * B * S:40 * B * S].reshape(B, S, 8)
nt = t[4 * B * S:5 * B * S].reshape(B, S)
names = ["recompute", "S-wait", "E-steps", "status-wait", "tile-epilogue", "other", "tc-stage+epi", "tc-mma"]
print(sys.argv[1], "fused" if fused else "unfused", {k: round(v, 3) for k, v in ph.items()})
med = np.median(cy.reshape(-1, 8), axis=0)
print("  per strip (median, kcycles):", dict(zip(names, [round(float(v) / 1e3, 1) for v in med])),
      "live tiles/strip %.2f" % nt.mean())
tot = cy.sum(axis=(0, 1))
print("  totals share:", dict(zip(names, [round(float(v / tot.sum()), 3) for v in tot])))
bot = cy[:, -1, :]
print("  bottom strip (no S wait) kcycles:", dict(zip(names, [round(float(v) / 1e3, 1) for v in np.median(bot, axis=0)])),
      "tiles", np.median(nt[:, -1]))
