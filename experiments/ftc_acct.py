# Cycle accounting of the fused forward DP warps (trace mode), one config.
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2602_17206_b200 import Engine
B, N, M, D = (int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (32, 4096, 4096, 128)))
eng = Engine(0)
torch.manual_seed(0)
S = (N + 31) // 32
x = torch.randn((B, N, D), device="cuda"); y = torch.randn((B, M, D), device="cuda")
tr = torch.zeros(140 * B * S, dtype=torch.int64, device="cuda")  # forward and backward trace slots
eng.enable_timing(True)
for it in range(3):
    if it == 2:
        eng.lib.sdtw_debug_set_trace(eng.ctx, tr.data_ptr())
    tr.zero_()
    eng.sdtw_with_gradients(x, y, 0.1, fused=True)
    torch.cuda.synchronize()
    if it == 1:
        ph = eng.phase_times()
eng.lib.sdtw_debug_set_trace(eng.ctx, None)
cy = tr[24 * B * S:32 * B * S].cpu().numpy().reshape(B, S, 8)[..., :5].astype(np.float64)
steps = M + 31
names = ["tile-wait", "epilogue", "halo-wait", "backpressure", "steps"]
med = np.median(cy.reshape(-1, 5), axis=0) / steps
print(os.environ.get("SDTW_LIB", "main"), f"B={B} N={N} M={M}", "phases(untraced)", {k: round(v, 3) for k, v in ph.items()})
print("   cycles/step:", dict(zip(names, [round(float(v), 1) for v in med])), "sum", round(float(med.sum()), 1))
for w in range(4):
    mw = np.median(cy[:, w::4].reshape(-1, 5), axis=0) / steps
    print("   strip%%4 == %d:" % w, dict(zip(names, [round(float(v), 1) for v in mw])))
