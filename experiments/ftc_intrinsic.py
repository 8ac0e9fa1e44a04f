# Intrinsic step time of the fused tensor-core forward: few strips, long rows.
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2602_17206_b200 import Engine
eng = Engine(0)
for (B, N, M, D) in [(1, 32, 16384, 128), (1, 64, 16384, 128), (1, 128, 16384, 128), (2, 128, 16384, 128),
                     (148, 128, 8192, 128), (296, 128, 8192, 128), (296, 256, 4096, 128)]:
    S = (N + 31) // 32
    x = torch.randn((B, N, D), device="cuda"); y = torch.randn((B, M, D), device="cuda")
    tr = torch.zeros(32 * B * S, dtype=torch.int64, device="cuda")
    eng.lib.sdtw_debug_set_trace(eng.ctx, tr.data_ptr())
    for _ in range(2):
        tr.zero_()
        eng.sdtw_with_gradients(x, y, 0.1, fused=True)
        torch.cuda.synchronize()
    t = tr[16 * B * S:20 * B * S].cpu().numpy().reshape(B, S, 4).astype(np.float64)
    first, mid, end = t[..., 1], t[..., 2], t[..., 3]
    C = (M + 31) // 32
    steps2 = (M + 31) - 32 * (C // 2)
    rate = (end - mid) / steps2
    rate1 = (mid - first) / (32 * (C // 2) - 32)
    print(f"B={B} N={N} M={M}: ns/step 2nd half by strip {np.round(np.median(rate, axis=0)[:8], 1)}"
          f" 1st half {np.round(np.median(rate1, axis=0)[:8], 1)}  (cycles {np.median(rate) * 1.965:.0f})")
eng.lib.sdtw_debug_set_trace(eng.ctx, None)
# cycle accounting of the first strips (trace mode)
for (B, N, M, D) in [(1, 128, 16384, 128), (32, 1024, 1024, 128), (32, 4096, 4096, 128)]:
    S = (N + 31) // 32
    x = torch.randn((B, N, D), device="cuda"); y = torch.randn((B, M, D), device="cuda")
    tr = torch.zeros(32 * B * S, dtype=torch.int64, device="cuda")
    eng.lib.sdtw_debug_set_trace(eng.ctx, tr.data_ptr())
    for _ in range(2):
        tr.zero_()
        eng.sdtw_with_gradients(x, y, 0.1, fused=True)
        torch.cuda.synchronize()
    cy = tr[24 * B * S:32 * B * S].cpu().numpy().reshape(B, S, 8)[..., :5].astype(np.float64)
    steps = M + 31
    names = ["tile-wait", "epilogue", "halo-wait", "backpressure", "steps"]
    med = np.median(cy.reshape(-1, 5), axis=0) / steps
    print(f"B={B} N={N} M={M} cycles/step (median strip):", dict(zip(names, np.round(med, 1))), "sum", round(float(med.sum()), 1))
    for w in range(min(4, S)):
        m = np.median(cy[:, w, :], axis=0) / steps
        print("   strip", w, dict(zip(names, np.round(m, 1))))
    eng.lib.sdtw_debug_set_trace(eng.ctx, None)
