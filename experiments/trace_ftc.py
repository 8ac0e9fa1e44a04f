# Strip timeline of the fused tensor-core forward (sdtw_fused.cuh trace slots).
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import CONFIGS
from paper_2602_17206_b200 import Engine
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
B, L, D = cfg["B"], cfg["L"], cfg["D"]
S = (L + 31) // 32
C = S
eng = Engine(0)
from bench import bench_inputs
xh, yh = bench_inputs(B, L, D, 42)
x, y = torch.from_numpy(xh).cuda(), torch.from_numpy(yh).cuda()
tr = torch.zeros(140 * B * S, dtype=torch.int64, device="cuda")  # forward and backward trace slots
eng.lib.sdtw_debug_set_trace(eng.ctx, tr.data_ptr())
for _ in range(2):
    tr.zero_()
    eng.sdtw_with_gradients(x, y, cfg["gamma"], fused=True)
    torch.cuda.synchronize()
t = tr[16 * B * S:20 * B * S].cpu().numpy().reshape(B, S, 4).astype(np.float64)
t0 = t[:, :, 0][t[:, :, 0] > 0].min()
t = (t - t0) / 1e3
tick, first, mid, end = t[..., 0], t[..., 1], t[..., 2], t[..., 3]
steps2 = (L + 31) - 32 * (C // 2)
rate = (end - mid) / steps2 * 1e3  # ns / step, second half
rate1 = (mid - first) / (32 * (C // 2) - 32) * 1e3
print(cfg)
print("ns/step second half: by strip%%4:", [round(float(np.median(rate[:, w::4])), 1) for w in range(4)],
      " strip0:", round(float(np.median(rate[:, 0])), 1))
print("ns/step first half:  by strip%%4:", [round(float(np.median(rate1[:, w::4])), 1) for w in range(4)],
      " strip0:", round(float(np.median(rate1[:, 0])), 1))
lag = np.diff(first, axis=1)  # first-32-columns-done gap between consecutive strips
print("lag (us) strip s-1 -> s by s%%4:", [round(float(np.median(lag[:, (w - 1)::4])), 2) for w in range(1, 5)])
print("ticket->first: median %.1f us" % np.median(first - tick))
print("pair 0 first:", np.round(first[0, :12], 1))
print("pair 0 end:  ", np.round(end[0, :12], 1))
print("total span us %.1f" % end.max())
# how busy the slots are over time: strips in flight (ticket .. end) per 100 us
span = end.max()
for q in np.arange(0, span, span / 12):
    print("t=%7.1f us  strips in flight %5d" % (q, int(((tick <= q) & (end > q)).sum())))
