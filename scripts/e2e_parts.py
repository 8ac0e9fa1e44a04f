# Components of the e2e call at C2: PCIe copies, per-chunk device time.
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_17206_b200 import Engine
B, L, D, g = 32, 1024, 128, 0.1
x = torch.randn(B, L, D, device="cuda"); y = torch.randn(B, L, D, device="cuda")
xh = x.cpu().pin_memory(); yh = y.cpu().pin_memory()
def tm(f, n=5):
    f(); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); [f() for _ in range(n)]; e.record(); e.synchronize()
    return s.elapsed_time(e) / n
xd = torch.empty_like(x)
print("H2D 16.8 MB ms", tm(lambda: xd.copy_(xh, non_blocking=True)))
print("D2H 16.8 MB ms", tm(lambda: xh.copy_(xd, non_blocking=True)))
eng = Engine(0)
for b in (8, 16, 32):
    outs = (torch.empty(b, device="cuda"), torch.empty(b, L, D, device="cuda"), torch.empty(b, L, D, device="cuda"))
    eng.set_stream(torch.cuda.current_stream().cuda_stream)
    print(f"device fwd+bwd B={b} ms", tm(lambda: eng.sdtw_with_gradients(x[:b], y[:b], g, out=outs)))
lh = torch.empty(B).pin_memory(); gxh = torch.empty(B, L, D).pin_memory(); gyh = torch.empty(B, L, D).pin_memory()
for n in ("1", "2", "4"):
    os.environ["SDTW_E2E_CHUNKS"] = n
    t = tm(lambda: eng.sdtw_with_gradients(xh, yh, g, out=(lh, gxh, gyh)))
    print("host call chunks", n, "ms", t)
