# Timeline (CUPTI via torch.profiler) of one host-pointer call: copies and
# kernels per stream, to check copy/compute overlap.
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import CONFIGS
from paper_2602_17206_b200 import Engine
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
B, L, D, g = cfg["B"], cfg["L"], cfg["D"], cfg["gamma"]
x = torch.randn(B, L, D); y = torch.randn(B, L, D)
xh = x.pin_memory(); yh = y.pin_memory()
lh = torch.empty(B).pin_memory(); gxh = torch.empty(B, L, D).pin_memory(); gyh = torch.empty(B, L, D).pin_memory()
eng = Engine(0)
for _ in range(2):
    eng.sdtw_with_gradients(xh, yh, g, out=(lh, gxh, gyh))
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    eng.sdtw_with_gradients(xh, yh, g, out=(lh, gxh, gyh))
    torch.cuda.synchronize()
prof.export_chrome_trace("/tmp/tl.json")
ev = [e for e in json.load(open("/tmp/tl.json"))["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
t0 = min(e["ts"] for e in ev)
rows = sorted(ev, key=lambda e: e["ts"])
for e in rows:
    if e["dur"] < 5 and e.get("cat") != "gpu_memcpy":
        continue
    print(f'{(e["ts"] - t0) / 1e3:8.3f} {e["dur"] / 1e3:7.3f} ms  s{e.get("args", {}).get("stream", "?")}  {e["name"][:70]}')
print("span ms", (max(e["ts"] + e["dur"] for e in ev) - t0) / 1e3)
