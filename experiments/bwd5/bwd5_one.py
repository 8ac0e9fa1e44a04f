"""One backward call on a given shape with a short spin limit; prints the
timed-out waits.  python scripts/bwd5_one.py B N M D gamma"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SITES = {1: "lock", 2: "slot-outstanding", 3: "queue-full", 4: "helper-idle", 5: "ring-free", 6: "producer-ring",
         7: "wait-below", 8: "tile-ready", 10: "helper-jobseq"}


def main():
    from paper_2602_17206_b200 import Engine
    from paper_2602_17206_b200.capi import load_library
    lib = load_library()
    eng = Engine(0)
    B, N, M, D = (int(v) for v in sys.argv[1:5])
    g = float(sys.argv[5])
    rng = np.random.default_rng(1)
    x = rng.standard_normal((B, N, D)).astype(np.float32)
    y = rng.standard_normal((B, M, D)).astype(np.float32)
    reps = int(sys.argv[6]) if len(sys.argv) > 6 else 1
    dev = len(sys.argv) > 7 and sys.argv[7] == "dev"
    try:
        if dev:
            import torch
            x, y = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        import time
        for r in range(reps):
            t0 = time.time()
            eng.sdtw_with_gradients(x, y, g)
            rec = (C.c_int * 260)()
            n = lib.sdtw_debug_waits(0, rec, 260)
            print("ok", r, f"{time.time() - t0:.3f}s waits={n}", flush=True)
    except Exception as e:
        rec = (C.c_int * 260)()
        n = lib.sdtw_debug_waits(0, rec, 260)
        rs = [(SITES.get(rec[4 + 4 * k], rec[4 + 4 * k]), rec[5 + 4 * k], rec[6 + 4 * k], rec[7 + 4 * k])
              for k in range(min(n, 40))]
        print(f"FAIL {e}; waits={n}", flush=True)
        for r in rs:
            print("  ", r, flush=True)


if __name__ == "__main__":
    main()
