"""One process: parity spot checks + C1/C2/C3 phase timing + counters for the
pair-pipeline backward.  Prints one line per item, flushes as it goes."""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    t0 = time.time()
    import torch
    import bench
    import oracle
    from paper_2602_17206_b200 import Engine
    from paper_2602_17206_b200.capi import load_library
    from tests.tolerances import grad_stats, rel_err
    lib = load_library()
    eng = Engine(0)
    print(f"[setup] {time.time() - t0:.1f}s", flush=True)
    o = oracle.OracleC()
    rng = np.random.default_rng(3)
    for (B, N, M, D, g) in [(2, 256, 256, 128, 1.0), (2, 130, 333, 100, 1.0), (3, 300, 170, 16, 0.1),
                            (1, 64, 64, 8, 0.01), (2, 500, 480, 32, 0.1)]:
        x = rng.standard_normal((B, N, D)).astype(np.float32)
        y = rng.standard_normal((B, M, D)).astype(np.float32)
        try:
            l, gx, gy = eng.sdtw_with_gradients(x, y, g)
            rc, rl, rgx, rgy = o.sdtw_with_gradients(x.astype(np.float64), y.astype(np.float64), g)
            print(f"[parity] {B}x{N}x{M} D={D} g={g}: loss {rel_err(l, rl).max():.2e} gx {grad_stats(gx, rgx)} "
                  f"gy {grad_stats(gy, rgy)}", flush=True)
        except Exception as e:
            print(f"[parity] {B}x{N}x{M} D={D} g={g}: ERROR {e}", flush=True)
    side = torch.cuda.Stream()
    torch.cuda.set_stream(side)
    eng.set_stream(side.cuda_stream)
    for cfg_name in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["c2", "c3", "c1"]):
        cfg = bench.CONFIGS[cfg_name]
        B, L, D, g = cfg["B"], cfg["L"], cfg["D"], cfg["gamma"]
        xh, yh = bench.bench_inputs(B, L, D, 42)
        x, y = torch.from_numpy(xh).cuda(), torch.from_numpy(yh).cuda()
        outs = (torch.empty(B, device="cuda"), torch.empty((B, L, D), device="cuda"),
                torch.empty((B, L, D), device="cuda"))
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        try:
            tot, ph, _, _ = bench.time_engine(eng, torch, x, y, outs, False, g, 5, 3, flush)
            eng.sdtw_with_gradients(x, y, g, out=outs)  # synchronous: surfaces timeouts
            S = (L + 31) // 32
            tr = torch.zeros(128 * B * S, dtype=torch.int64, device="cuda")
            lib.sdtw_debug_set_trace(eng.ctx, C.c_void_p(tr.data_ptr()))
            eng.sdtw_with_gradients(x, y, g, out=outs)
            cnt = (C.c_uint * 16)()
            lib.sdtw_debug_counters(eng.ctx, cnt, 16)
            lib.sdtw_debug_set_trace(eng.ctx, None)
            print(json.dumps({"config": cfg_name, "ms": round(tot / 5, 4),
                              "phases": {k: round(v / 5, 4) for k, v in ph.items()},
                              "counters": list(cnt)}), flush=True)
        except Exception as e:
            print(f"[{cfg_name}] ERROR {e}", flush=True)
    eng.close()


if __name__ == "__main__":
    main()
