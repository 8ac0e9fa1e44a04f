"""Backward-v5 counters (sdtw_debug_counters) and phase times per config."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
NAMES = ["live", "stored", "ovf", "_3", "jobs", "skipped", "tiles_rc", "E_tile_kcyc", "E_below_kcyc",
         "E_req_kcyc", "E_strip_kcyc", "runs", "tiles_entered", "H_busy_kcyc", "H_idle_kcyc", "E_start_kcyc"]


def main():
    import torch
    import bench
    from paper_2602_17206_b200 import Engine
    from paper_2602_17206_b200.capi import load_library
    lib = load_library()
    for cfg_name in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["c2", "c3"]):
        cfg = bench.CONFIGS[cfg_name]
        B, L, D, g = cfg["B"], cfg["L"], cfg["D"], cfg["gamma"]
        xh, yh = bench.bench_inputs(B, L, D, 42)
        x, y = torch.from_numpy(xh).cuda(), torch.from_numpy(yh).cuda()
        eng = Engine(0)
        outs = (torch.empty(B, device="cuda"), torch.empty((B, L, D), device="cuda"),
                torch.empty((B, L, D), device="cuda"))
        eng.enable_timing(True)
        eng.sdtw_with_gradients(x, y, g, out=outs)
        ph_plain = eng.phase_times()
        S = (L + 31) // 32
        tr = torch.zeros(128 * B * S, dtype=torch.int64, device="cuda")
        lib.sdtw_debug_set_trace(eng.ctx, C.c_void_p(tr.data_ptr()))
        eng.sdtw_with_gradients(x, y, g, out=outs)
        cnt = (C.c_uint * 16)()
        lib.sdtw_debug_counters(eng.ctx, cnt, 16)
        lib.sdtw_debug_set_trace(eng.ctx, None)
        print(json.dumps({"config": cfg_name, "knobs": os.environ.get("SDTW_KNOBS"),
                          "phases": {k: round(v, 4) for k, v in ph_plain.items()},
                          "counters": dict(zip(NAMES, list(cnt)))}), flush=True)
        eng.close()


if __name__ == "__main__":
    main()
