"""Backward timing over SDTW_KNOBS settings (one process per setting is not
needed: the knobs are read per call)."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    from paper_2602_17206_b200 import Engine
    from paper_2602_17206_b200.capi import load_library
    lib = load_library()
    eng = Engine(0)
    side = torch.cuda.Stream()
    torch.cuda.set_stream(side)
    eng.set_stream(side.cuda_stream)
    cfgs = sys.argv[1].split(",")
    knobsets = sys.argv[2].split(";")
    for cfg_name in cfgs:
        cfg = bench.CONFIGS[cfg_name]
        B, L, D, g = cfg["B"], cfg["L"], cfg["D"], cfg["gamma"]
        xh, yh = bench.bench_inputs(B, L, D, 42)
        x, y = torch.from_numpy(xh).cuda(), torch.from_numpy(yh).cuda()
        outs = (torch.empty(B, device="cuda"), torch.empty((B, L, D), device="cuda"),
                torch.empty((B, L, D), device="cuda"))
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        for ks in knobsets:
            os.environ["SDTW_KNOBS"] = ks
            try:
                tot, ph, _, _ = bench.time_engine(eng, torch, x, y, outs, False, g, 3, 2, flush)
                eng.sdtw_with_gradients(x, y, g, out=outs)
                print(json.dumps({"config": cfg_name, "knobs": ks, "backward": round(ph.get("backward", 0) / 3, 4),
                                  "ms": round(tot / 3, 4)}), flush=True)
            except Exception as e:
                print(f"{cfg_name} {ks} ERROR {e}", flush=True)
                return
    eng.close()


if __name__ == "__main__":
    main()
