"""A/B of per-phase device times for one config: the library in SDTW_LIB
(default: the in-tree build) on reference-generator or torch.randn inputs.

    SDTW_LIB=... python scripts/ab_phases.py --config c3 --data ref
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--data", default="ref", choices=["ref", "randn"])
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--modes", default="fused,unfused")
    a = ap.parse_args()
    import torch
    import bench
    from paper_2602_17206_b200 import Engine
    cfg = bench.CONFIGS[a.config]
    B, L, D, g = cfg["B"], cfg["L"], cfg["D"], cfg["gamma"]
    if a.data == "ref":
        xh, yh = bench.bench_inputs(B, L, D, 42)
        x, y = torch.from_numpy(xh).cuda(), torch.from_numpy(yh).cuda()
    else:
        gen = torch.Generator(device="cuda").manual_seed(42)
        x = torch.randn((B, L, D), generator=gen, device="cuda")
        y = torch.randn((B, L, D), generator=gen, device="cuda")
    eng = Engine(0)
    side = torch.cuda.Stream()
    torch.cuda.set_stream(side)
    eng.set_stream(side.cuda_stream)
    outs = (torch.empty(B, device="cuda"), torch.empty((B, L, D), device="cuda"),
            torch.empty((B, L, D), device="cuda"))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    res = {"lib": os.environ.get("SDTW_LIB", "in-tree"), "config": a.config, "data": a.data}
    for mode in a.modes.split(","):
        tot, ph, _, peak = bench.time_engine(eng, torch, x, y, outs, mode == "fused", g, a.steps, 3, flush)
        res[mode] = {"ms": tot / a.steps, **{k: round(v / a.steps, 4) for k, v in ph.items()}}
        # one synchronous call: surfaces dependency-wait timeouts as an error
        eng.sdtw_with_gradients(x, y, g, fused=mode == "fused", out=outs)
    print(json.dumps(res), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
