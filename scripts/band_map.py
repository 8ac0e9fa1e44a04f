"""Per-strip live-tile ranges of the fp32 alignment gradient E (non-zero 32x32
tiles), for band-prediction analysis: prints lo/hi chunk per strip."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import bench
    from paper_2602_17206_b200 import Engine
    eng = Engine(0)
    out = {}
    for cfg_name, pairs in (("c3", [0, 7]), ("c2", [0]), ("c1", [0])):
        cfg = bench.CONFIGS[cfg_name]
        B, L, D, g = cfg["B"], cfg["L"], cfg["D"], cfg["gamma"]
        x, y = bench.bench_inputs(B, L, D, 42)
        for p in pairs:
            _, E = eng.forward_backward_E(np.ascontiguousarray(x[p:p + 1]), np.ascontiguousarray(y[p:p + 1]), g)
            E = E[0, 1:-1, 1:-1]
            S, Cc = (L + 31) // 32, (L + 31) // 32
            nz = np.zeros((S, Cc), bool)
            for s in range(S):
                for c in range(Cc):
                    nz[s, c] = np.any(E[32 * s:32 * s + 32, 32 * c:32 * c + 32] != 0)
            rng = []
            for s in range(S):
                cs = np.nonzero(nz[s])[0]
                rng.append([int(cs.min()), int(cs.max()), int(len(cs))] if len(cs) else [-1, -1, 0])
            out[f"{cfg_name}_p{p}"] = rng
    print(json.dumps(out))


if __name__ == "__main__":
    main()
