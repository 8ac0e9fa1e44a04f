"""Where is the C3 gradient's worst element vs the fp64 reference?"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import oracle
    from paper_2602_17206_b200 import Engine
    from tests.tolerances import rel_err
    ref = oracle.Reference()
    x, y = ref.bench_inputs(32, 4096, 128)
    pairs = [int(p) for p in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["0", "31"])]
    xs, ys = np.ascontiguousarray(x[pairs]), np.ascontiguousarray(y[pairs])
    rc, rl, rgx, rgy = ref.sdtw_with_gradients(xs.astype(np.float64), ys.astype(np.float64), 0.01)
    eng = Engine(0)
    for fused in (False, True):
        l, gx, gy = eng.sdtw_with_gradients(xs, ys, 0.01, fused=fused)
        for nm, a, r in (("gx", gx, rgx), ("gy", gy, rgy)):
            e = rel_err(a, r)
            idx = np.unravel_index(np.argmax(e), e.shape)
            rows = (e.max(axis=2) > 1e-4)
            print(f"fused={fused} {nm} max {e.max():.3e} at {idx} got {a[idx]:.6f} want {r[idx]:.6f}; "
                  f"rows>1e-4 per pair {rows.sum(axis=1)}; loss rel {rel_err(l, rl)}", flush=True)
            for b in range(len(pairs)):
                bad = np.nonzero(rows[b])[0]
                if len(bad):
                    print("   pair", pairs[b], "bad rows", bad[:20], flush=True)
    eng.close()


if __name__ == "__main__":
    main()
