"""Band-cache misses of one fused call, printed by the debug build:
SDTW_LIB=paper_2602_17206_b200/libsdtw_dbg.so python scripts/band_debug.py B L D gamma"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import bench
    from paper_2602_17206_b200 import Engine
    B, L, D = (int(v) for v in sys.argv[1:4])
    gamma = float(sys.argv[4])
    x, y = bench.bench_inputs(B, L, D, 42)
    eng = Engine(0)
    eng.sdtw_with_gradients(x, y, gamma, fused=True)
    print("band stats", eng.band_stats(), flush=True)


if __name__ == "__main__":
    main()
