"""Generates tests/golden/*.npz from the REFERENCE ITSELF.

Runs the unmodified reference (oracle/_ref/libsdtw_ref.so, compiled from
/root/reference/proj/include by oracle/Makefile) in its T=double
instantiation on seeded inputs, and stores inputs + outputs.  Re-run with

    make -C oracle && python tests/golden/make_golden.py

The fixtures pin (a) the C restatement in oracle/ (bit-exact) and (b) the
CUDA engine (within the tolerances in tests/tolerances.py) without needing
/root/reference at test time.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Reference  # noqa: E402


def main():
    ref = Reference()
    rng = np.random.default_rng(20261018)
    cases = []
    # (B, N, M, D, gamma, bandwidth)
    shapes = [
        (1, 1, 1, 1, 1.0, 0),
        (1, 2, 2, 1, 1.0, 0),
        (2, 7, 5, 3, 1.0, 0),
        (3, 12, 12, 4, 0.1, 0),
        (2, 9, 14, 2, 10.0, 0),
        (2, 33, 31, 5, 0.5, 0),
        (1, 40, 40, 3, 0.01, 0),
        (2, 20, 20, 2, 1.0, 3),
        (1, 17, 23, 3, 0.2, 8),
        (2, 65, 70, 8, 0.05, 0),
        (1, 1, 9, 2, 1.0, 0),
        (1, 11, 1, 2, 1.0, 0),
    ]
    for idx, (B, N, M, D, g, bw) in enumerate(shapes):
        if idx == 1:  # the worked example of test_forward.cpp:43-57
            x = np.array([[[0.0], [1.0]]]); y = np.array([[[0.0], [1.0]]])
        elif idx == 0:  # test_forward.cpp:33-41 / test_backward.cpp:51-61
            x = np.array([[[2.0]]]); y = np.array([[[5.0]]])
        else:
            # fp32-representable inputs so fp32 engines see identical values
            x = rng.uniform(-1, 1, (B, N, D)).astype(np.float32).astype(np.float64)
            y = rng.uniform(-1, 1, (B, M, D)).astype(np.float32).astype(np.float64)
        rc, loss, R, d, E = ref.tables(x, y, g, bandwidth=bw)
        assert rc == 0, rc
        rc, loss2, gx, gy = ref.sdtw_with_gradients(x, y, g, bandwidth=bw)
        assert rc == 0 and np.array_equal(loss, loss2)
        rc, _, _, _, El = ref.tables(x, y, g, bandwidth=bw, log_space=False)
        assert rc == 0
        cases.append(dict(x=x, y=y, gamma=g, bandwidth=bw, loss=loss, R=R, costs=d, E=E,
                          E_linear=El, grad_x=gx, grad_y=gy))
    out = {}
    for k, c in enumerate(cases):
        for name, v in c.items():
            out[f"c{k}_{name}"] = np.asarray(v)
    out["n_cases"] = np.array(len(cases))
    np.savez_compressed(os.path.join(HERE, "sdtw_small.npz"), **out)

    # Barycenter objective on blockwave members (datasets.hpp:21-80, seed 2024
    # as acceptance.cpp:312-313), K=6, L=24, D=2.
    rc, members = ref.generate_dataset(0, 6, 24, 2, 0.05, 2024)
    assert rc == 0
    z = members.mean(axis=0)
    w = np.array([1.0, 0.5, 0.0, 2.0, 1.0, 1.0])
    rc, val, grad = ref.barycenter_objective(z, members, 1.0)
    rc2, valw, gradw = ref.barycenter_objective(z, members, 1.0, weights=w)
    assert rc == 0 and rc2 == 0
    rc, obj, conv, zf = ref.solve_barycenter(members, 24, gamma=1.0, lr=0.01, max_iters=20, tol=0.0)
    assert rc == 0
    np.savez_compressed(os.path.join(HERE, "barycenter_small.npz"), members=members, z=z,
                        value=val, grad=grad, weights=w, value_w=valw, grad_w=gradw,
                        trace=obj, final_z=zf)
    # bench generator spec (bench.hpp:61-66): first values, to pin the input
    # generator used by bench.py against the reference's.
    x, y = ref.bench_inputs(2, 4, 3, 42)
    np.savez_compressed(os.path.join(HERE, "bench_inputs_small.npz"), x=x, y=y)
    print("wrote", len(cases), "cases")


if __name__ == "__main__":
    main()
