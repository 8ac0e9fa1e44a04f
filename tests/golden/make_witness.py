"""Generates tests/golden/witness.npz: the reference's fp32 stability witness.

The witness (proj/tests/test_backward.cpp:286-321, acceptance.cpp:96-134):
L = 2048, D = 2, gamma = 1e-3, x = 2 u, y = 7 - 2 u with u drawn by
std::uniform_real_distribution<float> from std::mt19937_64(1), x then y.
The draw is implementation-defined, so a tiny C++ program compiled with the
same libstdc++ as the reference reproduces it bit for bit; the expected
outputs come from the unmodified reference (oracle/_ref/libsdtw_ref.so) in
T=double on those fp32 inputs (the fp32 reference's own
gradients are not the bar).  Re-run with

    make -C oracle && python tests/golden/make_witness.py
"""
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Reference  # noqa: E402

GEN = r"""
#include <cstdio>
#include <random>
#include <vector>
int main() {
    std::mt19937_64 rng(1);
    const std::size_t L = 2048, D = 2;
    std::uniform_real_distribution<float> u(0.0f, 1.0f);
    std::vector<float> xs(L * D), ys(L * D);
    for (auto &v : xs) v = 2.0f * u(rng);
    for (auto &v : ys) v = 7.0f - 2.0f * u(rng);
    std::fwrite(xs.data(), sizeof(float), xs.size(), stdout);
    std::fwrite(ys.data(), sizeof(float), ys.size(), stdout);
    return 0;
}
"""


def witness_inputs():
    with tempfile.TemporaryDirectory() as d:
        src, exe = os.path.join(d, "gen.cpp"), os.path.join(d, "gen")
        with open(src, "w") as fh:
            fh.write(GEN)
        subprocess.run(["g++", "-O2", "-std=c++20", src, "-o", exe], check=True)
        raw = subprocess.run([exe], check=True, capture_output=True).stdout
    v = np.frombuffer(raw, np.float32)
    n = 2048 * 2
    return v[:n].reshape(1, 2048, 2).copy(), v[n:].reshape(1, 2048, 2).copy()


def main():
    ref = Reference()
    x, y = witness_inputs()
    g = 1e-3
    rc, loss, gx, gy = ref.sdtw_with_gradients(x.astype(np.float64), y.astype(np.float64), g)
    assert rc == 0, rc
    rc, _, _, _, E = ref.tables(x.astype(np.float64), y.astype(np.float64), g)
    assert rc == 0, rc
    out = dict(x=x, y=y, gamma=np.float64(g), loss=loss, grad_x=gx, grad_y=gy,
               E11=np.float64(E[0, 1, 1]), E_rowsum=E[0, 1:-1, 1:-1].sum(axis=1))
    path = os.path.join(HERE, "witness.npz")
    np.savez_compressed(path, **out)
    print(path, "loss", loss, "E11", E[0, 1, 1])


if __name__ == "__main__":
    main()
