import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI)")
    config.addinivalue_line("markers", "slow: larger parity sizes")


@pytest.fixture(scope="session")
def golden():
    d = np.load(os.path.join(ROOT, "tests", "golden", "sdtw_small.npz"))
    n = int(d["n_cases"])
    cases = []
    for k in range(n):
        c = {}
        for name in ("x", "y", "gamma", "bandwidth", "loss", "R", "costs", "E", "E_linear",
                     "grad_x", "grad_y"):
            c[name] = d[f"c{k}_{name}"]
        c["gamma"] = float(c["gamma"])
        c["bandwidth"] = int(c["bandwidth"])
        cases.append(c)
    return cases


@pytest.fixture(scope="session")
def bary_golden():
    return dict(np.load(os.path.join(ROOT, "tests", "golden", "barycenter_small.npz")))


@pytest.fixture(scope="session")
def engine():
    from paper_2602_17206_b200 import Engine
    from paper_2602_17206_b200.build import build
    build()
    eng = Engine(0)
    yield eng
    eng.close()


@pytest.fixture(scope="session")
def oracle_c():
    import oracle
    return oracle.OracleC()


@pytest.fixture(scope="session")
def reference():
    import oracle
    if not oracle.have_reference():
        try:
            oracle.build_oracle()
        except Exception:
            pass
    if not oracle.have_reference():
        pytest.skip("reference library oracle/_ref/libsdtw_ref.so not built")
    return oracle.Reference()
