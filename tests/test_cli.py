"""The reference's own command-line front end (proj/tools/sdtw.cpp, compiled
unchanged) on the engine: tools/_bin/sdtw is built with
include/softdtw_redirect first on the include path, so its library calls run
on the B200; oracle/_ref/sdtw_ref_cli is the same source on the reference's
CPU implementation (test infrastructure).  Both read and write the
reference's file formats (io.hpp: CSV series, SDTW v1 binary, manifests)."""
import os
import subprocess

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CLI = os.path.join(ROOT, "tools", "_bin", "sdtw")
REF_CLI = os.path.join(ROOT, "oracle", "_ref", "sdtw_ref_cli")
REF_SRC = "/root/reference/proj/tools/sdtw.cpp"


def _run(exe, *args, cwd=None):
    r = subprocess.run([exe, *args], capture_output=True, text=True, timeout=600, cwd=cwd)
    assert r.returncode == 0, (exe, args, r.stdout[-2000:], r.stderr[-2000:])
    return r.stdout


@pytest.mark.skipif(not os.path.exists(REF_SRC), reason="reference sources not mounted (GPU box)")
def test_cli_builds_against_engine():
    from paper_2602_17206_b200.build import build
    build()
    r = subprocess.run(["make", "-C", os.path.join(ROOT, "tools")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    assert os.path.exists(CLI) and os.path.exists(REF_CLI)


def _losses(csv_text):
    rows = [ln.split(",") for ln in csv_text.strip().splitlines()[1:]]
    return np.array([float(r[1]) for r in rows])


@pytest.mark.gpu
def test_cli_matches_reference_cli(tmp_path):
    for exe in (CLI, REF_CLI):
        if not os.path.exists(exe):
            pytest.fail(f"{exe} missing: build it where the reference is mounted (make -C tools)")
    data = tmp_path / "data"
    _run(CLI, "generate", "--kind", "blockwave", "--count", "4", "--length", "96", "--dim", "3",
         "--out-dir", str(data))
    files = sorted(str(p) for p in data.glob("*.csv"))
    assert len(files) == 4
    manifest = tmp_path / "pairs.txt"
    manifest.write_text("\n".join(f"{files[i]},{files[i + 1]}" for i in range(3)) + "\n")
    for prec, tol in (("f64", 1e-10), ("f32", 1e-5)):
        for mode in ("unfused", "fused"):
            args = ["sdtw", "--manifest", str(manifest), "--gamma", "0.3", "--precision", prec, "--mode", mode]
            got, want = _losses(_run(CLI, *args)), _losses(_run(REF_CLI, *args))
            assert got.shape == (3,)
            assert (np.abs(got - want) / np.maximum(1, np.abs(want))).max() <= tol, (prec, mode, got, want)
    # gradients written as SDTW v1 binary series by both
    gp, rp = tmp_path / "g_eng", tmp_path / "g_ref"
    _run(CLI, "sdtw", files[0], files[1], "--gamma", "0.3", "--grad", str(gp))
    _run(REF_CLI, "sdtw", files[0], files[1], "--gamma", "0.3", "--grad", str(rp))
    for side in ("x", "y"):
        a = np.fromfile(f"{gp}_0_{side}.bin", dtype=np.uint8)
        b = np.fromfile(f"{rp}_0_{side}.bin", dtype=np.uint8)
        assert a.size == b.size
    # the benchmark matrix: same CSV columns, one row per (length, mode)
    out = _run(CLI, "bench", "--batches", "4", "--lengths", "64", "--dims", "8", "--repeats", "1")
    lines = out.strip().splitlines()
    assert lines[0] == _run(REF_CLI, "bench", "--batches", "1", "--lengths", "8", "--dims", "1",
                            "--repeats", "1").strip().splitlines()[0]
    assert len(lines) == 3 and all(ln.endswith("ok") for ln in lines[1:])
    # barycenter: same objective trace (f64 members, 3 Adam iterations)
    for exe, tag in ((CLI, "eng"), (REF_CLI, "ref")):
        _run(exe, "barycenter", str(data), "--iters", "3", "--gamma", "1.0", "-o", str(tmp_path / f"bc_{tag}.csv"),
             "--trace", str(tmp_path / f"tr_{tag}.csv"))
    te = np.loadtxt(tmp_path / "tr_eng.csv", delimiter=",", skiprows=1)
    tr = np.loadtxt(tmp_path / "tr_ref.csv", delimiter=",", skiprows=1)
    assert np.allclose(te[:, 1], tr[:, 1], rtol=1e-9, atol=1e-9), (te, tr)
