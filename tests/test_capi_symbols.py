"""CPU: the C-ABI library builds for sm_100a, loads, and exports every symbol
include/sdtw_capi.h declares.  No compute calls (no GPU here)."""
import ctypes
import os
import re
import subprocess

from tests.conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "sdtw_capi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(sdtw_[A-Za-z0-9_]+)\s*\(", src))
    return sorted(names)


def test_library_builds_and_exports_all_symbols():
    from paper_2602_17206_b200.build import build
    from paper_2602_17206_b200 import capi
    lib_path = build()
    lib = ctypes.CDLL(lib_path)
    declared = _declared()
    assert len(declared) >= 25
    missing = [n for n in declared if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(capi.EXPORTED) == declared


def test_library_is_sm100a():
    from paper_2602_17206_b200.build import build
    lib_path = build()
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True)
    assert "sm_100a" in out.stdout, out.stdout + out.stderr


def test_no_cpu_fallback_without_gpu():
    """Creating a context without a usable B200 fails loudly."""
    import torch
    if torch.cuda.is_available():
        return
    from paper_2602_17206_b200 import Engine, DeviceError
    try:
        Engine(0)
    except DeviceError as e:
        assert "CPU fallback" in str(e) or "device" in str(e).lower()
    else:
        raise AssertionError("engine constructed without a GPU")
