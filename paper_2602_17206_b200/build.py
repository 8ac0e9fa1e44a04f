"""Builds the engine's CUDA shared library for sm_100a (B200), in-tree.

    python -m paper_2602_17206_b200.build      # or __graft_entry__.build()

Output: paper_2602_17206_b200/libsdtw_b200.so (git-ignored, travels to the GPU
box with the gpurun snapshot).  nvcc cross-compiles without a GPU.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsdtw_b200.so")
# the host side (sdtw_capi.cu) and the DP kernels in their own translation
# units (sdtw_kernels.h), compiled in parallel and linked into one library
SOURCES = ["sdtw_capi.cu", "k_fwd_f32.cu", "k_fwd_f64.cu", "k_bwd4.cu",
           "k_gemm.cu"]
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith((".cuh", ".h")))
OBJDIR = os.path.join(HERE, "_obj")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _obj(src: str) -> str:
    return os.path.join(OBJDIR, src.replace(".cu", ".o"))


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    global LIB, OBJDIR, NVCC_FLAGS
    if os.environ.get("SDTW_BUILD_DEBUG"):  # bounds-checked variant (experiments)
        LIB = os.path.join(HERE, "libsdtw_dbg.so")
        OBJDIR = os.path.join(HERE, "_obj_dbg")
        NVCC_FLAGS = NVCC_FLAGS + ["-DSDTW_B5_DEBUG"]
    hdrs = [os.path.join(CSRC, f) for f in HEADERS] + [os.path.join(ROOT, "include", "sdtw_capi.h")]
    os.makedirs(OBJDIR, exist_ok=True)
    todo = [src for src in SOURCES
            if force or _stale(_obj(src), [os.path.join(CSRC, src)] + hdrs)]
    procs = []
    for src in todo:
        cmd = [_nvcc(), *NVCC_FLAGS, "-c", "-o", _obj(src) + ".tmp", os.path.join(CSRC, src)]
        procs.append((src, cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    log_parts, failed = [], []
    for src, cmd, pr in procs:
        out, err = pr.communicate()
        log_parts.append(" ".join(cmd) + "\n" + out + err)
        if pr.returncode != 0:
            failed.append((src, err))
        else:
            os.replace(_obj(src) + ".tmp", _obj(src))
    objs = [_obj(src) for src in SOURCES]
    if not failed and (todo or _stale(LIB, objs)):
        cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB + ".tmp", *objs, "-ldl"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        log_parts.append(" ".join(cmd) + "\n" + res.stdout + res.stderr)
        if res.returncode != 0:
            failed.append(("link", res.stderr))
        else:
            os.replace(LIB + ".tmp", LIB)
    if todo:
        with open(os.path.join(HERE, "build.log"), "w") as fh:
            fh.write("\n".join(log_parts))
    if failed:
        for src, err in failed:
            sys.stderr.write(f"--- {src}\n{err[-6000:]}\n")
        raise RuntimeError(f"nvcc failed: {[f for f, _ in failed]} (see build.log)")
    if verbose:
        sys.stdout.write("\n".join(log_parts))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
