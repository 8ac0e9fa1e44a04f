"""ctypes bindings of the oracle libraries (TEST INFRASTRUCTURE ONLY)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
ORACLE_SO = os.path.join(REF_DIR, "libsdtw_oracle.so")
REF_SO = os.path.join(REF_DIR, "libsdtw_ref.so")

P, S, D, I, U = C.c_void_p, C.c_size_t, C.c_double, C.c_int, C.c_uint


def build_oracle(quiet: bool = True) -> None:
    """make -C oracle (builds the C restatement; the reference too when
    /root/reference is present)."""
    res = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + res.stdout + res.stderr)
    if not quiet:
        print(res.stdout)


def have_reference() -> bool:
    return os.path.exists(REF_SO)


def _ptr(a):
    return None if a is None else a.ctypes.data


class OracleC:
    """The C restatement (fp64)."""

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            build_oracle()
        lib = C.CDLL(ORACLE_SO)
        lib.oracle_softmin.restype = D
        lib.oracle_softmin.argtypes = [D, D, D, D]
        lib.oracle_logsumexp3.restype = D
        lib.oracle_logsumexp3.argtypes = [D, D, D]
        lib.oracle_costs.argtypes = [P, P, S, S, S, S, P]
        lib.oracle_forward.restype = I
        lib.oracle_forward.argtypes = [P, P, S, S, S, S, D, S, P, P]
        lib.oracle_backward.restype = I
        lib.oracle_backward.argtypes = [P, P, S, S, S, D, S, I]
        lib.oracle_input_gradients.argtypes = [P, P, P, S, S, S, S, P, P]
        lib.oracle_sdtw_with_gradients.restype = I
        lib.oracle_sdtw_with_gradients.argtypes = [P, P, S, S, S, S, D, S, I, P, P, P]
        lib.oracle_barycenter_objective.restype = D
        lib.oracle_barycenter_objective.argtypes = [P, S, P, S, S, S, D, S, P, P]
        lib.oracle_adam_step.argtypes = [P, P, P, P, S, S, D, D, D, D]
        self.lib = lib

    def softmin(self, a, b, c, g):
        return self.lib.oracle_softmin(a, b, c, g)

    def logsumexp3(self, a, b, c):
        return self.lib.oracle_logsumexp3(a, b, c)

    def costs(self, x, y):
        x = np.ascontiguousarray(x, np.float64); y = np.ascontiguousarray(y, np.float64)
        B, N, Dm = x.shape; M = y.shape[1]
        d = np.empty((B, N, M), np.float64)
        self.lib.oracle_costs(_ptr(x), _ptr(y), B, N, M, Dm, _ptr(d))
        return d

    def forward(self, x, y, gamma, bandwidth=0):
        x = np.ascontiguousarray(x, np.float64); y = np.ascontiguousarray(y, np.float64)
        B, N, Dm = x.shape; M = y.shape[1]
        R = np.empty((B, N + 2, M + 2), np.float64)
        loss = np.empty(B, np.float64)
        rc = self.lib.oracle_forward(_ptr(x), _ptr(y), B, N, M, Dm, gamma, bandwidth, _ptr(R), _ptr(loss))
        return rc, loss, R

    def backward(self, R, d, gamma, bandwidth=0, log_space=True):
        slab = np.ascontiguousarray(R, np.float64).copy()
        d = np.ascontiguousarray(d, np.float64)
        B, N2, M2 = slab.shape
        rc = self.lib.oracle_backward(_ptr(slab), _ptr(d), B, N2 - 2, M2 - 2, gamma, bandwidth,
                                      1 if log_space else 0)
        return rc, slab

    def input_gradients(self, E, x, y):
        x = np.ascontiguousarray(x, np.float64); y = np.ascontiguousarray(y, np.float64)
        E = np.ascontiguousarray(E, np.float64)
        B, N, Dm = x.shape; M = y.shape[1]
        gx = np.empty_like(x); gy = np.empty_like(y)
        self.lib.oracle_input_gradients(_ptr(E), _ptr(x), _ptr(y), B, N, M, Dm, _ptr(gx), _ptr(gy))
        return gx, gy

    def sdtw_with_gradients(self, x, y, gamma, bandwidth=0):
        x = np.ascontiguousarray(x, np.float64); y = np.ascontiguousarray(y, np.float64)
        B, N, Dm = x.shape; M = y.shape[1]
        loss = np.empty(B); gx = np.empty_like(x); gy = np.empty_like(y)
        rc = self.lib.oracle_sdtw_with_gradients(_ptr(x), _ptr(y), B, N, M, Dm, gamma, bandwidth, 1,
                                                 _ptr(loss), _ptr(gx), _ptr(gy))
        return rc, loss, gx, gy

    def barycenter_objective(self, z, members, gamma, bandwidth=0, weights=None):
        z = np.ascontiguousarray(z, np.float64); m = np.ascontiguousarray(members, np.float64)
        Lz, Dm = z.shape; K, L, _ = m.shape
        w = None if weights is None else np.ascontiguousarray(weights, np.float64)
        grad = np.empty_like(z)
        v = self.lib.oracle_barycenter_objective(_ptr(z), Lz, _ptr(m), K, L, Dm, gamma, bandwidth,
                                                 _ptr(w), _ptr(grad))
        return v, grad


class Reference:
    """The reference itself, compiled from /root/reference (ref_shim.cpp)."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            build_oracle()
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        lib = C.CDLL(REF_SO)
        for suf in ("f64", "f32"):
            f = getattr(lib, f"ref_sdtw_with_gradients_{suf}")
            f.restype = I
            f.argtypes = [P, P, S, S, S, S, D, S, I, I, U, P, P, P]
            f = getattr(lib, f"ref_tables_{suf}")
            f.restype = I
            f.argtypes = [P, P, S, S, S, S, D, S, I, I, U, P, P, P, P]
            f = getattr(lib, f"ref_barycenter_objective_{suf}")
            f.restype = I
            f.argtypes = [P, S, P, S, S, S, D, S, P, U, P, P]
        lib.ref_solve_barycenter_f64.restype = I
        lib.ref_solve_barycenter_f64.argtypes = [P, S, S, S, S, D, S, D, S, D, U, P,
                                                 C.POINTER(S), C.POINTER(I), P]
        lib.ref_run_bench_row.restype = I
        lib.ref_run_bench_row.argtypes = [S, S, S, D, I, I, S, S, U, C.c_ulonglong,
                                          C.POINTER(D), C.POINTER(D), C.POINTER(S),
                                          C.POINTER(C.c_float)]
        lib.ref_bench_inputs.restype = None
        lib.ref_bench_inputs.argtypes = [S, S, S, C.c_ulonglong, P, P]
        lib.ref_generate_dataset.restype = I
        lib.ref_generate_dataset.argtypes = [I, S, S, S, D, C.c_ulonglong, P]
        lib.ref_hardware_threads.restype = U
        self.lib = lib

    @staticmethod
    def _dt(dtype):
        return "f32" if np.dtype(dtype) == np.float32 else "f64"

    def sdtw_with_gradients(self, x, y, gamma, bandwidth=0, fused=False, log_space=True,
                            threads=0, dtype=np.float64):
        x = np.ascontiguousarray(x, dtype); y = np.ascontiguousarray(y, dtype)
        B, N, Dm = x.shape; M = y.shape[1]
        loss = np.empty(B, dtype); gx = np.empty_like(x); gy = np.empty_like(y)
        rc = getattr(self.lib, f"ref_sdtw_with_gradients_{self._dt(dtype)}")(
            _ptr(x), _ptr(y), B, N, M, Dm, gamma, bandwidth, int(fused), int(log_space), threads,
            _ptr(loss), _ptr(gx), _ptr(gy))
        return rc, loss, gx, gy

    def tables(self, x, y, gamma, bandwidth=0, fused=False, log_space=True, threads=0,
               dtype=np.float64, want_E=True):
        x = np.ascontiguousarray(x, dtype); y = np.ascontiguousarray(y, dtype)
        B, N, Dm = x.shape; M = y.shape[1]
        loss = np.empty(B, dtype)
        R = np.empty((B, N + 2, M + 2), dtype)
        d = np.empty((B, N, M), dtype)
        E = np.empty((B, N + 2, M + 2), dtype) if want_E else None
        rc = getattr(self.lib, f"ref_tables_{self._dt(dtype)}")(
            _ptr(x), _ptr(y), B, N, M, Dm, gamma, bandwidth, int(fused), int(log_space), threads,
            _ptr(loss), _ptr(R), _ptr(d), _ptr(E))
        return rc, loss, R, d, E

    def barycenter_objective(self, z, members, gamma, bandwidth=0, weights=None, threads=0,
                             dtype=np.float64):
        z = np.ascontiguousarray(z, dtype); m = np.ascontiguousarray(members, dtype)
        Lz, Dm = z.shape; K, L, _ = m.shape
        w = None if weights is None else np.ascontiguousarray(weights, np.float64)
        grad = np.empty_like(z)
        val = C.c_double()
        rc = getattr(self.lib, f"ref_barycenter_objective_{self._dt(dtype)}")(
            _ptr(z), Lz, _ptr(m), K, L, Dm, gamma, bandwidth, _ptr(w), threads, C.byref(val),
            _ptr(grad))
        return rc, val.value, grad

    def solve_barycenter(self, members, Lz, gamma=1.0, bandwidth=0, lr=0.01, max_iters=100,
                         tol=0.0, threads=0):
        m = np.ascontiguousarray(members, np.float64)
        K, L, Dm = m.shape
        obj = np.empty(max_iters + 1)
        iters = C.c_size_t(); conv = C.c_int()
        z = np.empty((Lz, Dm))
        rc = self.lib.ref_solve_barycenter_f64(_ptr(m), K, L, Dm, Lz, gamma, bandwidth, lr,
                                               max_iters, tol, threads, _ptr(obj), C.byref(iters),
                                               C.byref(conv), _ptr(z))
        return rc, obj[: iters.value + 1], bool(conv.value), z

    def run_bench_row(self, B, L, D_, gamma=1.0, fused=False, repeats=1, warmup=0, threads=0,
                      seed=42):
        mean, std, peak, l0 = C.c_double(), C.c_double(), C.c_size_t(), C.c_float()
        rc = self.lib.ref_run_bench_row(B, L, D_, gamma, int(fused), 1, repeats, warmup, threads,
                                        seed, C.byref(mean), C.byref(std), C.byref(peak),
                                        C.byref(l0))
        return rc, mean.value, std.value, peak.value, l0.value

    def bench_inputs(self, B, L, D_, seed=42):
        x = np.empty((B, L, D_), np.float32); y = np.empty((B, L, D_), np.float32)
        self.lib.ref_bench_inputs(B, L, D_, seed, _ptr(x), _ptr(y))
        return x, y

    def generate_dataset(self, kind, count, length, dim, noise, seed):
        out = np.empty((count, length, dim), np.float64)
        rc = self.lib.ref_generate_dataset(kind, count, length, dim, noise, seed, _ptr(out))
        return rc, out

    def hardware_threads(self) -> int:
        return int(self.lib.ref_hardware_threads())
