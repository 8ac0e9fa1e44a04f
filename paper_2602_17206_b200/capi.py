"""ctypes binding of the engine's C-ABI (include/sdtw_capi.h).

This is the binding a Python caller (the tests, bench.py) uses; a C++ caller
uses the drop-in headers include/softdtw/*.hpp over the same C-ABI.  Arrays
are numpy arrays (host, the call stages them) or torch CUDA tensors (device
pointers, no copies).  There is no CPU fallback: if the shared library or a
B200 is missing, construction fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsdtw_b200.so")

SDTW_OK, SDTW_EINVAL, SDTW_ENOMEM, SDTW_EUNREACHABLE, SDTW_EINCOMPLETE, SDTW_ECUDA, SDTW_ENCCL = range(7)
COST_UNFUSED, COST_FUSED = 0, 1
BWD_LOG, BWD_LINEAR = 0, 1
PTR_HOST, PTR_DEVICE, FLAG_ASYNC = 0, 1, 0x100

# Every symbol include/sdtw_capi.h declares (checked by tests/test_capi_symbols.py).
EXPORTED = [
    "sdtw_ctx_create", "sdtw_ctx_destroy", "sdtw_ctx_set_stream", "sdtw_ctx_stream",
    "sdtw_ctx_synchronize", "sdtw_mem_stats", "sdtw_mem_reset_peak", "sdtw_set_mem_limit",
    "sdtw_mem_trim", "sdtw_launch_count", "sdtw_reset_launch_count", "sdtw_ctx_enable_timing",
    "sdtw_phase_times", "sdtw_debug_set_trace", "sdtw_debug_phase_status", "sdtw_debug_band_stats",
    "sdtw_last_error",
    "sdtw_last_oom_bytes", "sdtw_fwd_bwd_f32", "sdtw_fwd_bwd_f64", "sdtw_forward_f32",
    "sdtw_forward_f64", "sdtw_backward_table_f32", "sdtw_backward_table_f64",
    "sdtw_forward_backward_E_f32", "sdtw_forward_backward_E_f64", "sdtw_input_grads_f32",
    "sdtw_input_grads_f64", "sdtw_barycenter_objective_f32", "sdtw_barycenter_objective_f64",
    "sdtw_adam_step_f32", "sdtw_adam_step_f64", "sdtw_nccl_get_unique_id", "sdtw_nccl_init",
    "sdtw_nccl_finalize", "sdtw_allreduce_grad_f32", "sdtw_fwd_bwd_multi_f32", "sdtw_fwd_bwd_multi_f64",
    "sdtw_nccl_init_all", "sdtw_barycenter_objective_multi_f32", "sdtw_device_count",
]


class SdtwError(RuntimeError):
    """Base error (softdtw::Error, types.hpp:17-20)."""


class ValidationError(SdtwError):
    pass


class OutOfMemoryError(SdtwError):
    def __init__(self, msg: str, requested: int):
        super().__init__(msg)
        self.requested_bytes = requested


class UnreachableEndError(SdtwError):
    pass


class IncompleteTableError(SdtwError):
    pass


class DeviceError(SdtwError):
    pass


class sdtw_config(C.Structure):
    _fields_ = [
        ("gamma", C.c_double),
        ("bandwidth", C.c_size_t),
        ("cost_mode", C.c_int),
        ("backward_space", C.c_int),
        ("normalized", C.c_int),
    ]


_lib = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Loads libsdtw_b200.so; raises ImportError if it was not built.
    SDTW_LIB overrides the path (experiment builds)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("SDTW_LIB") or path
    if not os.path.exists(path):
        raise ImportError(
            f"CUDA engine library missing at {path}: run `python -m paper_2602_17206_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(path)
    P, S, D, I, U64 = C.c_void_p, C.c_size_t, C.c_double, C.c_int, C.c_uint64
    cfgp = C.POINTER(sdtw_config)
    sig = {
        "sdtw_ctx_create": (I, [I, C.POINTER(P)]),
        "sdtw_ctx_destroy": (I, [P]),
        "sdtw_ctx_set_stream": (I, [P, P]),
        "sdtw_ctx_stream": (P, [P]),
        "sdtw_ctx_synchronize": (I, [P]),
        "sdtw_mem_stats": (I, [P, C.POINTER(S), C.POINTER(S)]),
        "sdtw_mem_reset_peak": (I, [P]),
        "sdtw_set_mem_limit": (I, [P, S]),
        "sdtw_mem_trim": (I, [P]),
        "sdtw_launch_count": (U64, [P]),
        "sdtw_reset_launch_count": (None, [P]),
        "sdtw_last_error": (C.c_char_p, []),
        "sdtw_ctx_enable_timing": (I, [P, I]),
        "sdtw_phase_times": (I, [P, C.POINTER(C.c_float), I]),
        "sdtw_debug_set_trace": (I, [P, P]),
        "sdtw_debug_phase_status": (I, [P, C.POINTER(C.c_int), I]),
        "sdtw_debug_band_stats": (I, [P, C.POINTER(C.c_ulonglong)]),
        "sdtw_last_oom_bytes": (S, []),
        "sdtw_nccl_get_unique_id": (I, [P]),
        "sdtw_nccl_init": (I, [P, P, I, I]),
        "sdtw_nccl_finalize": (I, [P]),
        "sdtw_allreduce_grad_f32": (I, [P, P, S, P]),
        "sdtw_nccl_init_all": (I, [C.POINTER(P), I]),
        "sdtw_device_count": (I, [C.POINTER(I)]),
        "sdtw_barycenter_objective_multi_f32": (I, [C.POINTER(P), I, P, S, P, S, S, S, D, S, P, I, P, P]),
    }
    for suf in ("f32", "f64"):
        sig[f"sdtw_fwd_bwd_{suf}"] = (I, [P, P, P, S, S, S, S, cfgp, I, P, P, P])
        sig[f"sdtw_forward_{suf}"] = (I, [P, P, P, S, S, S, S, cfgp, I, P, P, P, P])
        sig[f"sdtw_backward_table_{suf}"] = (I, [P, P, P, P, P, S, S, S, S, cfgp, I, P])
        sig[f"sdtw_forward_backward_E_{suf}"] = (I, [P, P, P, S, S, S, S, cfgp, I, P, P])
        sig[f"sdtw_input_grads_{suf}"] = (I, [P, P, P, P, S, S, S, S, I, P, P])
        sig[f"sdtw_barycenter_objective_{suf}"] = (I, [P, P, S, P, S, S, S, D, S, P, I, P, P])
        sig[f"sdtw_adam_step_{suf}"] = (I, [P, P, P, P, P, S, S, D, D, D, D, I])
        sig[f"sdtw_fwd_bwd_multi_{suf}"] = (I, [C.POINTER(P), I, P, P, S, S, S, S, cfgp, I, P, P, P])
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _raise(rc: int) -> None:
    if rc == SDTW_OK:
        return
    lib = load_library()
    msg = (lib.sdtw_last_error() or b"").decode()
    if rc == SDTW_EINVAL:
        raise ValidationError(msg)
    if rc == SDTW_ENOMEM:
        raise OutOfMemoryError(msg, int(lib.sdtw_last_oom_bytes()))
    if rc == SDTW_EUNREACHABLE:
        raise UnreachableEndError(msg)
    if rc == SDTW_EINCOMPLETE:
        raise IncompleteTableError(msg)
    raise DeviceError(f"[{rc}] {msg}")


def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


class _Args:
    """Collects pointers for one call; all arrays must share residency."""

    def __init__(self, dtype):
        self.dtype = np.dtype(dtype)
        self.keep = []
        self.kind = None

    def _set_kind(self, kind):
        if self.kind is None:
            self.kind = kind
        elif self.kind != kind:
            raise ValidationError("mixing host and device arrays in one call")

    def inp(self, a):
        if a is None:
            return None
        if _is_torch(a):
            import torch
            if not a.is_cuda:
                a = a.detach().cpu().numpy()
            else:
                want = torch.float32 if self.dtype == np.float32 else torch.float64
                if a.dtype != want or not a.is_contiguous():
                    raise ValidationError("device tensors must be contiguous and of the call dtype")
                self._set_kind(PTR_DEVICE)
                self.keep.append(a)
                return a.data_ptr()
        arr = np.ascontiguousarray(a, dtype=self.dtype)
        self._set_kind(PTR_HOST)
        self.keep.append(arr)
        return arr.ctypes.data

    def out(self, a):
        if a is None:
            return None
        if _is_torch(a) and not a.is_cuda:
            a = a.numpy()  # host tensor (e.g. pinned): a view, written in place
        if _is_torch(a):
            self._set_kind(PTR_DEVICE)
            self.keep.append(a)
            return a.data_ptr()
        if not (a.flags.c_contiguous and a.dtype == self.dtype):
            raise ValidationError("output arrays must be C-contiguous of the call dtype")
        self._set_kind(PTR_HOST)
        self.keep.append(a)
        return a.ctypes.data


class Engine:
    """One engine context (sdtw_ctx) on one CUDA device."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        h = C.c_void_p()
        _raise(self.lib.sdtw_ctx_create(int(device), C.byref(h)))
        self.ctx = h
        self.device = device

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.sdtw_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- plumbing ------------------------------------------------------
    def set_stream(self, stream_ptr: int | None):
        _raise(self.lib.sdtw_ctx_set_stream(self.ctx, stream_ptr or None))

    def synchronize(self):
        _raise(self.lib.sdtw_ctx_synchronize(self.ctx))

    def mem_stats(self):
        live, peak = C.c_size_t(), C.c_size_t()
        _raise(self.lib.sdtw_mem_stats(self.ctx, C.byref(live), C.byref(peak)))
        return live.value, peak.value

    def reset_peak(self):
        _raise(self.lib.sdtw_mem_reset_peak(self.ctx))

    def set_mem_limit(self, limit: int):
        _raise(self.lib.sdtw_set_mem_limit(self.ctx, int(limit)))

    def trim(self):
        _raise(self.lib.sdtw_mem_trim(self.ctx))

    PHASES = ("norms", "costs", "forward", "backward", "grads")

    def enable_timing(self, on: bool = True):
        _raise(self.lib.sdtw_ctx_enable_timing(self.ctx, 1 if on else 0))

    def phase_times(self) -> dict:
        arr = (C.c_float * len(self.PHASES))()
        _raise(self.lib.sdtw_phase_times(self.ctx, arr, len(self.PHASES)))
        return {k: float(v) for k, v in zip(self.PHASES, arr) if v >= 0}

    def band_stats(self) -> tuple:
        """(fused backward passes that used the band cache, band misses that
        reran on the tensor cores) since the context was created."""
        arr = (C.c_ulonglong * 2)()
        _raise(self.lib.sdtw_debug_band_stats(self.ctx, arr))
        return int(arr[0]), int(arr[1])

    @property
    def launches(self) -> int:
        return int(self.lib.sdtw_launch_count(self.ctx))

    def reset_launches(self):
        self.lib.sdtw_reset_launch_count(self.ctx)

    @staticmethod
    def _cfg(gamma, bandwidth, fused, linear, normalized=False):
        return sdtw_config(float(gamma), int(bandwidth), COST_FUSED if fused else COST_UNFUSED,
                           BWD_LINEAR if linear else BWD_LOG, 1 if normalized else 0)

    @staticmethod
    def _suffix(dtype):
        return "f32" if np.dtype(dtype) == np.float32 else "f64"

    @staticmethod
    def _dims(x, y):
        if len(x.shape) != 3 or len(y.shape) != 3:
            raise ValidationError("series must be B x L x D")
        B, N, D = (int(v) for v in x.shape)
        B2, M, D2 = (int(v) for v in y.shape)
        if B != B2:
            raise ValidationError("batch size mismatch")
        if D != D2:
            raise ValidationError("feature dim mismatch")
        return B, N, M, D

    def _alloc_like(self, x, shape, dtype):
        if _is_torch(x) and x.is_cuda:
            import torch
            return torch.empty(shape, dtype=torch.float32 if np.dtype(dtype) == np.float32 else torch.float64,
                               device=x.device)
        return np.empty(shape, dtype=dtype)

    # ---- sdtw_with_gradients (backward.hpp:276-304) ----------------------
    def sdtw_with_gradients(self, x, y, gamma=1.0, bandwidth=0, fused=False, dtype=np.float32,
                            grads=True, out=None, sync=True):
        B, N, M, D = self._dims(x, y)
        a = _Args(dtype)
        px, py = a.inp(x), a.inp(y)
        if out is None:
            loss = self._alloc_like(x, (B,), dtype)
            gx = self._alloc_like(x, (B, N, D), dtype) if grads else None
            gy = self._alloc_like(x, (B, M, D), dtype) if grads else None
        else:
            loss, gx, gy = out
        pl, pgx, pgy = a.out(loss), a.out(gx), a.out(gy)
        cfg = self._cfg(gamma, bandwidth, fused, False)
        kind = a.kind | (0 if sync else FLAG_ASYNC)
        fn = getattr(self.lib, f"sdtw_fwd_bwd_{self._suffix(dtype)}")
        _raise(fn(self.ctx, px, py, B, N, M, D, C.byref(cfg), kind, pl, pgx, pgy))
        return loss, gx, gy

    # ---- forward (forward.hpp:43-81) ------------------------------------
    def forward(self, x, y, gamma=1.0, bandwidth=0, fused=False, dtype=np.float64, table=False,
                costs=False, norms=False, normalized=False):
        B, N, M, D = self._dims(x, y)
        a = _Args(dtype)
        px, py = a.inp(x), a.inp(y)
        loss = self._alloc_like(x, (B,), dtype)
        R = self._alloc_like(x, (B, N + 2, M + 2), dtype) if table else None
        dc = self._alloc_like(x, (B, N, M), dtype) if costs else None
        nm = self._alloc_like(x, (B * (N + M),), dtype) if norms else None
        cfg = self._cfg(gamma, bandwidth, fused, False, normalized)
        fn = getattr(self.lib, f"sdtw_forward_{self._suffix(dtype)}")
        _raise(fn(self.ctx, px, py, B, N, M, D, C.byref(cfg), a.kind, a.out(loss), a.out(R),
                  a.out(dc), a.out(nm)))
        return loss, R, dc, nm

    # ---- backward over a table (backward.hpp:183-203) -------------------
    def backward_table(self, R, gamma=1.0, bandwidth=0, costs=None, x=None, y=None, linear=False,
                       dtype=np.float64):
        B, N2, M2 = (int(v) for v in R.shape)
        N, M = N2 - 2, M2 - 2
        D = int(x.shape[2]) if x is not None else 0
        a = _Args(dtype)
        pR, pc, px, py = a.inp(R), a.inp(costs), a.inp(x), a.inp(y)
        E = self._alloc_like(R, (B, N + 2, M + 2), dtype)
        cfg = self._cfg(gamma, bandwidth, costs is None, linear)
        fn = getattr(self.lib, f"sdtw_backward_table_{self._suffix(dtype)}")
        _raise(fn(self.ctx, pR, pc, px, py, B, N, M, D, C.byref(cfg), a.kind, a.out(E)))
        return E

    # ---- loss + E from the engine's own forward -------------------------
    def forward_backward_E(self, x, y, gamma=1.0, bandwidth=0, fused=False, dtype=np.float32):
        B, N, M, D = self._dims(x, y)
        a = _Args(dtype)
        px, py = a.inp(x), a.inp(y)
        loss = self._alloc_like(x, (B,), dtype)
        E = self._alloc_like(x, (B, N + 2, M + 2), dtype)
        cfg = self._cfg(gamma, bandwidth, fused, False)
        fn = getattr(self.lib, f"sdtw_forward_backward_E_{self._suffix(dtype)}")
        _raise(fn(self.ctx, px, py, B, N, M, D, C.byref(cfg), a.kind, a.out(loss), a.out(E)))
        return loss, E

    # ---- input_gradients (backward.hpp:208-266) -------------------------
    def input_gradients(self, E, x, y, dtype=np.float64):
        B, N, M, D = self._dims(x, y)
        a = _Args(dtype)
        pE, px, py = a.inp(E), a.inp(x), a.inp(y)
        gx = self._alloc_like(x, (B, N, D), dtype)
        gy = self._alloc_like(x, (B, M, D), dtype)
        fn = getattr(self.lib, f"sdtw_input_grads_{self._suffix(dtype)}")
        _raise(fn(self.ctx, pE, px, py, B, N, M, D, a.kind, a.out(gx), a.out(gy)))
        return gx, gy

    # ---- barycenter_objective (barycenter.hpp:60-86) --------------------
    def barycenter_objective(self, z, members, gamma=1.0, bandwidth=0, weights=None,
                             dtype=np.float32, grad_out=None, value_out=None):
        Lz, D = (int(v) for v in z.shape[-2:])
        K, L, D2 = (int(v) for v in members.shape)
        if D != D2:
            raise ValidationError("barycenter: members disagree on feature dim")
        a = _Args(dtype)
        pz, pm = a.inp(z), a.inp(members)
        w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
        grad = grad_out if grad_out is not None else self._alloc_like(z, (Lz, D), dtype)
        if value_out is not None:
            val_arr = value_out
        elif a.kind == PTR_DEVICE:
            import torch
            val_arr = torch.zeros(1, dtype=torch.float64, device=z.device)
        else:
            val_arr = np.zeros(1, dtype=np.float64)
        pv = val_arr.data_ptr() if _is_torch(val_arr) else val_arr.ctypes.data
        fn = getattr(self.lib, f"sdtw_barycenter_objective_{self._suffix(dtype)}")
        _raise(fn(self.ctx, pz, Lz, pm, K, L, D, float(gamma), int(bandwidth),
                  None if w is None else w.ctypes.data, a.kind, pv, a.out(grad)))
        value = float(val_arr[0]) if value_out is None else None
        return value, grad

    def adam_step(self, z, grad, m1, m2, t, lr=0.01, beta1=0.9, beta2=0.999, eps=1e-8,
                  dtype=np.float32):
        n = int(np.prod(z.shape))
        a = _Args(dtype)
        pz = a.out(z)
        pg = a.inp(grad)
        kind = a.kind
        p1 = m1.data_ptr() if _is_torch(m1) else m1.ctypes.data
        p2 = m2.data_ptr() if _is_torch(m2) else m2.ctypes.data
        fn = getattr(self.lib, f"sdtw_adam_step_{self._suffix(dtype)}")
        _raise(fn(self.ctx, pz, pg, p1, p2, n, int(t), lr, beta1, beta2, eps, kind))

    # ---- NCCL ----------------------------------------------------------
    def nccl_unique_id(self) -> bytes:
        buf = C.create_string_buffer(128)
        _raise(self.lib.sdtw_nccl_get_unique_id(buf))
        return buf.raw

    def nccl_init(self, uid: bytes, nranks: int, rank: int):
        buf = C.create_string_buffer(uid, 128)
        _raise(self.lib.sdtw_nccl_init(self.ctx, buf, nranks, rank))

    def allreduce_grad(self, grad_dev, value_dev=None):
        _raise(self.lib.sdtw_allreduce_grad_f32(self.ctx, grad_dev.data_ptr(), grad_dev.numel(),
                                                None if value_dev is None else value_dev.data_ptr()))


# ---- multi-GPU in one process (sdtw_fwd_bwd_multi_*) ------
def _ctx_array(engines):
    arr = (C.c_void_p * len(engines))()
    for g, e in enumerate(engines):
        arr[g] = e.ctx
    return arr


def sdtw_with_gradients_multi(engines, x, y, gamma=1.0, bandwidth=0, fused=False, dtype=np.float32):
    """The B pairs in len(engines) contiguous shards, one per engine context
    (normally one per GPU), run concurrently; host (numpy) arrays only.
    Bit-identical to one engine's sdtw_with_gradients."""
    lib = load_library()
    x = np.ascontiguousarray(x, dtype)
    y = np.ascontiguousarray(y, dtype)
    B, N, D = x.shape
    M = y.shape[1]
    loss = np.empty(B, dtype)
    gx = np.empty_like(x)
    gy = np.empty_like(y)
    cfg = Engine._cfg(gamma, bandwidth, fused, False)
    fn = getattr(lib, f"sdtw_fwd_bwd_multi_{Engine._suffix(dtype)}")
    _raise(fn(_ctx_array(engines), len(engines), x.ctypes.data, y.ctypes.data, B, N, M, D, C.byref(cfg),
              PTR_HOST, loss.ctypes.data, gx.ctypes.data, gy.ctypes.data))
    return loss, gx, gy


def nccl_init_all(engines):
    """One NCCL communicator over the engines' devices (ncclCommInitAll)."""
    _raise(load_library().sdtw_nccl_init_all(_ctx_array(engines), len(engines)))


def barycenter_objective_multi(engines, z, members, gamma=1.0, bandwidth=0, weights=None):
    """barycenter_objective over len(engines) GPUs: member shards + one NCCL
    allreduce of grad_z and the objective (fp32; host arrays)."""
    lib = load_library()
    z = np.ascontiguousarray(z, np.float32)
    m = np.ascontiguousarray(members, np.float32)
    Lz, D = z.shape
    K, L, _ = m.shape
    w = None if weights is None else np.ascontiguousarray(weights, np.float64)
    grad = np.empty_like(z)
    val = C.c_double()
    _raise(lib.sdtw_barycenter_objective_multi_f32(_ctx_array(engines), len(engines), z.ctypes.data, Lz,
                                                  m.ctypes.data, K, L, D, gamma, bandwidth,
                                                  None if w is None else w.ctypes.data, PTR_HOST,
                                                  C.byref(val), grad.ctypes.data))
    return val.value, grad
