"""B200-native Soft-DTW engine (drop-in for arxiv/paper_2602_17206's hot path).

The product is the CUDA shared library libsdtw_b200.so behind the C-ABI in
include/sdtw_capi.h; C++ callers use the drop-in headers include/softdtw/,
Python callers use :class:`Engine` (ctypes).  There is no CPU fallback.
"""
from .capi import (  # noqa: F401
    BWD_LINEAR,
    BWD_LOG,
    COST_FUSED,
    COST_UNFUSED,
    DeviceError,
    Engine,
    IncompleteTableError,
    OutOfMemoryError,
    SdtwError,
    UnreachableEndError,
    ValidationError,
    load_library,
)
