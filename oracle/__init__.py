"""Parity checkers (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package.  It binds two shared libraries built by
oracle/Makefile:

  _ref/libsdtw_oracle.so  the plain-C restatement (sdtw_oracle.c), fp64
  _ref/libsdtw_ref.so     the UNMODIFIED reference compiled from
                          /root/reference/proj/include (ref_shim.cpp)
"""
from .bind import (  # noqa: F401
    OracleC,
    Reference,
    build_oracle,
    have_reference,
)
