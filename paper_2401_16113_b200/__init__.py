"""B200-native (sm_100a, fp64) all-at-once Crank–Nicolson solver with the block α-circulant
parallel-in-time preconditioner of arxiv 2401.16113.

The compute path is the C-ABI library ``libcnpint.so`` (hand-written CUDA, include/cnpint.h);
``cnpint`` is its ctypes binding and ``problems`` the caller-side workload setup.
"""
from .cnpint import (CnpintError, OperatorSpec, Solver, load_library, stream_copy, EXPORTS,  # noqa: F401
                     LIB_PATH)
