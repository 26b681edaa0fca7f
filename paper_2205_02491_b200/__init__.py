"""B200-native ChASE (arXiv 2205.02491): Chebyshev-filtered subspace iteration on sm_100a.

The product is the C-ABI library `libchase_b200.so` (include/chase.h).  This package holds its
CUDA sources (`csrc/`), the in-tree build (`build.py`) and a thin ctypes binding (`_lib.py`).
"""
from ._lib import (Chase, ChaseError, Report, load, version, EXPORTS, nccl_unique_id,  # noqa: F401
                   kernel_launches)
