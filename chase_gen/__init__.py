"""Seeded synthetic inputs for ChASE tests and benchmarks (§4.1, Table 1).

Shared by the oracle tests and the CUDA path as the single source of *inputs*; contains none of
the method's arithmetic (no filter, QR, Rayleigh-Ritz, residual or Lanczos code).
"""
from .spectra import spectrum, FAMILIES, tridiagonal, sturm_bisection  # noqa: F401
from .dense import G1Matrix, G2Matrix, R2Matrix, make_matrix, block_partition  # noqa: F401
