"""CPU oracle for ChASE (arXiv 2205.02491) -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline` leg and
`--impl reference`) may import, call or execute anything in this package.  The CUDA product
path (`paper_2205_02491_b200/`) shares no code with it and never falls back to it.

Contents
  chase.py  plain numpy complex128 implementation of Alg. 1 step by step:
            filter (three-term recurrence P:385-390), Lanczos + DoS bounds,
            QR of [Y V], Rayleigh-Ritz, residuals, degrees,
            deflation & locking, bound update, sort.
  rng.py    the counter-based start-vector generator (oracle side; the CUDA side implements
            the same definition independently).

Pinning (tests/test_oracle_*.py): closed-form Table 1 spectra, exact G2 eigenvectors, the
closed-form Chebyshev filter in the eigenbasis, SPEC worked examples, brute-force Jacobi on tiny
n, and the condition numbers printed at P:765.  Parity unpinned: the paper's iteration counts
and matvecs (Table 2, P:658-661 / P:685-688) -- they depend on unpublished DEMAGIS inputs and
on heuristics the paper does not state (ledger #10); DESIGN.md lists them.
"""
from .chase import (  # noqa: F401
    filter_interval, filter_coefficients, hemm_step, hemm_step_rows, chebyshev_filter, chebyshev_T,
    lanczos, LanczosResult, qr_locked, rayleigh_ritz, residual_norms, optimal_degrees,
    lock_prefix, chase_solve, Report,
)
from .rng import random_block, philox4x32_10, STREAM_START_V, STREAM_LANCZOS  # noqa: F401
