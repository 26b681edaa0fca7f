"""Prescribed spectra of the paper's test-matrix suite (§4.1, Table 1).

SEEDED INPUT GENERATION ONLY -- this module holds none of ChASE's arithmetic.  It is shared by
the oracle tests and the CUDA-path tests/bench as the source of *inputs* and of the exact
spectra the results are pinned to.

Citations (P:L = /root/reference/PAPER.md line L):
  * Uniform    lambda_k = d_max (eps + (k-1)(1-eps)/(n-1))          P:613 (Table 1)
  * Geometric  lambda_k = d_max eps^((n-k)/(n-1))                    P:615 (Table 1)
  * (1-2-1)    lambda_k = 2 - 2 cos(pi k/(n+1)), tridiag(1, 2, 1)    P:561, P:617 (Table 1)
  * Wilkinson  tridiagonal, unit off-diagonals, diagonal (m, ..., 1, ..., m), m=(n-1)/2
               "all positive but one, roughly in pairs"
Readings (SURVEY §8(c) ledger #8-#10):
  * d_max = 1, eps = 1e-4 (kappa = 1/eps = 1.0e4 as printed at P:765).
  * Wilkinson diagonal d_i = |i - (n-1)/2|, i = 0..n-1 (standard W+ for odd n; half-integers for
    even n).  This is the only reading that reproduces the paper's kappa(n=20000) = 4.7e4.
"""
from __future__ import annotations

import numpy as np

FAMILIES = ("uniform", "geometric", "121", "wilkinson")


def uniform(n: int, d_max: float = 1.0, eps: float = 1e-4) -> np.ndarray:
    """Table 1 'Uniform'."""
    k = np.arange(1, n + 1, dtype=np.float64)
    if n == 1:
        return np.array([d_max * eps])
    return d_max * (eps + (k - 1.0) * (1.0 - eps) / (n - 1.0))


def geometric(n: int, d_max: float = 1.0, eps: float = 1e-4) -> np.ndarray:
    """Table 1 'Geometric'."""
    k = np.arange(1, n + 1, dtype=np.float64)
    if n == 1:
        return np.array([d_max])
    return d_max * eps ** ((n - k) / (n - 1.0))


def one_two_one(n: int) -> np.ndarray:
    """Table 1 '(1-2-1)': 2 - 2cos(pi k/(n+1)) written as 4 sin^2(pi k / (2(n+1)))
    (the same number, without the cancellation near k = 1)."""
    k = np.arange(1, n + 1, dtype=np.float64)
    return 4.0 * np.sin(np.pi * k / (2.0 * (n + 1))) ** 2


def wilkinson_diagonal(n: int) -> np.ndarray:
    """Diagonal of the Wilkinson matrix under ledger reading #8: d_i = |i - (n-1)/2|."""
    i = np.arange(n, dtype=np.float64)
    return np.abs(i - (n - 1) / 2.0)


def sturm_count(d: np.ndarray, e: np.ndarray, x: np.ndarray) -> np.ndarray:
    """Number of eigenvalues < x of the symmetric tridiagonal (d, e), for each x (vectorised
    over x).  Plain LDL^T Sturm sequence (textbook; Golub & Van Loan 8.4)."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    cnt = np.zeros(x.shape, dtype=np.int64)
    q = d[0] - x
    tiny = 1e-300
    q = np.where(q == 0.0, -tiny, q)
    cnt += q < 0
    for i in range(1, len(d)):
        q = (d[i] - x) - e[i - 1] * e[i - 1] / q
        q = np.where(q == 0.0, -tiny, q)
        cnt += q < 0
    return cnt


def sturm_bisection(d: np.ndarray, e: np.ndarray, iters: int = 80) -> np.ndarray:
    """All eigenvalues of the symmetric tridiagonal (d, e) by Sturm bisection (small n only)."""
    n = len(d)
    r = np.zeros(n)
    r[:-1] += np.abs(e)
    r[1:] += np.abs(e)
    lo = np.full(n, np.min(d - r)) - 1.0
    hi = np.full(n, np.max(d + r)) + 1.0
    k = np.arange(n)
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        c = sturm_count(d, e, mid)
        go_hi = c > k          # more than k eigenvalues below mid -> lambda_k < mid
        hi = np.where(go_hi, mid, hi)
        lo = np.where(go_hi, lo, mid)
    return 0.5 * (lo + hi)


def wilkinson(n: int) -> np.ndarray:
    """Eigenvalues of the Wilkinson matrix (ledger #8), ascending.  Large n uses LAPACK's
    tridiagonal eigensolver (scipy); tests pin it to `sturm_bisection` and to P:765."""
    d = wilkinson_diagonal(n)
    e = np.ones(n - 1)
    if n <= 512:
        return np.sort(sturm_bisection(d, e))
    from scipy.linalg import eigvalsh_tridiagonal
    return np.sort(eigvalsh_tridiagonal(d, e))


def spectrum(family: str, n: int, d_max: float = 1.0, eps: float = 1e-4) -> np.ndarray:
    """Exact spectrum (ascending) of a Table 1 family."""
    family = family.lower()
    if family in ("uniform", "uni"):
        return uniform(n, d_max, eps)
    if family in ("geometric", "geo"):
        return geometric(n, d_max, eps)
    if family in ("121", "1-2-1", "onetwoone"):
        return one_two_one(n)
    if family in ("wilkinson", "wilk"):
        return wilkinson(n)
    raise ValueError(f"unknown spectral family {family!r}")


def tridiagonal(family: str, n: int):
    """(d, e) of the literal tridiagonal matrices (1-2-1 P:561; Wilkinson P:562-564)."""
    family = family.lower()
    if family in ("121", "1-2-1", "onetwoone"):
        return np.full(n, 2.0), np.ones(n - 1)
    if family in ("wilkinson", "wilk"):
        return wilkinson_diagonal(n), np.ones(n - 1)
    raise ValueError(f"{family!r} is not a tridiagonal family")
