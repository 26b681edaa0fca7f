"""Brute-force complex cyclic Jacobi eigensolver (tests only; pins the oracle and the generator
independently of LAPACK).  Textbook two-sided Jacobi (Golub & Van Loan 8.5) for Hermitian A."""
import numpy as np


def jacobi_eigvalsh(A, sweeps=30, tol=1e-15):
    A = np.array(A, dtype=np.complex128, copy=True)
    n = A.shape[0]
    for _ in range(sweeps):
        off = np.sqrt(max(np.sum(np.abs(A) ** 2) - np.sum(np.abs(np.diag(A)) ** 2), 0.0))
        if off <= tol * np.linalg.norm(A):
            break
        for p in range(n - 1):
            for q in range(p + 1, n):
                apq = A[p, q]
                if abs(apq) < 1e-300:
                    continue
                # make the (p,q) entry real with a phase, then a real Jacobi rotation
                ph = apq / abs(apq)
                app, aqq = A[p, p].real, A[q, q].real
                tau = (aqq - app) / (2.0 * abs(apq))
                t = np.sign(tau) / (abs(tau) + np.hypot(1.0, tau)) if tau != 0 else 1.0
                c = 1.0 / np.sqrt(1.0 + t * t)
                s = t * c
                # J = [[c, s*ph], [-s*conj(ph), c]] acting on columns p, q
                Ap = A[:, p].copy()
                Aq = A[:, q].copy()
                A[:, p] = c * Ap - s * np.conj(ph) * Aq
                A[:, q] = s * ph * Ap + c * Aq
                Ap = A[p, :].copy()
                Aq = A[q, :].copy()
                A[p, :] = c * Ap - s * ph * Aq
                A[q, :] = s * np.conj(ph) * Ap + c * Aq
    return np.sort(np.diag(A).real)
