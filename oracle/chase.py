"""Plain, slow, obviously-correct CPU ChASE (Alg. 1 of arXiv 2205.02491) in complex128 numpy.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import this package.  The CUDA product path never routes through it
(and shares no code with it: no kernels, headers, helpers or constant generators).

Every function cites the PAPER.md (P:L) / SPEC.md (S:L) passage it follows; readings of silent
or garbled passages are the numbered ledger items of SURVEY.md §8(c), restated in DESIGN.md.
Library primitives used as single steps: matrix products (@), numpy.linalg.qr (Householder),
numpy.linalg.eigh (dense Hermitian eigensolver, the "standard dense solver" of P:306).

Parity pins (tests/test_oracle_*.py, `-m "not gpu"`): closed-form spectra of Table 1, exact
eigenvectors of the G2 generator, the Chebyshev closed form C_m(t(H))/C_m(tau) evaluated in the
eigenbasis, SPEC worked examples (C_2(-3)=17, degrees 1/8/cap, locking prefix, full-Krylov
Lanczos), brute-force Jacobi on tiny n, and the paper's printed condition numbers.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .rng import random_block, STREAM_START_V, STREAM_LANCZOS


# ----------------------------------------------------------------------------------------------
# Filter (Alg. 1 line 4; three-term recurrence P:385-390; interval P:325)
# ----------------------------------------------------------------------------------------------
def filter_interval(b_sup: float, mu_ne: float):
    """c = (b_sup + mu_ne)/2, e = (b_sup - mu_ne)/2  (Alg. 1 line 10)."""
    return 0.5 * (b_sup + mu_ne), 0.5 * (b_sup - mu_ne)


def filter_coefficients(b_sup: float, mu_1: float, mu_ne: float, kmax: int):
    """Scalars (alpha_k, beta_k), gamma_k = c, of the three-term recurrence
    V_{k+1} = alpha_k (A - gamma_k I) V_k + beta_k V_{k-1}.
    Ledger #1: damped scaled Chebyshev, sigma_1 = e/(mu_1 - c);
      k = 1: alpha = sigma_1/e, beta = 0;
      k >= 2: sigma_k = 1/(2/sigma_1 - sigma_{k-1}), alpha = 2 sigma_k/e, beta = -sigma_{k-1} sigma_k.
    Returns (c, e, [(alpha_1, beta_1), ..., (alpha_kmax, beta_kmax)])."""
    c, e = filter_interval(b_sup, mu_ne)
    sigma1 = e / (mu_1 - c)
    out = [(sigma1 / e, 0.0)]
    sigma_prev = sigma1
    for _ in range(2, kmax + 1):
        sigma = 1.0 / (2.0 / sigma1 - sigma_prev)
        out.append((2.0 * sigma / e, -sigma_prev * sigma))
        sigma_prev = sigma
    return c, e, out


def hemm_step(H, X, Yprev, alpha, beta, gamma):
    """One filter step  alpha (H - gamma I) X + beta Yprev  (Eqs. w=av / v=aw P:393-397).
    Because H is Hermitian the forward (W = A V) and backward (V = A^H W) forms are the
    same operator; the distributed layouts only change where rows live, not the values."""
    Y = alpha * (H @ X - gamma * X)
    if beta != 0.0:
        Y = Y + beta * Yprev
    return Y


def hemm_step_rows(H_rows, row0, X, Yprev_rows, alpha, beta, gamma):
    """Rows [row0, row0 + H_rows.shape[0]) of hemm_step (the same definition restricted to a
    row panel of H; used for bounded CPU timing samples at sizes where H does not fit)."""
    nr = H_rows.shape[0]
    Y = alpha * (H_rows @ X - gamma * X[row0:row0 + nr])
    if beta != 0.0:
        Y = Y + beta * Yprev_rows
    return Y


def chebyshev_filter(H, V, degrees, b_sup, mu_1, mu_ne):
    """V-hat <- Filter(A, b_sup, mu_1, mu_ne, V-hat, m)  (Alg. 1 line 4).
    Column a receives the degree-m_a polynomial; a column leaves the product as soon as its
    degree is exhausted (P:329 'Sort ... according to m').  Serial 1x1 semantics.
    Returns (filtered V, matvecs = sum_a m_a  (P:729-731 footnote))."""
    degrees = np.asarray(degrees, dtype=np.int64)
    V = np.array(V, dtype=np.result_type(H, V, np.float64), copy=True)
    kmax = int(degrees.max()) if degrees.size else 0
    if kmax == 0:
        return V, 0
    c, _, coef = filter_coefficients(b_sup, mu_1, mu_ne, kmax)
    Y_prev = V.copy()                      # Y_0
    Y_cur = V.copy()
    act = degrees >= 1
    a1, _ = coef[0]
    Y_cur[:, act] = hemm_step(H, V[:, act], None, a1, 0.0, c)          # Y_1
    for k in range(2, kmax + 1):
        act = degrees >= k
        if not act.any():
            break
        ak, bk = coef[k - 1]
        Y_new = hemm_step(H, Y_cur[:, act], Y_prev[:, act], ak, bk, c)
        Y_prev[:, act] = Y_cur[:, act]
        Y_cur[:, act] = Y_new
    return Y_cur, int(degrees.sum())


def chebyshev_T(m: int, t):
    """Chebyshev polynomial of the first kind C_m(t) for any real t (closed form)."""
    t = np.asarray(t, dtype=np.float64)
    out = np.empty_like(t)
    inside = np.abs(t) <= 1.0
    out[inside] = np.cos(m * np.arccos(t[inside]))
    to = t[~inside]
    out[~inside] = np.sign(to) ** m * np.cosh(m * np.arccosh(np.abs(to)))
    return out


# ----------------------------------------------------------------------------------------------
# Lanczos + DoS (Alg. 1 line 2; DoS P:301)
# ----------------------------------------------------------------------------------------------
@dataclass
class LanczosResult:
    b_sup: float
    mu_1: float
    mu_ne: float
    nu: float                    # max |Ritz| (residual normalisation, ledger #5)
    ritz: np.ndarray             # pooled Ritz values (all runs)
    weights: np.ndarray          # pooled DoS weights |z_1k|^2 / L


def tridiag_eigh(alpha, beta):
    """Eigenpairs of the real symmetric tridiagonal T_m (library dense eigensolver step)."""
    m = len(alpha)
    T = np.diag(alpha) + np.diag(beta[: m - 1], 1) + np.diag(beta[: m - 1], -1)
    return np.linalg.eigh(T)


def lanczos(H, n_e: int, steps: int = 25, runs: int = 4, seed: int = 3, start=None) -> LanczosResult:
    """Spectral bounds by 'a small number of repeated Lanczos steps' + DoS.
    Ledger #14: `runs` independent runs of `steps` steps with full reorthogonalisation;
    b_sup = max_r (theta_max + |beta_m|); mu_1 = min theta; mu_ne = smallest pooled theta whose
    DoS CDF (weights |z_1k|^2 / runs) reaches n_e/N.  Degenerate-interval guard S:478."""
    N = H.shape[0]
    if start is None:
        start = random_block(seed, 0, N, 0, runs, STREAM_LANCZOS)
        if not np.iscomplexobj(H):
            start = start.real          # real-symmetric variant: real part of the same draw
    steps = min(steps, N)
    thetas, weights = [], []
    b_sup = -np.inf
    for r in range(runs):
        v = start[:, r] / np.linalg.norm(start[:, r])
        Q = [v]
        alpha, beta = [], []
        for j in range(steps):
            w = H @ Q[j]
            a = np.vdot(Q[j], w).real
            w = w - a * Q[j]
            if j > 0:
                w = w - beta[j - 1] * Q[j - 1]
            Qm = np.stack(Q, axis=1)
            w = w - Qm @ (Qm.conj().T @ w)          # full reorthogonalisation
            b = np.linalg.norm(w)
            alpha.append(a)
            beta.append(b)
            if j + 1 < steps:
                if b <= 1e-14 * max(1.0, abs(a)):   # invariant subspace found: stop the run
                    break
                Q.append(w / b)
        th, Z = tridiag_eigh(np.array(alpha), np.array(beta))
        b_sup = max(b_sup, th[-1] + abs(beta[len(alpha) - 1]))
        thetas.append(th)
        weights.append(np.abs(Z[0, :]) ** 2 / runs)
    ritz = np.concatenate(thetas)
    wts = np.concatenate(weights)
    order = np.argsort(ritz, kind="stable")
    ritz, wts = ritz[order], wts[order]
    mu_1 = float(ritz[0])
    cdf = np.cumsum(wts)
    idx = int(np.searchsorted(cdf, n_e / N - 1e-15))
    idx = min(idx, len(ritz) - 1)
    mu_ne = float(ritz[idx])
    if mu_ne >= b_sup - 1e-12 * max(1.0, abs(b_sup)):          # S:478 guard
        b_sup = b_sup + max(1.0, abs(b_sup)) * 1e-8
    nu = float(np.max(np.abs(ritz)))
    return LanczosResult(float(b_sup), mu_1, mu_ne, nu, ritz, wts)


# ----------------------------------------------------------------------------------------------
# QR (Alg. 1 line 5), Rayleigh-Ritz (line 6), residuals (line 7)
# ----------------------------------------------------------------------------------------------
def qr_locked(Y, V):
    """Q-hat <- QR([Y-hat V-hat])  (Alg. 1 line 5).  Ledger #13: the locked block Y is kept
    as is; the active block is made orthogonal to Y (two classical Gram-Schmidt passes) and then
    factored by Householder QR (deliberately a different algorithm from the GPU's CholQR2).
    The Q factor is normalised so that R has a positive real diagonal (the unique thin QR)."""
    V = np.array(V, copy=True)
    if Y is not None and Y.shape[1] > 0:
        for _ in range(2):
            V = V - Y @ (Y.conj().T @ V)
    Q, R = np.linalg.qr(V)
    d = np.diag(R)
    ph = np.where(np.abs(d) > 0, d / np.where(np.abs(d) > 0, np.abs(d), 1.0), 1.0)
    return Q * ph[None, :]


def rayleigh_ritz(H, Q):
    """(V-hat, Lambda-tilde) <- Rayleigh-Ritz(A, Q-hat)  (Alg. 1 line 6):
    G = Q^H A Q (symmetrised), G = Z Lambda Z^H, V = Q Z (back-transform).  Returns
    (ritz ascending, V, HV) with HV = (A Q) Z reused by the residuals."""
    HQ = H @ Q
    G = Q.conj().T @ HQ
    G = 0.5 * (G + G.conj().T)
    theta, Z = np.linalg.eigh(G)
    return theta, Q @ Z, HQ @ Z


def residual_norms(HV, V, theta):
    """Res(V, Lambda) = ||A v_a - lambda_a v_a||_2 per column (Alg. 1 line 7)."""
    return np.linalg.norm(HV - V * theta[None, :], axis=0)


# ----------------------------------------------------------------------------------------------
# Degrees (Alg. 1 line 12), locking (line 8), bounds (line 9), sort (line 14)
# ----------------------------------------------------------------------------------------------
def optimal_degrees(tol, res, theta, c, e, deg_max=36, extra=0):
    """m_a <- Degrees(tol, Res_a, lambda_a, c, e)  (Alg. 1 line 12).  Ledger #4:
    t_a = (c - theta_a)/e; rho_a = max |t_a +- sqrt(t_a^2 - 1)|; m_a = cap if |t_a| <= 1, else
    clamp(ceil(ln(res_a/tol)/ln rho_a), 1, cap); then rounded up to even.
    `extra` (reading 4b; "may differ in constants"): degrees added to the estimate
    before the cap -- the estimate aims exactly at tol, so a column just above tol gets m -> 1 and
    creeps (measured: 100+ iterations at res = 1.01 tol); chase_solve uses extra = 2."""
    res = np.atleast_1d(np.asarray(res, dtype=np.float64))
    theta = np.atleast_1d(np.asarray(theta, dtype=np.float64))
    cap_even = deg_max - (deg_max % 2)
    out = np.empty(res.shape, dtype=np.int64)
    for a in range(res.size):
        t = (c - theta[a]) / e
        if abs(t) <= 1.0:
            m = deg_max
        else:
            s = math.sqrt(t * t - 1.0)
            rho = max(abs(t + s), abs(t - s))
            ratio = res[a] / tol
            m = math.ceil(math.log(ratio) / math.log(rho)) if ratio > 0 else 1
            m = min(max(m, 1) + extra, deg_max)
        m = m + (m % 2)
        out[a] = min(m, cap_even) if deg_max >= 2 else m
    return out


def lock_prefix(res, tol):
    """Deflation & Locking (Alg. 1 line 8).  Ledger #15: a column locks only if
    every column with a smaller Ritz value (all earlier columns, Ritz order) also locks."""
    n = 0
    for r in np.atleast_1d(res):
        if r <= tol:
            n += 1
        else:
            break
    return n


@dataclass
class Report:
    iterations: int = 0
    locked: int = 0
    matvecs: int = 0
    b_sup: float = 0.0
    mu_1: float = 0.0
    mu_ne: float = 0.0
    nu: float = 0.0
    max_resid: float = 0.0
    trace: list = field(default_factory=list)


def chase_solve(H, nev: int, nex: int, deg: int = 20, tol: float = 1e-10, deg_max: int = 36,
                max_iter: int = 100, lanczos_steps: int = 25, lanczos_runs: int = 4, deg_extra: int = 2,
                seed_v: int = 2, seed_lanczos: int = 3, largest: bool = False, V0=None,
                lanczos_res: LanczosResult | None = None):
    """Alg. 1, serial semantics.  Returns (eigenvalues[nev] ascending,
    eigenvectors N x nev, Report).  `largest` solves on -H (ledger #17).  A real H selects the
    real-symmetric variant (the paper's setting): float64 arithmetic, real start vectors
    (the real part of the same counter-based draw)."""
    real = not np.iscomplexobj(H)
    H = np.asarray(H, dtype=np.float64 if real else np.complex128)
    if largest:
        H = -H
    N = H.shape[0]
    n_e = nev + nex
    if not (0 < nev and 0 < nex and n_e <= N and tol > 0 and deg >= 1):
        raise ValueError("invalid arguments (S:407)")
    rep = Report()
    lz = lanczos_res or lanczos(H, n_e, lanczos_steps, lanczos_runs, seed_lanczos)   # line 2
    b_sup, mu_1, mu_ne, nu = lz.b_sup, lz.mu_1, lz.mu_ne, lz.nu
    rep.b_sup, rep.nu = b_sup, nu
    if V0 is None:
        V = random_block(seed_v, 0, N, 0, n_e, STREAM_START_V)
        V = V.real.copy() if real else V
    else:
        V = np.array(V0, dtype=H.dtype)
    ritz = np.zeros(n_e)
    res = np.zeros(n_e)
    m = np.full(n_e, deg + (deg % 2), dtype=np.int64)                  # line 1 (even)
    locked = 0
    it = 0
    while locked < nev and it < max_iter:                               # line 3
        it += 1
        Va, mv = chebyshev_filter(H, V[:, locked:], m, b_sup, mu_1, mu_ne)   # line 4
        rep.matvecs += mv
        Q = qr_locked(V[:, :locked], Va)                                # line 5
        theta, Vr, HV = rayleigh_ritz(H, Q)                             # line 6
        r = residual_norms(HV, Vr, theta) / nu                          # line 7 (ledger #5)
        V[:, locked:] = Vr
        ritz[locked:] = theta
        res[locked:] = r
        nl = lock_prefix(r, tol)                                        # line 8
        locked += nl
        mu_1 = float(np.min(ritz))                                      # line 9
        mu_ne = float(np.max(ritz))
        c, e = filter_interval(b_sup, mu_ne)                            # line 10
        rep.trace.append(dict(iteration=it, locked=locked, max_resid=float(np.max(r)),
                              matvecs=mv, mu_1=mu_1, mu_ne=mu_ne))
        if locked >= nev:
            break
        act = slice(locked, n_e)
        m = optimal_degrees(tol, res[act], ritz[act], c, e, deg_max, deg_extra)   # lines 11-13
        order = np.argsort(m, kind="stable")                            # line 14
        V[:, act] = V[:, act][:, order]
        ritz[act] = ritz[act][order]
        res[act] = res[act][order]
        m = m[order]
    rep.iterations = it
    rep.locked = locked
    rep.mu_1, rep.mu_ne = mu_1, mu_ne
    k = min(locked, n_e) if locked >= nev else n_e
    lam = ritz[:k]
    order = np.argsort(lam, kind="stable")[:nev]
    vals = lam[order]
    vecs = V[:, :k][:, order]
    rep.max_resid = float(np.max(res[:k][order])) if k else 0.0
    if largest:
        vals = -vals[::-1]
        vecs = vecs[:, ::-1]
    return vals, vecs, rep
