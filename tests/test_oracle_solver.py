"""Pins for the oracle's Alg. 1 pieces and the whole solve -- CPU only.

References independent of the oracle: Table 1 exact spectra, exact G2 eigenvectors, brute-force
Jacobi, SPEC worked examples (degrees, locking, Lanczos, Rayleigh-Ritz), Weyl/Davis-Kahan
bounds, and mathematical invariants (orthonormality, containment, determinism)."""
import numpy as np
import pytest

import oracle
from chase_gen import make_matrix
from _jacobi import jacobi_eigvalsh


def test_degrees_worked_examples(golden):
    g = golden("method_examples.json")["degrees"]
    tol = 1e-10
    e = 1.0
    for case in g["cases"]:
        theta = 0.0
        c = theta + case["t"] * e          # t = (c - theta)/e
        m = oracle.optimal_degrees(tol, [case["res_over_tol"] * tol], [theta], c, e, 36)
        assert int(m[0]) == case["even"], case


def test_degrees_monotone():
    """non-increasing in rho, non-decreasing in res/tol (random valid inputs)."""
    rng = np.random.default_rng(0)
    tol = 1e-10
    for _ in range(200):
        t1, t2 = np.sort(rng.uniform(1.001, 50.0, 2))
        r = 10 ** rng.uniform(-9, 0)
        m1 = oracle.optimal_degrees(tol, [r], [0.0], t1, 1.0)[0]
        m2 = oracle.optimal_degrees(tol, [r], [0.0], t2, 1.0)[0]
        assert m2 <= m1
        r2 = r * 10 ** rng.uniform(0, 3)
        assert oracle.optimal_degrees(tol, [r2], [0.0], t1, 1.0)[0] >= m1


def test_locking_prefix(golden):
    g = golden("method_examples.json")["locking_prefix"]
    assert oracle.lock_prefix(g["res"], g["tol"]) == g["locked"]
    assert oracle.lock_prefix([1e-3, 1e-12], 1e-10) == 0
    assert oracle.lock_prefix([1e-12] * 5, 1e-10) == 5


def test_lanczos_full_krylov(golden):
    g = golden("method_examples.json")["lanczos_full_krylov"]
    A = np.diag(np.array(g["A_diag"], dtype=complex))
    lz = oracle.lanczos(A, 3, steps=g["steps"], runs=4, seed=3)
    np.testing.assert_allclose(np.unique(np.round(lz.ritz, 8)), g["ritz"], atol=1e-8)
    assert lz.b_sup >= 10.0 - 1e-12
    assert lz.mu_1 == pytest.approx(1.0, abs=1e-10)


@pytest.mark.parametrize("n_e", [1, 3, 5, 7, 9])
def test_lanczos_dos_quantile_uniform_weights(n_e):
    """mu_ne pin (ledger #14): full Krylov on diag(1..10) from all-ones start vectors.
    Every eigenvector carries the same share 1/N of the start vector, so the Ritz values are the
    exact eigenvalues, each DoS weight is exactly 1/(N L), the CDF after the L copies of lambda_k is
    k/N, and the n_e/N quantile is lambda_{n_e} = n_e.  b_sup = lambda_max + |beta_m| = 10."""
    N, L = 10, 4
    A = np.diag(np.arange(1.0, N + 1.0)).astype(complex)
    lz = oracle.lanczos(A, n_e, steps=N, runs=L, start=np.ones((N, L), dtype=complex))
    assert lz.mu_ne == pytest.approx(float(n_e), abs=1e-10)
    assert lz.mu_1 == pytest.approx(1.0, abs=1e-10)
    assert lz.b_sup == pytest.approx(10.0, abs=1e-8)
    np.testing.assert_allclose(lz.weights, 1.0 / (N * L), atol=1e-13)


@pytest.mark.parametrize("rotated", [False, True])
@pytest.mark.parametrize("n_e,expect", [(1, 3), (2, 5), (3, 6), (5, 7), (8, 9)])
def test_lanczos_dos_quantile_weighted_start(rotated, n_e, expect):
    """mu_ne pin with unequal weights: start vector s = Q (sqrt(k))_k on H = Q diag(1..10) Q^H.
    Full Krylov makes the Ritz values exact and the weight of lambda_k equal to k / sum(k) = k/55,
    so CDF(k) = k(k+1)/110 and mu_ne = smallest k with k(k+1)/110 >= n_e/10, worked by hand:
    n_e = 1 -> 3 (12/110 >= 0.1 > 6/110), 2 -> 5 (30/110 >= 0.2 > 20/110), 3 -> 6 (42/110 >= 0.3),
    5 -> 7 (56/110 >= 0.5 > 42/110), 8 -> 9 (90/110 >= 0.8 > 72/110).
    The rotated case (Haar Q) catches a conjugation / transposition slip in the weights."""
    N, L = 10, 2
    lam = np.arange(1.0, N + 1.0)
    Q = np.eye(N, dtype=complex)
    if rotated:
        rng = np.random.default_rng(7)
        Q, R = np.linalg.qr(rng.standard_normal((N, N)) + 1j * rng.standard_normal((N, N)))
    A = (Q * lam[None, :]) @ Q.conj().T
    s = Q @ np.sqrt(lam).astype(complex)
    lz = oracle.lanczos(A, n_e, steps=N, runs=L, start=np.stack([s, 2.5 * s], axis=1))
    assert lz.mu_ne == pytest.approx(float(expect), abs=1e-9)
    for k in range(1, N + 1):      # each eigenvalue's pooled weight: L copies of k/55 / L
        assert np.sum(lz.weights[np.abs(lz.ritz - k) < 1e-6]) == pytest.approx(k / 55.0, abs=1e-12)


@pytest.mark.parametrize("fam", ["uniform", "geometric", "121", "wilkinson"])
def test_lanczos_bounds_bracket_spectrum(fam):
    """b_sup >= lambda_max (else the filter amplifies the unwanted end) and mu_1 >= lambda_1."""
    M = make_matrix(fam, 500, "g2", seed=2)
    lz = oracle.lanczos(M.dense(), 60)
    assert lz.b_sup >= M.lam[-1]
    assert lz.mu_1 >= M.lam[0] - 1e-12
    assert lz.nu <= np.max(np.abs(M.lam)) + 1e-12


def test_rr_invariant_subspace(golden):
    g = golden("method_examples.json")["rr_invariant_subspace"]
    A = np.diag(np.array(g["A_diag"], dtype=complex))
    Q = np.eye(4, dtype=complex)[:, g["Q_columns"]]
    theta, V, HV = oracle.rayleigh_ritz(A, Q)
    np.testing.assert_allclose(theta, g["ritz"], atol=1e-15)
    assert np.max(oracle.residual_norms(HV, V, theta)) <= 1e-15


def test_rr_containment_and_exact_subspace():
    M = make_matrix("wilkinson", 50, "g2", seed=3)
    H = M.dense()
    rng = np.random.default_rng(1)
    Q, _ = np.linalg.qr(rng.standard_normal((50, 8)) + 1j * rng.standard_normal((50, 8)))
    theta, _, _ = oracle.rayleigh_ritz(H, Q)
    assert theta[0] >= M.lam[0] - 1e-12 and theta[-1] <= M.lam[-1] + 1e-12
    X = M.eigvecs([3, 7, 11])
    theta, V, HV = oracle.rayleigh_ritz(H, X)
    np.testing.assert_allclose(theta, M.lam[[3, 7, 11]], atol=1e-13)
    assert np.max(oracle.residual_norms(HV, V, theta)) <= 1e-12 * np.linalg.norm(H)


def test_residual_examples():
    A = np.diag([3.0, 1.0, 2.0]).astype(complex)
    v = np.array([[1.0], [0.0], [0.0]], dtype=complex)
    assert oracle.residual_norms(A @ v, v, np.array([0.0]))[0] == pytest.approx(3.0)
    assert oracle.residual_norms(A @ v, v, np.array([3.0]))[0] == 0.0


def test_qr_locked_properties():
    rng = np.random.default_rng(5)
    Y, _ = np.linalg.qr(rng.standard_normal((80, 5)) + 1j * rng.standard_normal((80, 5)))
    V = rng.standard_normal((80, 9)) + 1j * rng.standard_normal((80, 9))
    Q = oracle.qr_locked(Y, V)
    B = np.concatenate([Y, Q], axis=1)
    np.testing.assert_allclose(B.conj().T @ B, np.eye(14), atol=1e-13)
    # span([Y V]) preserved: V lies in span([Y Q])
    P = B @ (B.conj().T @ V)
    assert np.linalg.norm(P - V) <= 1e-12 * np.linalg.norm(V)
    # unique thin QR: R = Q^H (V - Y Y^H V) is upper triangular with positive diagonal
    R = Q.conj().T @ (V - Y @ (Y.conj().T @ V))
    assert np.max(np.abs(np.tril(R, -1))) <= 1e-12
    assert np.all(np.diag(R).real > 0) and np.max(np.abs(np.diag(R).imag)) <= 1e-12


def _check_solution(M, vals, vecs, rep, nev, tol, H):
    normH = np.max(np.abs(M.lam))
    assert rep.locked >= nev
    assert np.max(np.abs(vals - M.lam[:nev])) <= 1e-10 * normH           # ledger #6
    R = H @ vecs - vecs * vals[None, :]
    assert np.max(np.linalg.norm(R, axis=0)) <= tol * normH              # ledger #5
    np.testing.assert_allclose(vecs.conj().T @ vecs, np.eye(nev), atol=1e-12)
    locked_trace = [t["locked"] for t in rep.trace]
    assert locked_trace == sorted(locked_trace)                          # monotone locking


@pytest.mark.parametrize("fam,max_iter", [("uniform", 100), ("121", 100), ("wilkinson", 100), ("geometric", 400)])
def test_solve_n301_all_families(fam, max_iter):
    """S:609 analogue (complexified): n = 301, nev = 30, nex = 10, tol = 1e-10, vs exact spectrum."""
    M = make_matrix(fam, 301, "g2", seed=1)
    H = M.dense()
    vals, vecs, rep = oracle.chase_solve(H, 30, 10, tol=1e-10, max_iter=max_iter)
    _check_solution(M, vals, vecs, rep, 30, 1e-10, H)
    # brute force on the returned Ritz values: Jacobi on the projected matrix
    G = vecs.conj().T @ H @ vecs
    np.testing.assert_allclose(jacobi_eigvalsh(G), vals, atol=1e-12)


def test_solve_config1_uniform_g1():
    """BASELINE config 1: N=1000 Uniform (G1, the paper's Q^T D Q), nev=50, nex=25, tol=1e-10."""
    M = make_matrix("uniform", 1000, "g1", seed=1)
    H = M.dense()
    vals, vecs, rep = oracle.chase_solve(H, 50, 25, tol=1e-10)
    _check_solution(M, vals, vecs, rep, 50, 1e-10, H)
    # exact eigenvectors: subspace angles for isolated eigenvalues (ledger #7, Davis-Kahan)
    X = M.eigvecs(np.arange(50))
    s = np.linalg.svd(X.conj().T @ vecs, compute_uv=False)
    gap = M.lam[50] - M.lam[49]
    bound = 10 * 1e-10 / gap
    assert np.sqrt(max(0.0, 1 - s.min() ** 2)) <= max(1e-8, bound)


def test_solve_121_n1000_spec_acceptance():
    """OneTwoOne n=1000, nev=50, nex=20 -> lambda_k = 2-2cos(pi k/1001) to 1e-8."""
    M = make_matrix("121", 1000, "g2", seed=3)
    vals, _, rep = oracle.chase_solve(M.dense(), 50, 20, tol=1e-10)
    k = np.arange(1, 51)
    np.testing.assert_allclose(vals, 2 - 2 * np.cos(np.pi * k / 1001), atol=1e-8)


def test_one_iteration_matvecs(golden):
    """P:727-731 one-subspace-iteration protocol: matvecs = deg * (nev+nex)."""
    g = golden("method_examples.json")["matvec_one_iteration"]
    M = make_matrix("uniform", 400, "g2", seed=1)
    _, _, rep = oracle.chase_solve(M.dense(), g["nev"], g["nex"], deg=g["deg"], max_iter=1)
    assert rep.iterations == 1 and rep.matvecs == g["matvecs"]


def test_determinism_and_largest():
    M = make_matrix("wilkinson", 201, "g2", seed=4)
    H = M.dense()
    v1, _, r1 = oracle.chase_solve(H, 10, 6)
    v2, _, r2 = oracle.chase_solve(H, 10, 6)
    np.testing.assert_array_equal(v1, v2)
    assert (r1.iterations, r1.matvecs) == (r2.iterations, r2.matvecs)
    vl, _, _ = oracle.chase_solve(H, 5, 5, largest=True)
    np.testing.assert_allclose(vl, M.lam[-5:], atol=1e-10 * np.max(np.abs(M.lam)))


def test_invalid_arguments():
    H = np.eye(10, dtype=complex)
    with pytest.raises(ValueError):
        oracle.chase_solve(H, 8, 5)
    with pytest.raises(ValueError):
        oracle.chase_solve(H, 0, 5)


@pytest.mark.parametrize("fam,kind", [("uniform", "r1"), ("121", "r2"), ("wilkinson", "r2")])
def test_solve_real_symmetric(fam, kind):
    """Real-symmetric variant (f2; the paper's experimental field): float64 throughout."""
    M = make_matrix(fam, 301, kind, seed=2)
    H = M.dense()
    vals, vecs, rep = oracle.chase_solve(H, 30, 10, tol=1e-10)
    assert vecs.dtype == np.float64
    _check_solution(M, vals, vecs, rep, 30, 1e-10, H)


def test_degrees_extra_margin_hand_values():
    """Reading 4b: `extra` degrees are added to the estimate before the cap and the
    even rounding.  t = 1.5: rho = 1.5 + sqrt(1.25) = 2.618...; res/tol = 1e3 -> ln 1e3 / ln rho =
    7.18 -> 8 (+2 -> 10); res/tol = 1.01 -> 0.0103 -> 1 -> even 2 (+2 -> 3 -> even 4); the cap
    still binds (res/tol = 1e30 -> 72 -> cap 36)."""
    tol, e = 1e-10, 1.0
    c = 1.5                      # theta = 0 -> t = 1.5
    for ratio, base, plus2 in ((1e3, 8, 10), (1.01, 2, 4), (1e30, 36, 36)):
        assert int(oracle.optimal_degrees(tol, [ratio * tol], [0.0], c, e, 36)[0]) == base
        assert int(oracle.optimal_degrees(tol, [ratio * tol], [0.0], c, e, 36, extra=2)[0]) == plus2
