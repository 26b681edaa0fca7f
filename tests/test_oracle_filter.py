"""Pins for the oracle's Chebyshev filter (Alg. 1 line 4; recurrence P:385-390) -- CPU.

Independent references: the Chebyshev closed form C_m(t) = cos(m arccos t) / cosh(m arccosh|t|)
evaluated in the exact G2 eigenbasis (no recurrence, no eigh), SPEC worked examples, the
Chebyshev product identity, and the scalar law on diagonal matrices."""
import numpy as np
import pytest

import oracle
from chase_gen import make_matrix


def test_C2_of_minus3_is_17(golden):
    g = golden("method_examples.json")["chebyshev_C2_of_minus3"]
    A = np.diag(np.array(g["A_diag"], dtype=complex))
    c = 0.5 * (g["upper"] + g["lower"]); e = 0.5 * (g["upper"] - g["lower"])
    mu_1 = c - e          # tau = -1 -> C_m(tau) = +-1: the damping normalisation is 1 at m = 2
    x = np.array([[1.0], [0.0]], dtype=complex)
    y, mv = oracle.chebyshev_filter(A, x, [g["degree"]], g["upper"], mu_1, g["lower"])
    np.testing.assert_allclose(y[:, 0], [g["expected_amplification"], 0.0], atol=1e-13)
    assert mv == 2


def test_degree_one_is_scaled_matvec():
    """degree 1 with c = 0, e = 1 -> output parallel to A x."""
    rng = np.random.default_rng(0)
    A = make_matrix("uniform", 40, "g2", seed=3).dense()
    x = rng.standard_normal((40, 1)) + 0j
    # b_sup = 1, mu_ne = -1 -> c = 0, e = 1
    y, _ = oracle.chebyshev_filter(A, x, [1], 1.0, -3.0, -1.0)
    Ax = A @ x
    cosang = abs(np.vdot(y[:, 0], Ax[:, 0])) / (np.linalg.norm(y) * np.linalg.norm(Ax))
    assert cosang == pytest.approx(1.0, abs=1e-14)


def test_sigma_closed_form():
    """sigma_k = C_{k-1}(tau)/C_k(tau)  (SURVEY 8(a) closed form of the scaled recurrence)."""
    b_sup, mu_1, mu_ne = 2.0, -0.7, 0.4
    c, e, coef = oracle.filter_coefficients(b_sup, mu_1, mu_ne, 36)
    tau = (mu_1 - c) / e
    T = lambda m: float(oracle.chebyshev_T(m, np.array([tau]))[0])
    sig_prev = 1.0 / tau
    assert coef[0][0] == pytest.approx(sig_prev / e, rel=1e-15)
    for k in range(2, 37):
        a, b = coef[k - 1]
        sig = a * e / 2.0
        assert sig == pytest.approx(T(k - 1) / T(k), rel=1e-12)
        assert b == pytest.approx(-sig_prev * sig, rel=1e-12)
        sig_prev = sig


def _closed_form_filter(M, V, degrees, b_sup, mu_1, mu_ne):
    """sum_k v_k C_m(t(lambda_k))/C_m(tau) v_k^H V with the generator's exact eigenvectors."""
    X = M.eigvecs(np.arange(M.n))
    c = 0.5 * (b_sup + mu_ne); e = 0.5 * (b_sup - mu_ne)
    t = (M.lam - c) / e
    tau = (mu_1 - c) / e
    out = np.empty_like(V)
    for a, m in enumerate(degrees):
        g = oracle.chebyshev_T(int(m), t) / oracle.chebyshev_T(int(m), np.array([tau]))[0]
        out[:, a] = X @ (g * (X.conj().T @ V[:, a]))
    return out


@pytest.mark.parametrize("fam", ["uniform", "121", "wilkinson"])
def test_filter_matches_closed_form(fam):
    N = 200
    M = make_matrix(fam, N, "g2", seed=11)
    H = M.dense()
    rng = np.random.default_rng(1)
    degrees = np.array([0, 1, 2, 3, 5, 8, 13, 20, 20, 36, 36, 36])
    V = rng.standard_normal((N, len(degrees))) + 1j * rng.standard_normal((N, len(degrees)))
    lam = M.lam
    b_sup = lam[-1] + 0.05 * (lam[-1] - lam[0])
    mu_1, mu_ne = lam[0], lam[29]
    Y, mv = oracle.chebyshev_filter(H, V, degrees, b_sup, mu_1, mu_ne)
    Z = _closed_form_filter(M, V, degrees, b_sup, mu_1, mu_ne)
    assert mv == degrees.sum()
    for a in range(len(degrees)):
        rel = np.linalg.norm(Y[:, a] - Z[:, a]) / np.linalg.norm(Z[:, a])
        assert rel <= 1e-11, (a, degrees[a], rel)


def test_product_identity():
    """2 C_m(tau) C_n(tau) F_m F_n = C_{m+n}(tau) F_{m+n} + C_{|m-n|}(tau) F_{|m-n|} (ledger #1)."""
    N = 120
    H = make_matrix("uniform", N, "g2", seed=2).dense()
    rng = np.random.default_rng(4)
    V = rng.standard_normal((N, 3)) + 1j * rng.standard_normal((N, 3))
    b_sup, mu_1, mu_ne = 1.05, 1e-4, 0.2
    c = 0.5 * (b_sup + mu_ne); e = 0.5 * (b_sup - mu_ne)
    tau = np.array([(mu_1 - c) / e])
    T = lambda m: oracle.chebyshev_T(m, tau)[0]
    F = lambda m, X: oracle.chebyshev_filter(H, X, [m] * X.shape[1], b_sup, mu_1, mu_ne)[0]
    m, n = 6, 4
    lhs = 2 * T(m) * T(n) * F(m, F(n, V))
    rhs = T(m + n) * F(m + n, V) + T(m - n) * F(m - n, V)
    assert np.linalg.norm(lhs - rhs) / np.linalg.norm(rhs) <= 1e-12


@pytest.mark.parametrize("m", [2, 4, 8, 16, 20])
def test_scalar_law_diagonal(m):
    """S:374 / S:612: for diagonal A, e_k is amplified by C_m(t(lambda_k))/C_m(tau)."""
    lam = np.linspace(-1.0, 3.0, 50)
    A = np.diag(lam).astype(complex)
    b_sup, mu_1, mu_ne = 3.0, -1.0, 0.5
    c = 0.5 * (b_sup + mu_ne); e = 0.5 * (b_sup - mu_ne)
    Y, _ = oracle.chebyshev_filter(A, np.eye(50, dtype=complex), [m] * 50, b_sup, mu_1, mu_ne)
    expect = oracle.chebyshev_T(m, (lam - c) / e) / oracle.chebyshev_T(m, np.array([(mu_1 - c) / e]))[0]
    np.testing.assert_allclose(np.diag(Y).real, expect, rtol=1e-10, atol=1e-14)
    assert np.max(np.abs(Y - np.diag(np.diag(Y)))) == 0.0


def test_bounded_inside_interval():
    """an eigenvector inside [mu_ne, b_sup] is not amplified (|C_m(t)| <= 1, |t| <= 1)."""
    lam = np.linspace(0.0, 1.0, 30)
    A = np.diag(lam).astype(complex)
    Y, _ = oracle.chebyshev_filter(A, np.eye(30, dtype=complex)[:, 20:], [20] * 10, 1.0, 0.0, 0.5)
    assert np.max(np.abs(Y)) <= 1.0 + 1e-14


def test_hemm_step_definition_and_shift():
    rng = np.random.default_rng(3)
    H = make_matrix("uniform", 30, "g2", seed=4).dense()
    X = rng.standard_normal((30, 4)) + 1j * rng.standard_normal((30, 4))
    Y = rng.standard_normal((30, 4)) + 1j * rng.standard_normal((30, 4))
    out = oracle.hemm_step(H, X, Y, 0.7, -0.3, 0.25)
    ref = 0.7 * ((H - 0.25 * np.eye(30)) @ X) - 0.3 * Y
    np.testing.assert_allclose(out, ref, rtol=1e-14, atol=1e-14)
