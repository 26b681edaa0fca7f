"""Pins for the seeded input generators (chase_gen) -- CPU only.

The generator is the source of every input and of the exact spectra/eigenvectors the oracle and
the CUDA path are pinned to, so it is itself pinned to the paper (Table 1; kappa
values P:765) and to brute force (Jacobi, Sturm bisection)."""
import numpy as np
import pytest

from chase_gen import spectra, make_matrix, G2Matrix, block_partition
from _jacobi import jacobi_eigvalsh


def test_table1_worked_examples(golden):
    g = golden("table1_examples.json")
    np.testing.assert_allclose(spectra.uniform(3, 1.0, 0.1), g["uniform_n3_dmax1_eps0.1"]["values"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(spectra.geometric(3, 1.0, 0.25), g["geometric_n3_dmax1_eps0.25"]["values"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(spectra.one_two_one(3), g["one_two_one_n3"]["values"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(spectra.wilkinson(3), g["wilkinson_n3"]["values"], rtol=0, atol=1e-13)
    d, e = spectra.tridiagonal("121", 3)
    np.testing.assert_array_equal(np.diag(d) + np.diag(e, 1) + np.diag(e, -1), g["one_two_one_tridiag_n3"]["matrix"])
    d, e = spectra.tridiagonal("wilkinson", 3)
    np.testing.assert_array_equal(np.diag(d) + np.diag(e, 1) + np.diag(e, -1), g["wilkinson_tridiag_n3"]["matrix"])


def test_condition_numbers_match_paper(golden):
    """kappa of 1-2-1 / Geo / Uni / Wilk at n = 20k are 1.6e8 / 1.0e4 / 1.0e4 / 4.7e4.
    This pins ledger readings #8 (Wilkinson diagonal |i-(n-1)/2|), #9 and #10 (d_max=1, eps=1e-4)."""
    g = golden("table1_examples.json")["condition_numbers_n20000"]
    n = 20000
    for fam in ("121", "geometric", "uniform", "wilkinson"):
        lam = spectra.spectrum(fam, n)
        kappa = np.max(np.abs(lam)) / np.min(np.abs(lam))
        assert float(f"{kappa:.1e}") == pytest.approx(g[fam], rel=1e-12), (fam, kappa)


def test_wilkinson_properties():
    """'All positive, but one, roughly in pairs'; LAPACK path == Sturm bisection."""
    for n in (301, 1000):
        lam = spectra.wilkinson(n)
        assert np.sum(lam < 0) == 1
    d, e = spectra.tridiagonal("wilkinson", 701)
    from scipy.linalg import eigvalsh_tridiagonal
    np.testing.assert_allclose(np.sort(spectra.sturm_bisection(d, e)), eigvalsh_tridiagonal(d, e), atol=1e-12)


def test_one_two_one_closed_form_vs_bruteforce():
    n = 40
    d, e = spectra.tridiagonal("121", n)
    T = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    np.testing.assert_allclose(jacobi_eigvalsh(T), spectra.one_two_one(n), atol=1e-13)


@pytest.mark.parametrize("kind", ["g1", "g2"])
@pytest.mark.parametrize("fam", ["uniform", "geometric", "121", "wilkinson"])
def test_dense_generator_spectrum_bruteforce(kind, fam):
    """Spectral fidelity of the densified matrix against a brute-force Jacobi (no LAPACK)."""
    M = make_matrix(fam, 24, kind, seed=5)
    H = M.dense()
    assert np.max(np.abs(H - H.conj().T)) <= 1e-15 * np.max(np.abs(M.lam))
    np.testing.assert_allclose(jacobi_eigvalsh(H), M.lam, atol=1e-13 * np.max(np.abs(M.lam)))


@pytest.mark.parametrize("kind", ["g1", "g2"])
def test_dense_generator_exact_eigenvectors(kind):
    M = make_matrix("uniform", 257, kind, seed=9)
    H = M.dense()
    idx = np.arange(0, 257, 16)
    X = M.eigvecs(idx)
    R = H @ X - X * M.lam[idx][None, :]
    assert np.max(np.linalg.norm(R, axis=0)) <= 1e-13
    np.testing.assert_allclose(X.conj().T @ X, np.eye(len(idx)), atol=1e-13)


def test_g2_block_consistency_and_determinism():
    M = make_matrix("geometric", 101, "g2", seed=7)
    H = M.dense()
    np.testing.assert_array_equal(M.block(10, 30, 40, 25), H[10:40, 40:65])
    M2 = make_matrix("geometric", 101, "g2", seed=7)
    np.testing.assert_array_equal(M2.dense(), H)
    M3 = make_matrix("geometric", 101, "g2", seed=8)
    assert np.max(np.abs(M3.dense() - H)) > 1e-3


def test_g2_entries_are_dense_and_delocalised():
    """G2 entries have Haar-like magnitude statistics (median |h_ij| sqrt(N)/||H|| ~ 0.38)."""
    M = make_matrix("uniform", 512, "g2", seed=1)
    H = M.dense()
    med = np.median(np.abs(H)) * np.sqrt(512) / np.max(np.abs(M.lam))
    assert 0.2 < med < 0.6


def test_block_partition_remainder_rule():
    """Ledger #19: first (n mod parts) blocks get one extra row."""
    assert block_partition(10, 3) == [(0, 4), (4, 3), (7, 3)]
    assert block_partition(9, 3) == [(0, 3), (3, 3), (6, 3)]
    parts = block_partition(1001, 4)
    assert sum(l for _, l in parts) == 1001 and parts[-1][0] + parts[-1][1] == 1001


@pytest.mark.parametrize("kind", ["r1", "r2"])
@pytest.mark.parametrize("fam", ["uniform", "121", "wilkinson"])
def test_real_generators_spectrum_and_eigenvectors(kind, fam):
    """Real-symmetric inputs (f2): symmetric, exact spectrum (brute-force Jacobi), exact eigenvectors."""
    M = make_matrix(fam, 40, kind, seed=6)
    H = M.dense()
    assert H.dtype == np.float64 and np.max(np.abs(H - H.T)) <= 1e-15 * np.max(np.abs(M.lam))
    np.testing.assert_allclose(jacobi_eigvalsh(H), M.lam, atol=1e-13 * np.max(np.abs(M.lam)))
    idx = np.arange(0, 40, 3)
    X = M.eigvecs(idx)
    assert np.max(np.linalg.norm(H @ X - X * M.lam[idx][None, :], axis=0)) <= 1e-13 * np.max(np.abs(M.lam))
    np.testing.assert_allclose(X.T @ X, np.eye(len(idx)), atol=1e-13)
