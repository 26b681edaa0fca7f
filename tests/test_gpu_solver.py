"""GPU parity of the rest of the iteration and of the full chase_solve
(Alg. 1) through the C ABI, against the CPU oracle and the exact spectra/eigenvectors of the
generator.  Tolerances: north_star (eigenvalues 1e-10 relative to ||H||_2, ledger #6; residual
||Hv - lambda v||/||H|| <= 1e-10; orthonormality 1e-12)."""
import numpy as np
import pytest

import oracle
from chase_gen import make_matrix

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _dev(a):
    return torch.from_numpy(np.asfortranarray(a)).t().contiguous().t().cuda()


@pytest.fixture(scope="module")
def lib():
    import paper_2205_02491_b200 as pkg
    return pkg


def _check(M, H, vals, vecs, nev, tol=1e-10):
    normH = np.max(np.abs(M.lam))
    assert np.max(np.abs(vals - M.lam[:nev])) <= 1e-10 * normH
    R = H @ vecs - vecs * vals[None, :]
    assert np.max(np.linalg.norm(R, axis=0)) <= tol * normH
    np.testing.assert_allclose(vecs.conj().T @ vecs, np.eye(nev), atol=1e-12)


@pytest.mark.parametrize("fam", ["uniform", "wilkinson"])
def test_lanczos_matches_oracle(lib, fam):
    N, n_e = 700, 60
    M = make_matrix(fam, N, "g2", seed=4)
    H = M.dense()
    ch = lib.Chase(N, 40, 20)
    b_sup, mu_1, mu_ne, nu = ch.lanczos(_dev(H), n_e)
    lz = oracle.lanczos(H, n_e)
    scale = np.max(np.abs(M.lam))
    assert abs(b_sup - lz.b_sup) <= 1e-10 * scale
    assert abs(mu_1 - lz.mu_1) <= 1e-10 * scale
    assert abs(mu_ne - lz.mu_ne) <= 1e-10 * scale
    assert abs(nu - lz.nu) <= 1e-10 * scale
    assert b_sup >= M.lam[-1] and mu_1 >= M.lam[0] - 1e-12


def test_solve_config1_vs_oracle(lib):
    """BASELINE config 1: N=1000 complex double Uniform (G1), nev=50, nex=25, deg=20, tol=1e-10."""
    N, nev, nex = 1000, 50, 25
    M = make_matrix("uniform", N, "g1", seed=1)
    H = M.dense()
    ch = lib.Chase(N, nev, nex)
    vals, dvecs, rep, st = ch.solve(_dev(H), nev, nex, deg=20, tol=1e-10)
    assert st == 0, ch.last_error()
    vecs = dvecs.cpu().numpy()[:, :nev]
    _check(M, H, vals, vecs, nev)
    ov, ovec, orep = oracle.chase_solve(H, nev, nex, deg=20, tol=1e-10)
    assert np.max(np.abs(vals - ov)) <= 1e-10 * np.max(np.abs(M.lam))
    assert abs(rep["iterations"] - orep.iterations) <= 1          # tracked, +-1 allowed
    # subspace angle against the exact eigenvectors (ledger #7)
    X = M.eigvecs(np.arange(nev))
    s = np.linalg.svd(X.conj().T @ vecs, compute_uv=False)
    assert np.sqrt(max(0.0, 1 - s.min() ** 2)) <= max(1e-8, 10 * 1e-10 / (M.lam[nev] - M.lam[nev - 1]))
    assert rep["matvecs"] > 0 and rep["t_filter"] > 0 and rep["locked"] >= nev


@pytest.mark.parametrize("fam,max_iter", [("121", 100), ("wilkinson", 100), ("geometric", 400)])
def test_solve_families_n301(lib, fam, max_iter):
    N, nev, nex = 301, 30, 10
    M = make_matrix(fam, N, "g2", seed=1)
    H = M.dense()
    ch = lib.Chase(N, nev, nex)
    ch.set_option("max_iter", max_iter)
    vals, dvecs, rep, st = ch.solve(_dev(H), nev, nex, deg=20, tol=1e-10)
    assert st == 0, ch.last_error()
    _check(M, H, vals, dvecs.cpu().numpy()[:, :nev], nev)


def test_solve_one_iteration_protocol_and_maxiter(lib):
    """one subspace iteration -> matvecs = deg * (nev+nex); status CHASE_E_MAXITER."""
    N, nev, nex = 400, 50, 25
    M = make_matrix("uniform", N, "g2", seed=1)
    ch = lib.Chase(N, nev, nex)
    ch.set_option("max_iter", 1)
    vals, _, rep, st = ch.solve(_dev(M.dense()), nev, nex, deg=20)
    assert st == 8 and rep["iterations"] == 1 and rep["matvecs"] == 20 * (nev + nex)
    _, _, orep = oracle.chase_solve(M.dense(), nev, nex, deg=20, max_iter=1)
    assert rep["locked"] == orep.locked


def test_solve_largest_and_determinism(lib):
    N = 500
    M = make_matrix("wilkinson", N, "g2", seed=2)
    H = _dev(M.dense())
    ch = lib.Chase(N, 10, 10)
    v1, _, r1, _ = ch.solve(H, 10, 10)
    v2, _, r2, _ = ch.solve(H, 10, 10)
    assert np.array_equal(v1, v2) and r1["iterations"] == r2["iterations"] and r1["matvecs"] == r2["matvecs"]
    ch.set_option("largest", 1)
    vl, _, _, st = ch.solve(H, 10, 10)
    assert st == 0
    np.testing.assert_allclose(vl, M.lam[-10:], atol=1e-10 * np.max(np.abs(M.lam)))


def test_solve_rejects_bad_arguments(lib):
    N = 100
    ch = lib.Chase(N, 10, 5)
    H = _dev(np.eye(N, dtype=complex))
    with pytest.raises(lib.ChaseError):
        ch.solve(H, 20, 5)          # exceeds nev_max + nex_max
    with pytest.raises(lib.ChaseError):
        ch.solve(H, 5, 5, tol=-1.0)


def test_warm_start_sequence(lib):
    """Sequences of correlated eigenproblems: solve H1 cold, then
    H2 = H1 + small Hermitian perturbation warm-started (approx=1) from H1's Ritz vectors.  The warm
    solve must match the oracle's cold solve of H2 and need fewer iterations than a cold solve."""
    N, nev, nex = 600, 40, 20
    M = make_matrix("uniform", N, "g2", seed=21)
    H1 = M.dense()
    rng = np.random.default_rng(5)
    E = rng.standard_normal((N, N)) + 1j * rng.standard_normal((N, N))
    H2 = H1 + 1e-8 * (E + E.conj().T) / np.sqrt(N)
    ch = lib.Chase(N, nev, nex)
    vec = torch.zeros((nev + nex, N), dtype=torch.complex128, device="cuda").t()
    v1, vec, r1, st = ch.solve(_dev(H1), nev, nex, vectors=vec)
    assert st == 0
    vec[:, nev:] = torch.from_numpy(np.asfortranarray(oracle.random_block(7, 0, N, 0, nex, 0))).cuda()
    _, _, rc, _ = ch.solve(_dev(H2), nev, nex)                      # cold reference on the device
    ch.set_option("approx", 1)
    v2, vec2, rw, st = ch.solve(_dev(H2), nev, nex, vectors=vec)
    assert st == 0
    ov, _, _ = oracle.chase_solve(H2, nev, nex)
    assert np.max(np.abs(v2 - ov)) <= 1e-10 * np.max(np.abs(M.lam)) * 1.01
    assert rw["matvecs"] < rc["matvecs"] and rw["iterations"] <= rc["iterations"], \
        (rw["iterations"], rc["iterations"], rw["matvecs"], rc["matvecs"])


def test_subspace_angle_north_star(lib):
    """north_star: subspace angle <= 1e-8 (ledger #7).  Davis-Kahan: sin angle(V_k, X_k) <=
    ||R_k||_F / delta_k (delta_k = lambda_{k+1} - theta_k gap to the excluded spectrum), so 1e-8 is
    asserted on the leading k* columns where 10 x that bound (post-hoc FP64 residuals of the
    returned vectors, ||R_k||_2 of the block) is <= 1e-8; config-1 shape (eigenvalue gaps ~1e-3
    ||H||), tol 1e-13 so that the bound reaches 1e-8 (at tol 1e-10 it cannot: 10 x 1e-10 / 1e-3)."""
    N, nev, nex = 1000, 50, 25
    M = make_matrix("uniform", N, "g1", seed=1)
    H = M.dense()
    ch = lib.Chase(N, nev, nex)
    vals, dvecs, rep, st = ch.solve(_dev(H), nev, nex, deg=20, tol=1e-13)
    assert st == 0, ch.last_error()
    V = dvecs.cpu().numpy()[:, :nev]
    R = H @ V - V * vals[None, :]
    X = M.eigvecs(np.arange(nev))
    kstar = 0
    for k in range(1, nev + 1):
        delta = M.lam[k] - vals[k - 1]
        if delta > 0 and 10 * np.linalg.norm(R[:, :k], 2) / delta <= 1e-8:
            kstar = k
    assert kstar >= nev // 2, (kstar, np.linalg.norm(R, 2))
    Vk, Xk = V[:, :kstar], X[:, :kstar]
    # sin of the largest principal angle = ||(I - X X^H) V||_2 (no 1 - cos^2 cancellation)
    angle = np.linalg.norm(Vk - Xk @ (Xk.conj().T @ Vk), 2)
    assert angle <= 1e-8, (kstar, angle)


@pytest.mark.parametrize("pinned", [True, False])
def test_solve_from_host_buffers(lib, pinned):
    """chase_solve with H and the eigenvector buffer in host memory (pinned or pageable): the call
    stages them through device copies and returns the same bits as the device-resident solve."""
    N, nev, nex = 600, 30, 15
    M = make_matrix("uniform", N, "g2", seed=5)
    H = M.dense()
    ch = lib.Chase(N, nev, nex)
    vals_d, vec_d, rep_d, st = ch.solve(_dev(H), nev, nex, deg=20, tol=1e-10)
    assert st == 0
    Hh = torch.empty((N, N), dtype=torch.complex128, pin_memory=pinned).t()     # column-major
    Hh.copy_(torch.from_numpy(H))
    vh = torch.zeros((nev, N), dtype=torch.complex128, pin_memory=pinned).t()
    assert not Hh.is_cuda and not vh.is_cuda and Hh.is_pinned() == pinned
    vals_h, _, rep_h, st = ch.solve(Hh, nev, nex, deg=20, tol=1e-10, vectors=vh)
    assert st == 0
    assert np.array_equal(vals_h, vals_d) and rep_h["iterations"] == rep_d["iterations"]
    assert np.array_equal(vh.numpy(), vec_d.cpu().numpy()[:, :nev])


@pytest.mark.parametrize("dtype", ["c128", "r64"])
def test_solve_wide_block(lib, dtype):
    """nev + nex = 328 (six 64-blocks and a ragged tail): the recursive triangular inverse of
    CholQR, the block-Jacobi Rayleigh-Ritz and locking at a block width the small cases do not
    reach, against the exact spectrum."""
    N, nev, nex = 1400, 220, 108
    M = make_matrix("uniform", N, "r2" if dtype == "r64" else "g2", seed=21)
    H = M.dense()
    ch = lib.Chase(N, nev, nex, dtype=dtype)
    vals, dvecs, rep, st = ch.solve(_dev(H), nev, nex, deg=20, tol=1e-10)
    assert st == 0, ch.last_error()
    _check(M, H, vals, dvecs.cpu().numpy()[:, :nev], nev)
