"""GPU parity of the complex-single filter path (SURVEY §8 a2/a4 "c64 uses tcgen05 kind::tf32, 3xTF32
split for FP32 accuracy, with FP32 accumulation") through the C ABI (dtype CHASE_C64) against the
oracle (complex128 arithmetic on the same complex64-rounded inputs).  Tolerances:
a fused step is a length-K dot product in ~FP32 accuracy (3xTF32 + FP32 accumulation), so its
relative Frobenius error is ~ sqrt(K) 2^-24; 1xTF32 would sit near 2^-11 -- the 1e-5 bar separates
the two (1e-5 per step, 1e-4 for the full filter)."""
import numpy as np
import pytest

import oracle
from chase_gen import make_matrix

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _dev(a):
    return torch.from_numpy(np.asfortranarray(a.astype(np.complex64))).t().contiguous().t().cuda()


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def lib():
    import paper_2205_02491_b200 as pkg
    return pkg


@pytest.mark.parametrize("N,ncols", [(1000, 75), (512, 64), (1200, 130), (256, 7)])
@pytest.mark.parametrize("direction", [0, 1])
def test_c64_hemm_step(lib, N, ncols, direction):
    H = make_matrix("uniform", N, "g2", seed=N).dense().astype(np.complex64)
    rng = np.random.default_rng(N + ncols)
    X = (rng.standard_normal((N, ncols)) + 1j * rng.standard_normal((N, ncols))).astype(np.complex64)
    Y0 = (rng.standard_normal((N, ncols)) + 1j * rng.standard_normal((N, ncols))).astype(np.complex64)
    ch = lib.Chase(N, max(ncols, 2) - 1, 1, dtype="c64")
    dY = _dev(Y0)
    ch.hemm_step(direction, _dev(H), _dev(X), dY, ncols, 0.37, -0.81, 0.55)
    ref = oracle.hemm_step(H.astype(np.complex128), X.astype(np.complex128), Y0.astype(np.complex128), 0.37, -0.81, 0.55)
    err = _rel(dY.cpu().numpy().astype(np.complex128), ref)
    print("c64 step", N, ncols, direction, err)
    assert err <= 1e-5, err


def test_c64_filter_vs_oracle(lib):
    N = 1000
    M = make_matrix("uniform", N, "g2", seed=7)
    H = M.dense().astype(np.complex64)
    degrees = np.sort(np.array([0, 2, 4, 8, 14, 20, 20, 36] + [20] * 60))
    n = len(degrees)
    rng = np.random.default_rng(1)
    V = (rng.standard_normal((N, n)) + 1j * rng.standard_normal((N, n))).astype(np.complex64)
    b_sup, mu_1, mu_ne = M.lam[-1] * 1.02, M.lam[0], M.lam[n]
    ch = lib.Chase(N, n - 5, 5, dtype="c64")
    dV = _dev(V)
    dW = torch.zeros((n, N), dtype=torch.complex64, device="cuda").t()
    mv = ch.filter(_dev(H), dV, dW, degrees, b_sup, mu_1, mu_ne)
    ref, mv_ref = oracle.chebyshev_filter(H.astype(np.complex128), V.astype(np.complex128), degrees, b_sup, mu_1, mu_ne)
    assert mv == mv_ref
    out = dV.cpu().numpy().astype(np.complex128)
    errs = [_rel(out[:, a], ref[:, a]) for a in range(n)]
    assert max(errs) <= 1e-4, max(errs)


@pytest.mark.parametrize("grid", [(1, 2), (2, 2), (2, 1)])
def test_c64_emulated_grid_step(lib, grid):
    """Shift only on the intersection rows I_ij, row offsets inside the shard, partial sums."""
    r, c = grid
    N, n = 504, 19
    H = make_matrix("wilkinson", N, "g2", seed=5).dense().astype(np.complex64)
    rng = np.random.default_rng(2)
    X = (rng.standard_normal((N, n)) + 1j * rng.standard_normal((N, n))).astype(np.complex64)
    Y0 = (rng.standard_normal((N, n)) + 1j * rng.standard_normal((N, n))).astype(np.complex64)
    ref = oracle.hemm_step(H.astype(np.complex128), X.astype(np.complex128), Y0.astype(np.complex128), 1.3, -0.4, 0.77)
    for direction in (0, 1):
        acc = np.zeros((N, n), dtype=np.complex128)
        for rank in range(r * c):
            ch = lib.Chase(N, 16, 8, grid=(r, c), rank=rank, world_size=1, dtype="c64")
            r0, p, c0, q = ch.local_layout()
            dH = _dev(H[r0:r0 + p, c0:c0 + q])
            if direction == 0:
                dY = _dev(Y0[r0:r0 + p])
                ch.hemm_step(0, dH, _dev(X[c0:c0 + q]), dY, n, 1.3, -0.4, 0.77)
                acc[r0:r0 + p] += dY.cpu().numpy()
            else:
                dY = _dev(Y0[c0:c0 + q])
                ch.hemm_step(1, dH, _dev(X[r0:r0 + p]), dY, n, 1.3, -0.4, 0.77)
                acc[c0:c0 + q] += dY.cpu().numpy()
            ch.close()
        assert _rel(acc, ref) <= 1e-5, direction


def test_c64_rejects_misaligned_shard(lib):
    """TMA layout limits: an odd-order grid is refused at chase_init (the same answer on every
    rank, decided from N / r / c); an odd ldh or a misaligned H at the call."""
    from paper_2205_02491_b200._lib import ChaseError
    with pytest.raises(ChaseError) as e:
        lib.Chase(1001, 4, 4, dtype="c64")
    assert e.value.status == 2
    ch = lib.Chase(1000, 4, 4, dtype="c64")
    Hp = torch.zeros((1000, 1001), dtype=torch.complex64, device="cuda")
    H = Hp.t()[:1000, :1000]             # column-major view with ldh = 1001 (odd)
    X = torch.zeros((8, 1000), dtype=torch.complex64, device="cuda").t()
    Y = torch.zeros((8, 1000), dtype=torch.complex64, device="cuda").t()
    with pytest.raises(ChaseError) as e:
        ch.hemm_step(0, H, X, Y, 8, 1.0, 0.0, 0.0)
    assert e.value.status == 2


def test_c64_lanczos_vs_oracle(lib):
    N, n_e = 700, 60
    M = make_matrix("uniform", N, "g2", seed=4)
    H = M.dense().astype(np.complex64)
    ch = lib.Chase(N, 40, 20, dtype="c64")
    b_sup, mu_1, mu_ne, nu = ch.lanczos(_dev(H), n_e)
    lz = oracle.lanczos(H.astype(np.complex128), n_e)
    # FP64-accumulated products on the fp32 shard: the bounds agree to the fp32 input rounding
    for a, b in ((b_sup, lz.b_sup), (mu_1, lz.mu_1), (mu_ne, lz.mu_ne), (nu, lz.nu)):
        assert abs(a - b) <= 1e-9 * max(1.0, abs(b)), (a, b)


@pytest.mark.parametrize("fam,N", [("uniform", 600), ("wilkinson", 1000), ("121", 800)])
def test_c64_solve_vs_exact(lib, fam, N):
    """north_star: complex single eigenvalues to 1e-4 relative; here also 2e-5 ||H|| absolute and
    the residuals of the returned complex64 vectors against the c64 shard in FP64."""
    nev, nex = 40, 20
    M = make_matrix(fam, N, "g2", seed=3)
    H = M.dense().astype(np.complex64)
    ch = lib.Chase(N, nev, nex, dtype="c64")
    vals, dvecs, rep, st = ch.solve(_dev(H), nev, nex, deg=20, tol=1e-5)
    assert st == 0, ch.last_error()
    normH = np.max(np.abs(M.lam))
    vecs = dvecs.cpu().numpy()[:, :nev].astype(np.complex128)
    assert dvecs.dtype == torch.complex64
    lam = M.lam[:nev]
    assert np.max(np.abs(vals - lam) / np.maximum(np.abs(lam), 1e-300)) <= 1e-4 or \
        np.max(np.abs(vals - lam)) <= 2e-5 * normH
    assert np.max(np.abs(vals - lam)) <= 2e-5 * normH
    Hd = H.astype(np.complex128)
    res = np.linalg.norm(Hd @ vecs - vecs * vals[None, :], axis=0) / normH
    assert np.max(res) <= 1e-4, np.max(res)
    np.testing.assert_allclose(vecs.conj().T @ vecs, np.eye(nev), atol=1e-5)


def test_c64_random_block_is_rounded_generator(lib):
    from oracle.rng import random_block
    N = 404
    ch = lib.Chase(N, 10, 6, dtype="c64")
    dV = torch.zeros((16, N), dtype=torch.complex64, device="cuda").t()
    ch.random_block(dV, 3, 13, seed=99, stream=1)
    assert np.array_equal(dV.cpu().numpy()[:, :13], random_block(99, 0, N, 3, 13, 1).astype(np.complex64))


@pytest.mark.parametrize("fam,N", [("uniform", 1200), ("wilkinson", 1000)])
def test_f4_mixed_filter_c128_solve(lib, fam, N):
    """complex-double solve whose early filters run on the complex-single shadow; the
    returned pairs must meet the complex-double bars exactly as without it."""
    nev, nex = 40, 20
    M = make_matrix(fam, N, "g2", seed=3)
    H = M.dense()
    dH = torch.from_numpy(np.asfortranarray(H)).t().contiguous().t().cuda()
    ch = lib.Chase(N, nev, nex)
    ch.set_option("mixed_filter", 1e-3)
    vals, dvecs, rep, st = ch.solve(dH, nev, nex, deg=20, tol=1e-10)
    assert st == 0, ch.last_error()
    normH = np.max(np.abs(M.lam))
    vecs = dvecs.cpu().numpy()[:, :nev]
    assert np.max(np.abs(vals - M.lam[:nev])) <= 1e-10 * normH
    assert np.max(np.linalg.norm(H @ vecs - vecs * vals[None, :], axis=0)) <= 1e-10 * normH
    np.testing.assert_allclose(vecs.conj().T @ vecs, np.eye(nev), atol=1e-12)


def test_c64_solve_largest(lib):
    """`largest` (ledger #17) in complex single: the nev largest eigenvalues (ascending, as the
    complex-double path returns them)."""
    N, nev, nex = 800, 24, 12
    M = make_matrix("uniform", N, "g2", seed=11)
    H = M.dense().astype(np.complex64)
    ch = lib.Chase(N, nev, nex, dtype="c64")
    ch.set_option("largest", 1)
    vals, dvecs, rep, st = ch.solve(_dev(H), nev, nex, deg=20, tol=1e-5)
    assert st == 0, ch.last_error()
    top = np.sort(M.lam)[-nev:]
    assert np.max(np.abs(vals - top)) <= 2e-5 * np.max(np.abs(M.lam))
