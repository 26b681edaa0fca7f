"""GPU parity of the real-symmetric variant (the paper's own experimental field,
P:134) through the C ABI (dtype CHASE_R64) against the CPU oracle in float64 and the exact
spectra of the real generators (r1: real Haar Q, r2: Hartley-based, any n)."""
import numpy as np
import pytest

import oracle
from chase_gen import make_matrix, block_partition

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _dev(a):
    return torch.from_numpy(np.asfortranarray(a)).t().contiguous().t().cuda()


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def lib():
    import paper_2205_02491_b200 as pkg
    return pkg


@pytest.mark.parametrize("N,ncols", [(1000, 75), (333, 7), (257, 130), (64, 1), (1501, 200)])
@pytest.mark.parametrize("direction", [0, 1])
def test_real_hemm_step(lib, N, ncols, direction):
    H = make_matrix("uniform", N, "r2", seed=N).dense()
    rng = np.random.default_rng(N + ncols)
    X = rng.standard_normal((N, ncols))
    Y0 = rng.standard_normal((N, ncols))
    ch = lib.Chase(N, 1, 1, dtype="r64")
    dY = _dev(Y0)
    ch.hemm_step(direction, _dev(H), _dev(X), dY, ncols, 0.37, -0.81, 0.55)
    assert _rel(dY.cpu().numpy(), oracle.hemm_step(H, X, Y0, 0.37, -0.81, 0.55)) <= 1e-13


@pytest.mark.parametrize("grid", [(1, 2), (2, 2), (3, 2)])
def test_real_emulated_grid_step(lib, grid):
    """Odd shard sizes / row offsets (unaligned operands for the cp.async path) and the shift on I_ij."""
    r, c = grid
    N, n = 301, 19
    H = make_matrix("wilkinson", N, "r2", seed=5).dense()
    rng = np.random.default_rng(2)
    X, Y0 = rng.standard_normal((N, n)), rng.standard_normal((N, n))
    ref = oracle.hemm_step(H, X, Y0, 1.3, -0.4, 0.77)
    for direction in (0, 1):
        acc = np.zeros((N, n))
        for rank in range(r * c):
            ch = lib.Chase(N, 4, 4, grid=(r, c), rank=rank, world_size=1, dtype="r64")
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
        assert _rel(acc, ref) <= 1e-13, direction


def test_real_filter_vs_oracle(lib):
    N = 900
    M = make_matrix("121", N, "r2", seed=7)
    H = M.dense()
    degrees = np.sort(np.array([0, 2, 2, 4, 6, 8, 14, 20, 20, 36, 36] + [20] * 50))
    n = len(degrees)
    V = np.random.default_rng(1).standard_normal((N, n))
    b_sup, mu_1, mu_ne = M.lam[-1] * 1.02, M.lam[0], M.lam[n]
    ch = lib.Chase(N, n - 5, 5, dtype="r64")
    dV = _dev(V)
    dW = torch.zeros((n, N), dtype=torch.float64, device="cuda").t()
    mv = ch.filter(_dev(H), dV, dW, degrees, b_sup, mu_1, mu_ne)
    ref, mv_ref = oracle.chebyshev_filter(H, V, degrees, b_sup, mu_1, mu_ne)
    assert mv == mv_ref
    out = dV.cpu().numpy()
    for a in range(n):
        assert _rel(out[:, a], ref[:, a]) <= 1e-11, (a, degrees[a])


def test_real_random_block_and_generator_twin(lib):
    from oracle.rng import random_block
    from chase_gen.device import DeviceR2
    N = 777
    ch = lib.Chase(N, 10, 6, dtype="r64")
    dV = torch.zeros((16, N), dtype=torch.float64, device="cuda").t()
    ch.random_block(dV, 3, 13, seed=99, stream=1)
    assert np.array_equal(dV.cpu().numpy()[:, :13], random_block(99, 0, N, 3, 13, 1).real)
    M = make_matrix("geometric", 513, "r2", seed=9)
    out = torch.empty((300, 201), dtype=torch.float64, device="cuda").t()
    DeviceR2(M).fill(out, 100, 150)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), M.block(100, 201, 150, 300))


def test_real_lanczos_vs_oracle(lib):
    N, n_e = 700, 60
    M = make_matrix("uniform", N, "r2", seed=4)
    H = M.dense()
    ch = lib.Chase(N, 40, 20, dtype="r64")
    b_sup, mu_1, mu_ne, nu = ch.lanczos(_dev(H), n_e)
    lz = oracle.lanczos(H, n_e)
    for a, b in ((b_sup, lz.b_sup), (mu_1, lz.mu_1), (mu_ne, lz.mu_ne), (nu, lz.nu)):
        assert abs(a - b) <= 1e-10


@pytest.mark.parametrize("fam,kind,N", [("uniform", "r1", 600), ("wilkinson", "r2", 1001), ("121", "r2", 800)])
def test_real_solve_vs_exact_and_oracle(lib, fam, kind, N):
    nev, nex = 40, 20
    M = make_matrix(fam, N, kind, seed=3)
    H = M.dense()
    ch = lib.Chase(N, nev, nex, dtype="r64")
    vals, dvecs, rep, st = ch.solve(_dev(H), nev, nex, deg=20, tol=1e-10)
    assert st == 0, ch.last_error()
    normH = np.max(np.abs(M.lam))
    vecs = dvecs.cpu().numpy()[:, :nev]
    assert vecs.dtype == np.float64
    assert np.max(np.abs(vals - M.lam[:nev])) <= 1e-10 * normH
    assert np.max(np.linalg.norm(H @ vecs - vecs * vals[None, :], axis=0)) <= 1e-10 * normH
    np.testing.assert_allclose(vecs.T @ vecs, np.eye(nev), atol=1e-12)
    ov, _, orep = oracle.chase_solve(H, nev, nex, deg=20, tol=1e-10)
    assert np.max(np.abs(vals - ov)) <= 1e-10 * normH
    assert abs(rep["iterations"] - orep.iterations) <= 1
