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
    ch = lib.Chase(1001, 4, 4, dtype="c64")
    H = torch.zeros((1001, 1001), dtype=torch.complex64, device="cuda")
    X = torch.zeros((8, 1001), dtype=torch.complex64, device="cuda").t()
    Y = torch.zeros((8, 1001), dtype=torch.complex64, device="cuda").t()
    with pytest.raises(Exception):
        ch.hemm_step(0, H, X, Y, 8, 1.0, 0.0, 0.0)
