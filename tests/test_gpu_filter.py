"""GPU parity of the filter hot path through the C ABI vs the CPU oracle.

Shapes span several 128x64 tiles and ragged tails in M, N and K; tolerances are derived in
DESIGN.md ("Tolerances"): a fused step is a length-K FP64 dot product per entry, so its relative
Frobenius error is ~ sqrt(K) u; 1e-13 is the SURVEY §8(c) per-step bar."""
import numpy as np
import pytest

import oracle
from chase_gen import make_matrix, block_partition

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _dev(a):
    """numpy complex (n, m) -> column-major complex128 CUDA tensor."""
    t = torch.from_numpy(np.asfortranarray(a))
    return t.t().contiguous().t().cuda() if t.dim() == 2 else t.cuda()


def _host(t):
    return t.cpu().numpy()


@pytest.fixture(scope="module")
def lib():
    import paper_2205_02491_b200 as pkg
    assert torch.cuda.is_available()
    return pkg


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("N,ncols", [(1000, 75), (333, 7), (257, 130), (64, 1), (1500, 200)])
@pytest.mark.parametrize("direction", [0, 1])
def test_hemm_step_1x1(lib, N, ncols, direction):
    M = make_matrix("uniform", N, "g2", seed=N)
    H = M.dense()
    rng = np.random.default_rng(N + ncols)
    X = rng.standard_normal((N, ncols)) + 1j * rng.standard_normal((N, ncols))
    Y0 = rng.standard_normal((N, ncols)) + 1j * rng.standard_normal((N, ncols))
    ch = lib.Chase(N, 1, 1)
    dH, dX, dY = _dev(H), _dev(X), _dev(Y0)
    alpha, beta, gamma = 0.37, -0.81, 0.55
    ch.hemm_step(direction, dH, dX, dY, ncols, alpha, beta, gamma)
    ref = oracle.hemm_step(H, X, Y0, alpha, beta, gamma)
    out = _host(dY)
    assert _rel(out, ref) <= 1e-13
    # element-wise too (a single wrong entry must not hide in the Frobenius norm)
    assert np.max(np.abs(out - ref)) <= 1e-13 * np.max(np.abs(ref))
    ch.close()


def test_hemm_step_no_shift_no_beta_ld_padding(lib):
    N, n = 700, 33
    H = make_matrix("wilkinson", N, "g2", seed=3).dense()
    rng = np.random.default_rng(0)
    X = rng.standard_normal((N, n)) + 1j * rng.standard_normal((N, n))
    # padded leading dimensions (ld > rows) for H, X, Y
    Hp = torch.zeros((N + 13, N), dtype=torch.complex128)
    Hp[:N] = torch.from_numpy(H)
    dH = Hp.t().contiguous().t().cuda()[:N]           # ld = N + 13
    Xp = torch.zeros((N + 5, n), dtype=torch.complex128)
    Xp[:N] = torch.from_numpy(X)
    dX = Xp.t().contiguous().t().cuda()[:N]
    dY = torch.full((n, N + 7), complex(np.nan, np.nan), dtype=torch.complex128).t().cuda()[:N]
    ch = lib.Chase(N, 4, 4)
    ch.hemm_step(1, dH, dX, dY, n, 1.0, 0.0, 0.0)     # beta = 0 must not read Y (NaN poison)
    assert _rel(_host(dY), H.conj().T @ X) <= 1e-13


@pytest.mark.parametrize("fam", ["uniform", "121"])
def test_filter_1x1_vs_oracle(lib, fam):
    N = 900
    M = make_matrix(fam, N, "g2", seed=7)
    H = M.dense()
    degrees = np.array([0, 2, 2, 4, 4, 6, 8, 10, 14, 20, 20, 20, 20, 36, 36] + [20] * 50)
    degrees = np.sort(degrees)
    n = len(degrees)
    rng = np.random.default_rng(1)
    V = rng.standard_normal((N, n)) + 1j * rng.standard_normal((N, n))
    lam = M.lam
    b_sup = lam[-1] * 1.02
    mu_1, mu_ne = lam[0], lam[n]
    ch = lib.Chase(N, n - 5, 5)
    dH, dV = _dev(H), _dev(V)
    dW = torch.zeros((n, N), dtype=torch.complex128, device="cuda").t()
    mv = ch.filter(dH, dV, dW, degrees, b_sup, mu_1, mu_ne)
    ref, mv_ref = oracle.chebyshev_filter(H, V, degrees, b_sup, mu_1, mu_ne)
    assert mv == mv_ref == degrees.sum()
    out = _host(dV)
    for a in range(n):
        assert _rel(out[:, a], ref[:, a]) <= 1e-11, (a, degrees[a])


def test_filter_rejects_odd_or_unsorted_degrees(lib):
    N = 64
    ch = lib.Chase(N, 2, 2)
    dH = torch.eye(N, dtype=torch.complex128, device="cuda").t().contiguous().t()
    dV = torch.zeros((N, 4), dtype=torch.complex128, device="cuda").t().contiguous().t()
    dW = torch.zeros_like(dV)
    with pytest.raises(lib.ChaseError):
        ch.filter(dH, dV, dW, [2, 3, 4, 4], 2.0, 0.0, 1.0)
    with pytest.raises(lib.ChaseError):
        ch.filter(dH, dV, dW, [4, 2, 4, 4], 2.0, 0.0, 1.0)


def test_empty_block_and_degree_zero(lib):
    """Degenerate cases of the filter (Alg. 1 line 4): an empty block is a no-op through
    every entry point, and degree 0 is C_0 = 1 (the column is returned bitwise unchanged, 0
    matvecs)."""
    N = 300
    H = make_matrix("uniform", N, "g2", seed=11).dense()
    ch = lib.Chase(N, 4, 4)
    dH = _dev(H)
    empty = torch.zeros((N, 0), dtype=torch.complex128, device="cuda")
    for d in (0, 1):
        ch.hemm_step(d, dH, empty, empty, 0, 1.0, 0.5, 0.25)
    dW = torch.zeros((N, 8), dtype=torch.complex128, device="cuda").t().contiguous().t()
    assert ch.filter(dH, empty, dW, [], 2.0, 0.0, 1.0) == 0
    ch.random_block(empty, 0, 0, 1, 0)
    rng = np.random.default_rng(5)
    V = rng.standard_normal((N, 8)) + 1j * rng.standard_normal((N, 8))
    dV = _dev(V)
    lam = make_matrix("uniform", N, "g2", seed=11).lam
    assert ch.filter(dH, dV, dW, [0] * 8, lam[-1] * 1.01, lam[0], lam[8]) == 0
    assert np.array_equal(_host(dV), V)
    with pytest.raises(lib.ChaseError):         # empty interval b_sup <= mu_ne (chase.h)
        ch.filter(dH, dV, dW, [2] * 8, lam[8], lam[0], lam[8])
    ch.close()


@pytest.mark.parametrize("grid", [(1, 2), (2, 1), (2, 2), (2, 3), (3, 2)])
def test_emulated_grid_hemm_step(lib, grid):
    """Grid neutrality of the fused step: per-rank partials (emulated-grid mode) summed
    over the row comm (forward) / column comm (backward) equal the serial oracle step, including
    the intersection shift E_ij and the single beta owner per communicator."""
    r, c = grid
    N, n = 301, 19
    H = make_matrix("wilkinson", N, "g2", seed=5).dense()
    rng = np.random.default_rng(2)
    X = rng.standard_normal((N, n)) + 1j * rng.standard_normal((N, n))
    Y0 = rng.standard_normal((N, n)) + 1j * rng.standard_normal((N, n))
    alpha, beta, gamma = 1.3, -0.4, 0.77
    ref = oracle.hemm_step(H, X, Y0, alpha, beta, gamma)
    rows, cols = block_partition(N, r), block_partition(N, c)
    for direction in (0, 1):
        acc = np.zeros((N, n), dtype=complex)
        for rank in range(r * c):
            i, j = rank % r, rank // r
            ch = lib.Chase(N, 4, 4, grid=(r, c), rank=rank, world_size=1)
            r0, p, c0, q = ch.local_layout()
            assert (r0, p, c0, q) == (rows[i][0], rows[i][1], cols[j][0], cols[j][1])
            dH = _dev(H[r0:r0 + p, c0:c0 + q])
            if direction == 0:
                dX, dY = _dev(X[c0:c0 + q]), _dev(Y0[r0:r0 + p])
                ch.hemm_step(0, dH, dX, dY, n, alpha, beta, gamma)
                acc[r0:r0 + p] += _host(dY)
            else:
                dX, dY = _dev(X[r0:r0 + p]), _dev(Y0[c0:c0 + q])
                ch.hemm_step(1, dH, dX, dY, n, alpha, beta, gamma)
                acc[c0:c0 + q] += _host(dY)
            ch.close()
        assert _rel(acc, ref) <= 1e-13, direction


def test_random_block_matches_oracle_bitwise(lib):
    from oracle.rng import random_block
    N = 777
    ch = lib.Chase(N, 10, 6)
    dV = torch.zeros((16, N), dtype=torch.complex128, device="cuda").t()
    ch.random_block(dV, 3, 13, seed=12345678901, stream=1)
    ref = random_block(12345678901, 0, N, 3, 13, 1)
    assert np.array_equal(_host(dV)[:, :13], ref)


def test_generator_device_twin_bitwise():
    from chase_gen.device import DeviceG2
    M = make_matrix("geometric", 513, "g2", seed=9)
    dg = DeviceG2(M)
    out = torch.empty((300, 200), dtype=torch.complex128, device="cuda").t()    # 200 x 300, ld 200
    dg.fill(out, 100, 150)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), M.block(100, 200, 150, 300))


@pytest.mark.parametrize("N,ncols", [(1000, 75), (333, 7), (257, 130), (1500, 200)])
@pytest.mark.parametrize("direction", [0, 1])
@pytest.mark.parametrize("algo", [0, 1])
def test_hemm_step_3m_and_4m(lib, N, ncols, direction, algo):
    """Both complex-product kernels (4M: algo 0, 3M Gauss: algo 1) of the fused step: 1e-13 bar."""
    M = make_matrix("uniform", N, "g2", seed=N + 1)
    H = M.dense()
    rng = np.random.default_rng(N + 2 * ncols)
    X = rng.standard_normal((N, ncols)) + 1j * rng.standard_normal((N, ncols))
    Y0 = rng.standard_normal((N, ncols)) + 1j * rng.standard_normal((N, ncols))
    ch = lib.Chase(N, 1, 1)
    ch.set_option("gemm3m", algo)
    dH, dX, dY = _dev(H), _dev(X), _dev(Y0)
    ch.hemm_step(direction, dH, dX, dY, ncols, 0.37, -0.81, 0.55)
    ref = oracle.hemm_step(H, X, Y0, 0.37, -0.81, 0.55)
    assert _rel(_host(dY), ref) <= 1e-13
    ch.close()


def test_filter_3m_vs_oracle(lib):
    N = 900
    M = make_matrix("wilkinson", N, "g2", seed=8)
    H = M.dense()
    degrees = np.sort(np.array([0, 2, 4, 8, 14, 20, 20, 36] + [20] * 40))
    n = len(degrees)
    V = np.random.default_rng(3).standard_normal((N, n)) + 0j
    b_sup, mu_1, mu_ne = M.lam[-1] * 1.02, M.lam[0], M.lam[n]
    ch = lib.Chase(N, n - 5, 5)
    ch.set_option("gemm3m", 1)
    dV = _dev(V)
    dW = torch.zeros((n, N), dtype=torch.complex128, device="cuda").t()
    ch.filter(_dev(H), dV, dW, degrees, b_sup, mu_1, mu_ne)
    ref, _ = oracle.chebyshev_filter(H, V, degrees, b_sup, mu_1, mu_ne)
    out = _host(dV)
    for a in range(n):
        assert _rel(out[:, a], ref[:, a]) <= 1e-11, (a, degrees[a])
