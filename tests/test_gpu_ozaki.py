"""f4 research branch: complex-double filter steps with the FP64 products emulated on the INT8
tensor cores (Ozaki scheme; csrc/ozaki.cu, option fp64_emulation = S slices).

  * exactness: operands that are small integers times powers of two are represented exactly by
    the first slices, so the emulated product must equal the exact product bit for bit (the int8
    tcgen05 MMA, the TMA operand layout, the slice recombination and the 3M combination are all
    checked by this one identity);
  * accuracy: one fused step (shift, beta, both directions, ragged M / N / K) vs oracle.hemm_step
    at the complex-double bar 1e-13 for S = 7; the error falls with S as
    ~2^-7S (table in DESIGN.md);
  * the filter and a whole solve with emulated products meet the complex-double bars."""
import numpy as np
import pytest

import oracle
from chase_gen import make_matrix

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _dev(a):
    return torch.from_numpy(np.asfortranarray(a)).t().contiguous().t().cuda()


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("crt", [0, 1], ids=["slices", "crt"])
@pytest.mark.parametrize("direction", [0, 1])
@pytest.mark.parametrize("N,n", [(600, 37), (777, 300), (130, 1)])
def test_emulated_product_is_exact_on_representable_inputs(direction, N, n, crt):
    import paper_2205_02491_b200 as pkg
    rng = np.random.default_rng(N + n)
    Hr, Hi = rng.integers(-100, 101, (N, N)), rng.integers(-100, 101, (N, N))
    Xr, Xi = rng.integers(-50, 51, (N, n)), rng.integers(-50, 51, (N, n))
    H = (Hr + 1j * Hi) * 2.0 ** -10          # not Hermitian: the step does not need it
    X = (Xr + 1j * Xi) * 2.0 ** -3
    # exact integer products (int64), scaled by 2^-13 (exact in FP64: |sums| < 2^53)
    if direction == 0:
        Ar, Ai = Hr, Hi
    else:                                   # op(H) = H^H
        Ar, Ai = Hr.T, -Hi.T
    re = Ar @ Xr - Ai @ Xi
    im = Ar @ Xi + Ai @ Xr
    ref = (re + 1j * im) * 2.0 ** -13
    ch = pkg.Chase(N, n, 1)
    ch.set_option("fp64_emulation", 7)
    ch.set_option("oz_crt", crt)
    dY = _dev(np.zeros((N, n), dtype=complex))
    ch.hemm_step(direction, _dev(H), _dev(X), dY, n, 1.0, 0.0, 0.0)
    assert np.array_equal(dY.cpu().numpy(), ref)


@pytest.mark.parametrize("crt", [0, 1], ids=["slices", "crt"])
@pytest.mark.parametrize("direction", [0, 1])
@pytest.mark.parametrize("N,n", [(1000, 75), (1300, 257), (333, 7)])
def test_emulated_step_vs_oracle(direction, N, n, crt):
    import paper_2205_02491_b200 as pkg
    M = make_matrix("uniform", N, "g2", seed=N)
    H = M.dense()
    rng = np.random.default_rng(n)
    X = rng.standard_normal((N, n)) + 1j * rng.standard_normal((N, n))
    Y0 = rng.standard_normal((N, n)) + 1j * rng.standard_normal((N, n))
    ref = oracle.hemm_step(H, X, Y0, 0.37, -0.81, 0.55)
    ch = pkg.Chase(N, n, 1)
    ch.set_option("fp64_emulation", 7)
    ch.set_option("oz_crt", crt)
    dY = _dev(Y0)
    ch.hemm_step(direction, _dev(H), _dev(X), dY, n, 0.37, -0.81, 0.55)
    err = _rel(dY.cpu().numpy(), ref)
    assert err <= 1e-13, err
    # beta = 0 must not read Y (NaN poison)
    dY = torch.full((n, N), complex(np.nan, np.nan), dtype=torch.complex128).cuda().t()
    ch.hemm_step(direction, _dev(H), _dev(X), dY, n, 1.0, 0.0, 0.0)
    assert _rel(dY.cpu().numpy(), H @ X) <= 1e-13


def test_emulated_filter_and_solve():
    import paper_2205_02491_b200 as pkg
    N, nev, nex = 900, 40, 20
    M = make_matrix("wilkinson", N, "g2", seed=7)
    H = M.dense()
    degrees = np.sort(np.array([0, 2, 4, 6, 10, 20, 36] + [20] * 30))
    V = oracle.random_block(5, 0, N, 0, len(degrees), 0)
    b_sup, mu_1, mu_ne = M.lam[-1] * 1.01, M.lam[0], M.lam[60]
    fref, mv = oracle.chebyshev_filter(H, V, degrees, b_sup, mu_1, mu_ne)
    ch = pkg.Chase(N, nev, nex)
    ch.set_option("fp64_emulation", 7)
    dH, dV = _dev(H), _dev(V)
    dW = _dev(np.zeros((N, len(degrees)), dtype=complex))
    assert ch.filter(dH, dV, dW, degrees, b_sup, mu_1, mu_ne) == mv
    out = dV.cpu().numpy()
    colerr = np.linalg.norm(out - fref, axis=0) / np.linalg.norm(fref, axis=0)
    assert np.max(colerr) <= 1e-11
    vals, vecs, rep, st = ch.solve(dH, nev, nex, deg=20, tol=1e-10)
    assert st == 0
    normH = np.max(np.abs(M.lam))
    assert np.max(np.abs(vals - M.lam[:nev])) <= 1e-10 * normH
    Vv = vecs.cpu().numpy()[:, :nev]
    assert np.max(np.linalg.norm(H @ Vv - Vv * vals[None, :], axis=0)) <= 1e-10 * normH


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_shard_rewritten_in_place_is_resliced(dtype):
    """Derived copies of the shard (Ozaki slices; the c64 3xTF32 lo part) are rebuilt on every API
    call: rewriting H in place (same pointer) between calls must change the result."""
    import paper_2205_02491_b200 as pkg
    N, n = 512, 16
    cdt = np.complex64 if dtype == "c64" else np.complex128
    H1 = make_matrix("uniform", N, "g2", seed=1).dense().astype(cdt)
    H2 = make_matrix("wilkinson", N, "g2", seed=2).dense().astype(cdt)
    rng = np.random.default_rng(0)
    X = (rng.standard_normal((N, n)) + 1j * rng.standard_normal((N, n))).astype(cdt)
    ch = pkg.Chase(N, n, 1, dtype=dtype)
    dH, dX = _dev(H1), _dev(X)
    tol = 1e-5 if dtype == "c64" else 1e-13
    for H in (H1, H2):
        dH.copy_(torch.from_numpy(np.asfortranarray(H)))
        dY = _dev(np.zeros((N, n), dtype=cdt))
        ch.hemm_step(0, dH, dX, dY, n, 1.0, 0.0, 0.0)
        ref = H.astype(complex) @ X.astype(complex)
        assert _rel(dY.cpu().numpy().astype(complex), ref) <= tol


@pytest.mark.parametrize("direction", [0, 1])
def test_real_emulated_product_exact_and_step_vs_oracle(direction):
    """Real-symmetric variant (f2): one real product per step (no 3M)."""
    import paper_2205_02491_b200 as pkg
    N, n = 700, 45
    rng = np.random.default_rng(3)
    Hi = rng.integers(-100, 101, (N, N))
    Xi = rng.integers(-50, 51, (N, n))
    ref = ((Hi if direction == 0 else Hi.T) @ Xi) * 2.0 ** -13
    ch = pkg.Chase(N, n, 1, dtype="r64")
    ch.set_option("fp64_emulation", 7)
    dY = _dev(np.zeros((N, n)))
    ch.hemm_step(direction, _dev(Hi * 2.0 ** -10), _dev(Xi * 2.0 ** -3), dY, n, 1.0, 0.0, 0.0)
    assert np.array_equal(dY.cpu().numpy(), ref)
    M = make_matrix("uniform", N, "r2", seed=4)
    H = M.dense()
    X, Y0 = rng.standard_normal((N, n)), rng.standard_normal((N, n))
    ref = oracle.hemm_step(H, X, Y0, 0.37, -0.81, 0.55)
    dY = _dev(Y0)
    ch.hemm_step(direction, _dev(H), _dev(X), dY, n, 0.37, -0.81, 0.55)
    assert _rel(dY.cpu().numpy(), ref) <= 1e-13


def test_real_emulated_solve():
    import paper_2205_02491_b200 as pkg
    N, nev, nex = 800, 40, 20
    M = make_matrix("wilkinson", N, "r2", seed=7)
    H = M.dense()
    ch = pkg.Chase(N, nev, nex, dtype="r64")
    vals, vecs, rep, st = ch.solve(_dev(H), nev, nex, deg=20, tol=1e-10)
    assert st == 0
    normH = np.max(np.abs(M.lam))
    assert np.max(np.abs(vals - M.lam[:nev])) <= 1e-10 * normH
    V = vecs.cpu().numpy()[:, :nev]
    assert np.max(np.linalg.norm(H @ V - V * vals[None, :], axis=0)) <= 1e-10 * normH


@pytest.mark.parametrize("direction", [0, 1])
def test_emulated_step_graded_matrix(direction):
    """A graded Hermitian H = D A D (D spanning 1e-6 .. 1) and a graded block X: the row / column
    power-of-two equilibration of the splitting keeps the step at the complex-double bar."""
    import paper_2205_02491_b200 as pkg
    N, n = 640, 48
    rng = np.random.default_rng(11)
    A = make_matrix("uniform", N, "g2", seed=3).dense()
    d = np.logspace(-6, 0, N)
    H = (d[:, None] * A) * d[None, :]
    X = (rng.standard_normal((N, n)) + 1j * rng.standard_normal((N, n))) * np.logspace(0, -4, n)[None, :]
    Y0 = rng.standard_normal((N, n)) + 1j * rng.standard_normal((N, n))
    ref = oracle.hemm_step(H, X, Y0 * 1e-6, 0.9, 0.5, 1e-3)
    ch = pkg.Chase(N, n, 1)
    dY = _dev(Y0 * 1e-6)
    ch.hemm_step(direction, _dev(H), _dev(X), dY, n, 0.9, 0.5, 1e-3)
    out = dY.cpu().numpy()
    colerr = np.linalg.norm(out - ref, axis=0) / np.linalg.norm(ref, axis=0)
    assert np.max(colerr) <= 1e-13, float(np.max(colerr))


@pytest.mark.parametrize("dtype", ["c128", "r64"])
def test_iteration_gemms_on_the_emulation(dtype):
    """oz_gemm_min = oz_gemm_kmin = 0 routes every plain GEMM of the iteration (CGS, Gram, RR's Q^H (HQ), Q Z,
    (HQ) Z) through the INT8 emulation too (only V R^-1 stays on DMMA): the solve keeps the
    complex-double bars against the exact spectrum and the oracle."""
    import paper_2205_02491_b200 as pkg
    real = dtype == "r64"
    N, nev, nex = 700, 40, 20
    M = make_matrix("uniform", N, "r2" if real else "g2", seed=12)
    H = M.dense()
    ch = pkg.Chase(N, nev, nex, dtype=dtype)
    ch.set_option("oz_gemm_min", 0)
    ch.set_option("oz_gemm_kmin", 0)
    vals, vecs, rep, st = ch.solve(_dev(H), nev, nex, deg=20, tol=1e-10)
    assert st == 0
    normH = np.max(np.abs(M.lam))
    assert np.max(np.abs(vals - M.lam[:nev])) <= 1e-10 * normH
    ov, _, _ = oracle.chase_solve(H, nev, nex, deg=20, tol=1e-10)
    assert np.max(np.abs(vals - ov)) <= 1e-10 * normH
    V = vecs.cpu().numpy()[:, :nev]
    assert np.max(np.linalg.norm(H @ V - V * vals[None, :], axis=0)) <= 1e-10 * normH
    assert np.max(np.abs(V.conj().T @ V - np.eye(nev))) <= 1e-12


@pytest.mark.parametrize("dtype", ["c128", "r64"])
def test_crt_scheme_solve_and_graded_step(dtype):
    """Ozaki scheme II (oz_crt = 1: 16 CRT moduli, exact A'B' of the 52-bit scaled operands): the
    solve keeps the complex-double bars, and a graded H = D A D step stays at the 1e-13 bar."""
    import paper_2205_02491_b200 as pkg
    real = dtype == "r64"
    N, nev, nex = 700, 40, 20
    M = make_matrix("uniform", N, "r2" if real else "g2", seed=13)
    H = M.dense()
    ch = pkg.Chase(N, nev, nex, dtype=dtype)
    ch.set_option("oz_crt", 1)
    ch.set_option("oz_gemm_min", 0)
    ch.set_option("oz_gemm_kmin", 0)
    vals, vecs, rep, st = ch.solve(_dev(H), nev, nex, deg=20, tol=1e-10)
    assert st == 0
    normH = np.max(np.abs(M.lam))
    assert np.max(np.abs(vals - M.lam[:nev])) <= 1e-10 * normH
    V = vecs.cpu().numpy()[:, :nev]
    assert np.max(np.linalg.norm(H @ V - V * vals[None, :], axis=0)) <= 1e-10 * normH
    assert np.max(np.abs(V.conj().T @ V - np.eye(nev))) <= 1e-12
    n = 33
    rng = np.random.default_rng(5)
    d = np.logspace(-6, 0, N)
    G = (d[:, None] * H) * d[None, :]
    X = rng.standard_normal((N, n)) + (0 if real else 1j) * rng.standard_normal((N, n))
    ref = oracle.hemm_step(G, X, 0 * X, 0.9, 0.0, 1e-3)
    for direction in (0, 1):
        dY = _dev(np.zeros_like(X))
        ch.hemm_step(direction, _dev(G), _dev(X), dY, n, 0.9, 0.0, 1e-3)
        assert _rel(dY.cpu().numpy(), ref) <= 1e-13


def test_crt_falls_back_to_slices_when_residues_do_not_fit(monkeypatch):
    """oz_crt = 1 whose residue set does not fit (simulated: CHASE_OZ_CRT_MAXBYTES) continues on
    the 7-slice scheme -- bitwise the result of a slice-scheme handle -- not on DMMA."""
    import paper_2205_02491_b200 as pkg
    N, n = 500, 24
    H = make_matrix("uniform", N, "g2", seed=8).dense()
    rng = np.random.default_rng(2)
    X = rng.standard_normal((N, n)) + 1j * rng.standard_normal((N, n))
    out = {}
    for mode in ("slices", "crt-fallback", "crt"):
        if mode == "crt-fallback":
            monkeypatch.setenv("CHASE_OZ_CRT_MAXBYTES", "1000")
        else:
            monkeypatch.delenv("CHASE_OZ_CRT_MAXBYTES", raising=False)
        ch = pkg.Chase(N, n, 1)
        ch.set_option("oz_crt", 0 if mode == "slices" else 1)
        dY = _dev(np.zeros((N, n), dtype=complex))
        ch.hemm_step(0, _dev(H), _dev(X), dY, n, 1.0, 0.0, 0.0)
        out[mode] = dY.cpu().numpy()
        assert _rel(out[mode], H @ X) <= 1e-13, mode
        ch.close()
    assert np.array_equal(out["crt-fallback"], out["slices"])
    assert not np.array_equal(out["crt"], out["slices"])     # scheme II really ran without the cap


def test_ozaki_scheme_reported():
    """chase_get_option("ozaki_scheme"): 2 (scheme II) by default for complex double and real, 1
    with oz_crt = 0, 0 with the emulation off and for complex single; after a step the path that
    ran is the one reported."""
    import paper_2205_02491_b200 as pkg
    N, n = 256, 8
    H = make_matrix("uniform", N, "g2", seed=4).dense()
    X = np.ones((N, n), dtype=complex)
    ch = pkg.Chase(N, n, 1)
    assert ch.get_option("ozaki_scheme") == 2
    dY = _dev(np.zeros((N, n), dtype=complex))
    ch.hemm_step(0, _dev(H), _dev(X), dY, n, 1.0, 0.0, 0.0)
    assert ch.get_option("ozaki_scheme") == 2
    ch.set_option("oz_crt", 0)
    assert ch.get_option("ozaki_scheme") == 1 and ch.get_option("oz_crt") == 0
    ch.set_option("fp64_emulation", 0)
    assert ch.get_option("ozaki_scheme") == 0
    assert pkg.Chase(N, n, 1, dtype="r64").get_option("ozaki_scheme") == 2
    assert pkg.Chase(N, n, 1, dtype="c64").get_option("ozaki_scheme") == 0
