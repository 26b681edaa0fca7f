"""Robustness layer without compute-sanitizer (closed on this GPU pool): bounds and
race checks of our own on small cases.

  * Canaries: every output block sits inside a larger buffer whose padding rows (ld > rows) and
    trailing columns hold a sentinel bit pattern; after the call the sentinels must be intact
    (an out-of-bounds store in a GEMM epilogue, a fused-reduce peer store or a format kernel shows
    up here), and the read-only H shard (padded too) must be bitwise unchanged.
  * Determinism as a race detector: the fused f1 reduction (system-scope atomics, last-arriver
    peer stores; co-located 2x2 grid), the complex-single CTA-pair step (TMA, TMEM, cluster
    barriers) and a whole solve are repeated and must give identical bits every time -- a race
    or an unsynchronised read would make some repetition differ.
"""
import os

import numpy as np
import pytest

from chase_gen import make_matrix

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

SENT = {torch.complex128: complex(1.2345e300, -6.789e-300), torch.float64: 1.2345e300,
        torch.complex64: complex(1.2345e30, -6.789e-30)}


def _padded(a, dt, pad_rows=7, pad_cols=3):
    """column-major device buffer (rows+pad_rows) x (cols+pad_cols) of sentinels with `a` in the
    top-left corner; returns (full buffer, view of a)."""
    rows, cols = a.shape
    full = torch.full((cols + pad_cols, rows + pad_rows), SENT[dt], dtype=dt).t()     # ld = rows + pad_rows
    full[:rows, :cols] = torch.from_numpy(a)
    full = full.cuda()
    return full, full[:rows, :cols]


def _sentinels_intact(full, rows, cols, dt):
    h = full.cpu()
    s = torch.tensor(SENT[dt], dtype=dt)
    pad = torch.cat([h[rows:, :].reshape(-1), h[:, cols:].reshape(-1)])
    return bool(torch.all(pad == s))


@pytest.mark.parametrize("dtype", ["c128", "r64", "c64"])
@pytest.mark.parametrize("direction", [0, 1])
def test_canaries_hemm_step_and_filter(dtype, direction):
    import paper_2205_02491_b200 as pkg
    N, n = 516, 37
    real, single = dtype == "r64", dtype == "c64"
    dt = torch.float64 if real else (torch.complex64 if single else torch.complex128)
    npdt = np.float64 if real else (np.complex64 if single else np.complex128)
    M = make_matrix("uniform", N, "r2" if real else "g2", seed=11)
    H = M.dense().astype(npdt)
    rng = np.random.default_rng(3)
    def rnd(r, c):
        a = rng.standard_normal((r, c)) + (0 if real else 1j) * rng.standard_normal((r, c))
        return a.astype(npdt)
    ch = pkg.Chase(N, 40, 8, dtype=dtype)
    Hf, Hv = _padded(H, dt, pad_rows=8 if single else 5, pad_cols=2)     # c64: even ldh
    H0 = Hf.cpu().clone()
    Xf, Xv = _padded(rnd(N, n), dt)
    Yf, Yv = _padded(rnd(N, n), dt)
    ch.hemm_step(direction, Hv, Xv, Yv, n, 0.6, -0.4, 0.3)
    torch.cuda.synchronize()
    assert _sentinels_intact(Yf, N, n, dt)
    assert _sentinels_intact(Xf, N, n, dt)
    assert torch.equal(Hf.cpu(), H0)                # H is read-only
    assert torch.isfinite(torch.view_as_real(Yv.cpu()) if not real else Yv.cpu()).all()
    # filter: V and W padded
    degrees = sorted([0, 2, 4, 6, 10] * 6 + [20] * 7)
    Vf, Vv = _padded(rnd(N, len(degrees)), dt)
    Wf, Wv = _padded(np.zeros((N, len(degrees)), dtype=npdt), dt)
    ch.filter(Hv, Vv, Wv, degrees, M.lam[-1] * 1.01, M.lam[0], M.lam[45])
    torch.cuda.synchronize()
    assert _sentinels_intact(Vf, N, len(degrees), dt)
    assert _sentinels_intact(Wf, N, len(degrees), dt)
    assert torch.equal(Hf.cpu(), H0)
    ch.close()


def test_canaries_solve_vectors():
    """chase_solve writes exactly nev columns of q rows into ritz_vectors (ldv > q)."""
    import paper_2205_02491_b200 as pkg
    N, nev, nex = 400, 20, 10
    M = make_matrix("wilkinson", N, "g2", seed=5)
    ch = pkg.Chase(N, nev, nex)
    Hf, Hv = _padded(M.dense(), torch.complex128)
    H0 = Hf.cpu().clone()
    Vf, Vv = _padded(np.zeros((N, nev), dtype=complex), torch.complex128, pad_rows=9, pad_cols=4)
    vals, _, rep, st = ch.solve(Hv, nev, nex, deg=20, tol=1e-10, vectors=Vv)
    assert st == 0
    assert _sentinels_intact(Vf, N, nev, torch.complex128)
    assert torch.equal(Hf.cpu(), H0)


def test_repeatable_fused_reduce_colocated():
    """Fused f1 reduction on a co-located 2x2 grid, 8 repetitions: identical bits every time."""
    import paper_2205_02491_b200 as pkg
    from paper_2205_02491_b200.dist import run_colocated, shard
    N, grid = 600, (2, 2)
    M = make_matrix("wilkinson", N, "g2", seed=3)
    H = M.dense()
    degrees = sorted([2, 4, 8, 8] + [20] * 30)
    rng = np.random.default_rng(2)
    V = rng.standard_normal((N, len(degrees))) + 1j * rng.standard_normal((N, len(degrees)))
    key = os.urandom(128)

    def rank_fn(rank):
        r0, p, c0, q = shard(N, grid, rank)
        ch = pkg.Chase(N, len(degrees), 4, grid=grid, rank=rank, world_size=4, nccl_id=key, colocated=True)
        try:
            dH = torch.from_numpy(np.asfortranarray(H[r0:r0 + p, c0:c0 + q])).t().contiguous().t().cuda()
            outs = []
            for _ in range(8):
                dV = torch.from_numpy(np.asfortranarray(V[c0:c0 + q])).t().contiguous().t().cuda()
                dW = torch.zeros((len(degrees), p), dtype=torch.complex128, device="cuda").t()
                ch.filter(dH, dV, dW, degrees, M.lam[-1] * 1.01, M.lam[0], M.lam[50])
                outs.append(dV.cpu().numpy())
            return outs
        finally:
            ch.close()

    res = run_colocated(4, rank_fn)
    for outs in res:
        for o in outs[1:]:
            assert np.array_equal(o, outs[0])


def test_repeatable_c64_pair_step_and_solve():
    """Complex-single CTA-pair step (both directions) x 10 and a c128 solve x 2: identical bits."""
    import paper_2205_02491_b200 as pkg
    N, n = 1024, 300
    M = make_matrix("uniform", N, "g2", seed=2)
    H = torch.from_numpy(np.asfortranarray(M.dense().astype(np.complex64))).t().contiguous().t().cuda()
    g = torch.Generator().manual_seed(0)
    X = torch.randn((n, N), dtype=torch.complex64, generator=g).cuda().t()          # N x n column-major
    Y0 = torch.randn((n, N), dtype=torch.complex64, generator=g).cuda().t()
    ch = pkg.Chase(N, n, 8, dtype="c64")
    for d in (0, 1):
        ref = None
        for _ in range(10):
            Y = Y0.t().clone().t()
            ch.hemm_step(d, H, X, Y, n, 0.7, -0.3, 0.45)
            y = Y.cpu()
            if ref is None:
                ref = y
            assert torch.equal(y, ref)
    ch.close()
    M2 = make_matrix("uniform", 800, "g2", seed=9)
    dH = torch.from_numpy(np.asfortranarray(M2.dense())).t().contiguous().t().cuda()
    ch = pkg.Chase(800, 40, 20)
    a = ch.solve(dH, 40, 20, deg=20, tol=1e-10)
    b = ch.solve(dH, 40, 20, deg=20, tol=1e-10)
    assert np.array_equal(a[0], b[0]) and torch.equal(a[1][:, :40].cpu(), b[1][:, :40].cpu())
    assert a[2]["matvecs"] == b[2]["matvecs"]
