"""Multi-rank data plane on ONE GPU (e, f1): the r*c ranks of a grid run as
threads of this process, each with its own handle on cuda:0 (chase_init_args.colocated), so the
driver's single-GPU box exercises the row / column all-reduces, the fused last-arriver epilogue
reduction (f1) and the pipelined all-reduce path against the CPU oracle.

Per grid (1x2, 2x2, 2x4) and transport (fused f1 epilogue / all-reduce path, c128 / r64 / c64):
  * one fused step each way (a2+a3, a4+a5) vs oracle.hemm_step, element-wise:
    max |Y - Y_ref| <= tol * max |Y_ref| with tol = 1e-13 (c128, r64) / 1e-5 (c64);
  * the full filter (a1-a5, mixed degrees 0..36) vs oracle.chebyshev_filter, per column 1e-11 / 1e-4;
  * chase_solve vs the exact spectrum and the oracle's eigenvalues (1e-10 ||H|| / 2e-5 ||H||);
  * replicas bitwise identical: the V-layout outputs of the ranks of one column communicator, and
    the Ritz values of all ranks (ledger #20).
The tolerances are the single-GPU ones: a sum over the grid is the same length-K
dot product split into r or c partial sums."""
import os

import numpy as np
import pytest

import oracle
from chase_gen import make_matrix

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

GRIDS = [(1, 2), (2, 2), (2, 4)]
# c128-fused: FP64 DMMA steps with the f1 epilogue reduction; c128-allreduce: the default complex-
# double path (Ozaki INT8 emulation of the FP64 products, fp64_emulation = 7) with the pipelined
# all-reduce
MODES = ["c128-fused", "c128-allreduce", "r64-fused", "r64-allreduce", "c64-fused", "c64-allreduce"]
NEV, NEX = 40, 20


def _dev(a, dt):
    t = torch.from_numpy(np.asfortranarray(a.astype(dt)))
    return t.t().contiguous().t().cuda()


_CACHE = {}


def _problem(dtype):
    """H (host), exact spectrum, step / filter inputs and the oracle's references (cached)."""
    if dtype in _CACHE:
        return _CACHE[dtype]
    real, single = dtype == "r64", dtype == "c64"
    N = 1200 if single else 1201            # c64: every shard needs q % 4 == 0 and even p
    M = make_matrix("wilkinson", N, "r2" if real else "g2", seed=3)
    H = M.dense()
    if single:
        H = H.astype(np.complex64).astype(np.complex128)      # the complex64 shard, exactly
    rng = np.random.default_rng(0)
    n = 37

    def rnd(shape):
        a = rng.standard_normal(shape) + (0 if real else 1j) * rng.standard_normal(shape)
        return a.astype(np.complex64).astype(np.complex128) if single else a

    X, Y0 = rnd((N, n)), rnd((N, n))
    ab = (0.7, -0.3, 0.45)
    step_ref = oracle.hemm_step(H, X, Y0, *ab)
    degrees = np.sort(np.array([0, 2, 4, 8, 12, 20, 20, 36] + [20] * 20 + [6] * 9))
    V = oracle.random_block(9, 0, N, 0, len(degrees), 0)
    V = V.real.copy() if real else (V.astype(np.complex64).astype(np.complex128) if single else V)
    bounds = (M.lam[-1] * 1.01, M.lam[0], M.lam[60])
    filt_ref, mv = oracle.chebyshev_filter(H, V, degrees, *bounds)
    tol = 1e-5 if single else 1e-10
    ovals, _, _ = oracle.chase_solve(H, NEV, NEX, deg=20, tol=tol)
    _CACHE[dtype] = dict(N=N, M=M, H=H, X=X, Y0=Y0, ab=ab, n=n, step_ref=step_ref, degrees=degrees, V=V,
                         bounds=bounds, filt_ref=filt_ref, mv=mv, tol=tol, ovals=ovals, real=real, single=single)
    return _CACHE[dtype]


@pytest.mark.parametrize("grid", GRIDS, ids=lambda g: f"{g[0]}x{g[1]}")
@pytest.mark.parametrize("mode", MODES)
def test_colocated_grid(grid, mode, capfd, monkeypatch):
    import paper_2205_02491_b200 as pkg
    from paper_2205_02491_b200.dist import run_colocated, shard

    dtype, transport = mode.split("-")
    P = _problem(dtype)
    N, H, n = P["N"], P["H"], P["n"]
    real, single = P["real"], P["single"]
    hdt = np.float64 if real else (np.complex64 if single else np.complex128)
    tdt = torch.float64 if real else (torch.complex64 if single else torch.complex128)
    world = grid[0] * grid[1]
    key = os.urandom(128)
    monkeypatch.setenv("CHASE_DEBUG_PEER", "1")
    if transport == "allreduce":
        monkeypatch.setenv("CHASE_FILTER_CHUNKS", "3")     # pipelined all-reduce path (a3/a5 overlap)

    def rank_fn(rank):
        r0, p, c0, q = shard(N, grid, rank)
        ch = pkg.Chase(N, NEV, NEX, grid=grid, rank=rank, world_size=world, nccl_id=key, dtype=dtype,
                       colocated=True)
        try:
            assert ch.local_layout() == (r0, p, c0, q)
            if transport == "allreduce":
                ch.set_option("fused_reduce", 0)
            elif single:
                ch.set_option("fused_reduce_c64", 1)
            else:
                ch.set_option("fp64_emulation", 0)      # the fused epilogue lives in the DMMA kernels
            dH = _dev(H[r0:r0 + p, c0:c0 + q], hdt)
            out = {"r0": r0, "p": p, "c0": c0, "q": q, "i": rank % grid[0], "j": rank // grid[0]}
            # a2 + a3: forward step, W-layout rows [r0, r0+p)
            dY = _dev(P["Y0"][r0:r0 + p], hdt)
            ch.hemm_step(0, dH, _dev(P["X"][c0:c0 + q], hdt), dY, n, *P["ab"])
            out["fwd"] = dY.cpu().numpy()
            # a4 + a5: backward step on the same shard, V-layout rows [c0, c0+q)
            dY = _dev(P["Y0"][c0:c0 + q], hdt)
            ch.hemm_step(1, dH, _dev(P["X"][r0:r0 + p], hdt), dY, n, *P["ab"])
            out["bwd"] = dY.cpu().numpy()
            # a1-a5: the filter (f1 fused epilogue or the pipelined all-reduce path)
            dV = _dev(P["V"][c0:c0 + q], hdt)
            dW = torch.zeros((len(P["degrees"]), p), dtype=tdt, device="cuda").t()
            out["mv"] = ch.filter(dH, dV, dW, P["degrees"], *P["bounds"])
            out["filt"] = dV.cpu().numpy()
            # Alg. 1 end to end
            vals, vecs, rep, st = ch.solve(dH, NEV, NEX, deg=20, tol=P["tol"])
            out.update(vals=vals, vecs=vecs.cpu().numpy()[:, :NEV], st=st, it=rep["iterations"])
            return out
        finally:
            ch.close()

    res = run_colocated(world, rank_fn)
    err = capfd.readouterr().err
    step_tol, filt_tol, eig_tol = (1e-5, 1e-4, 2e-5) if single else (1e-13, 1e-11, 1e-10)
    ref = P["step_ref"]
    for o in res:
        fr = ref[o["r0"]:o["r0"] + o["p"]]
        br = ref[o["c0"]:o["c0"] + o["q"]]
        assert np.max(np.abs(o["fwd"] - fr)) <= step_tol * np.max(np.abs(fr)), ("fwd", o["i"], o["j"])
        assert np.max(np.abs(o["bwd"] - br)) <= step_tol * np.max(np.abs(br)), ("bwd", o["i"], o["j"])
        fl = P["filt_ref"][o["c0"]:o["c0"] + o["q"]]
        colerr = np.linalg.norm(o["filt"] - fl, axis=0) / np.maximum(np.linalg.norm(fl, axis=0), 1e-300)
        assert np.max(colerr) <= filt_tol, (o["i"], o["j"], float(np.max(colerr)))
        assert o["mv"] == P["mv"]
        assert o["st"] == 0
    # replicas: identical bits within each column communicator (same j), Ritz values everywhere
    for o in res:
        for o2 in res:
            if o2["j"] == o["j"]:
                assert np.array_equal(o["filt"], o2["filt"])
                assert np.array_equal(o["bwd"], o2["bwd"])
                assert np.array_equal(o["vecs"], o2["vecs"])
            if o2["i"] == o["i"]:
                assert np.array_equal(o["fwd"], o2["fwd"])
        assert np.array_equal(o["vals"], res[0]["vals"])
        assert o["it"] == res[0]["it"]
    normH = np.max(np.abs(P["M"].lam))
    vals = res[0]["vals"]
    assert np.max(np.abs(vals - P["M"].lam[:NEV])) <= eig_tol * normH
    assert np.max(np.abs(vals - P["ovals"])) <= eig_tol * normH
    full = np.zeros((N, NEV), dtype=float if real else complex)
    for o in res:
        if o["i"] == 0:
            full[o["c0"]:o["c0"] + o["q"]] = o["vecs"]
    resid = np.max(np.linalg.norm(H @ full - full * vals[None, :], axis=0)) / normH
    assert resid <= (1e-4 if single else 1e-10)
    # the transport that actually ran
    if transport == "fused":
        msg = "fused peer all-reduce ready for complex single" if single else "fused peer all-reduce ready"
        assert msg in err, err[-2000:]
    else:
        assert "fused peer all-reduce ready" not in err


def test_colocated_auto_grid_and_shapes():
    """chase_init with grid 0,0 picks r <= c, |r - c| minimal (ledger #19) for world
    = 2, 4, 6, 8 (co-located ranks, no compute)."""
    import paper_2205_02491_b200 as pkg
    from paper_2205_02491_b200.dist import run_colocated, shard, grid_shape

    expect = {2: (1, 2), 4: (2, 2), 6: (2, 3), 8: (2, 4)}
    for world, grid in expect.items():
        assert grid_shape(world) == grid
        key = os.urandom(128)
        N = 101

        def rank_fn(rank):
            ch = pkg.Chase(N, 4, 4, grid=(0, 0), rank=rank, world_size=world, nccl_id=key, colocated=True)
            try:
                return ch.local_layout()
            finally:
                ch.close()

        lay = run_colocated(world, rank_fn)
        assert lay == [shard(N, grid, r) for r in range(world)], (world, lay)


def test_colocated_uneven_c64_layout_agreed():
    """A complex-single grid whose shards violate the TMA layout (q % 4, even p) is refused at
    chase_init on EVERY rank (decided from the global N, r, c), never half-way into collectives."""
    import paper_2205_02491_b200 as pkg
    from paper_2205_02491_b200._lib import ChaseError
    from paper_2205_02491_b200.dist import run_colocated

    key = os.urandom(128)
    world, N = 4, 1202          # 1x4: column blocks 301, 301, 300, 300 -> q % 4 fails on some ranks

    def rank_fn(rank):
        try:
            pkg.Chase(N, 8, 8, grid=(1, 4), rank=rank, world_size=world, nccl_id=key, dtype="c64",
                      colocated=True)
        except ChaseError as e:
            return e.status
        return 0

    assert run_colocated(world, rank_fn) == [2] * world
