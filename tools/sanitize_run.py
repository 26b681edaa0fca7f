"""Small invocations of the library's kernels for compute-sanitizer: run as
  compute-sanitizer --tool {memcheck,racecheck,synccheck} --error-exitcode 99 python tools/sanitize_run.py MODE
MODE: filter-coloc  (2x2 grid as co-located ranks on one GPU: fused f1 epilogue reduction with
                     system-scope atomics and peer stores, plus the all-reduce path)
      c64-step      (complex-single CTA-pair tcgen05 step both ways: TMA, TMEM, cluster barriers)
      solve         (config-1-shape solve, N = 1000 (complex double) and N = 400 (real))
Inputs come from numpy and are copied to the device (no torch kernels in the checked process
besides copies); exits non-zero if a result is wrong, so a sanitizer that perturbs scheduling
cannot hide a race behind a wrong answer."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2205_02491_b200 as pkg  # noqa: E402
from paper_2205_02491_b200.dist import run_colocated, shard  # noqa: E402
from chase_gen import make_matrix  # noqa: E402


def dev(a):
    return torch.from_numpy(np.asfortranarray(a)).t().contiguous().t().cuda()


def filter_coloc():
    N, grid = 256, (2, 2)
    M = make_matrix("wilkinson", N, "g2", seed=3)
    H = M.dense()
    degrees = [2, 4, 4, 6]
    rng = np.random.default_rng(0)
    V = rng.standard_normal((N, 4)) + 1j * rng.standard_normal((N, 4))
    outs = {}
    for fused in (1, 0):
        key = os.urandom(128)

        def rank_fn(rank):
            r0, p, c0, q = shard(N, grid, rank)
            ch = pkg.Chase(N, 4, 4, grid=grid, rank=rank, world_size=4, nccl_id=key, colocated=True)
            try:
                ch.set_option("fused_reduce", fused)
                ch.set_option("fp64_emulation", 0)
                dV = dev(V[c0:c0 + q])
                dW = dev(np.zeros((p, 4), dtype=complex))
                ch.filter(dev(H[r0:r0 + p, c0:c0 + q]), dV, dW, degrees, M.lam[-1] * 1.01, M.lam[0], M.lam[40])
                return c0, q, dV.cpu().numpy()
            finally:
                ch.close()
        res = run_colocated(4, rank_fn)
        full = np.zeros((N, 4), dtype=complex)
        for c0, q, v in res:
            full[c0:c0 + q] = v
        outs[fused] = full
    err = np.linalg.norm(outs[1] - outs[0]) / np.linalg.norm(outs[0])
    assert err <= 1e-13, err


def c64_step():
    N, n = 512, 40
    M = make_matrix("uniform", N, "g2", seed=2)
    H = M.dense().astype(np.complex64)
    rng = np.random.default_rng(1)
    X = (rng.standard_normal((N, n)) + 1j * rng.standard_normal((N, n))).astype(np.complex64)
    Y = (rng.standard_normal((N, n)) + 1j * rng.standard_normal((N, n))).astype(np.complex64)
    ch = pkg.Chase(N, n, 8, dtype="c64")
    H64, X64, Y64 = (a.astype(np.complex128) for a in (H, X, Y))
    for d in (0, 1):
        dY = dev(Y)
        ch.hemm_step(d, dev(H), dev(X), dY, n, 0.7, -0.3, 0.45)
        ref = 0.7 * (H64 @ X64 - 0.45 * X64) - 0.3 * Y64 if d == 0 else 0.7 * (H64.conj().T @ X64 - 0.45 * X64) - 0.3 * Y64
        err = np.linalg.norm(dY.cpu().numpy() - ref) / np.linalg.norm(ref)
        assert err <= 1e-5, (d, err)


def solve():
    for dtype, N, nev, nex, fam in (("c128", 1000, 50, 25, "uniform"), ("r64", 400, 20, 10, "wilkinson")):
        M = make_matrix(fam, N, "r2" if dtype == "r64" else "g2", seed=1)
        H = M.dense()
        ch = pkg.Chase(N, nev, nex, dtype=dtype)
        vals, vecs, rep, st = ch.solve(dev(H), nev, nex, deg=20, tol=1e-10)
        assert st == 0, ch.last_error()
        assert np.max(np.abs(vals - M.lam[:nev])) <= 1e-10 * np.max(np.abs(M.lam))
        ch.close()


if __name__ == "__main__":
    {"filter-coloc": filter_coloc, "c64-step": c64_step, "solve": solve}[sys.argv[1]]()
    print("sanitize_run ok", sys.argv[1])
