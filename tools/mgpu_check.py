"""Multi-GPU parity check of the distributed path (one process per GPU, NCCL inside the library).

Run:  torchrun --nproc-per-node G --master-addr 127.0.0.1 --master-port 29511 tools/mgpu_check.py
Each rank owns H_ij of an r x c grid; rank 0 compares the distributed fused steps, filter and
chase_solve with the CPU oracle / exact spectrum.  Prints one JSON line per check on rank 0 and
exits non-zero on any failure."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2205_02491_b200 as pkg  # noqa: E402
from paper_2205_02491_b200.dist import grid_shape, shard, broadcast_nccl_id  # noqa: E402
from chase_gen import make_matrix  # noqa: E402


def dev(a):
    return torch.from_numpy(np.asfortranarray(a)).t().contiguous().t().cuda()


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    grid = grid_shape(world)
    if os.environ.get("MG_GRID"):                       # e.g. "1x4": a row communicator of 4 ranks
        grid = tuple(int(x) for x in os.environ["MG_GRID"].split("x"))
    dtype = os.environ.get("MG_DTYPE", "c128")
    real, single = dtype == "r64", dtype == "c64"
    # c64: TMA operand layout needs q % 4 == 0 and even p -> N = 1200 by default
    N, nev, nex = int(os.environ.get("MG_N", "1200" if single else "1201")), 40, 20
    M = make_matrix("wilkinson", N, "r2" if real else "g2", seed=3)
    H = M.dense()
    if single:
        H = H.astype(np.complex64).astype(np.complex128)     # the c64 shard, exactly
    cast = (lambda a: a.astype(np.complex64)) if single else (lambda a: a)
    tol = 1e-5 if single else 1e-10
    r0, p, c0, q = shard(N, grid, rank)
    nid = broadcast_nccl_id(rank)
    # c64 keeps its operand formats in the handle: size them for the 804-column pipelined filter check
    ch = pkg.Chase(N, 800 if single else nev, nex, grid=grid, rank=rank, world_size=world, nccl_id=nid, device=local,
                   dtype=dtype)
    assert ch.local_layout() == (r0, p, c0, q)
    if os.environ.get("MG_FUSED_C64"):
        ch.set_option("fused_reduce_c64", 1)
    if not single:
        ch.set_option("fp64_emulation", int(os.environ.get("MG_OZAKI", "0")))   # 0: DMMA + fused f1 epilogue
    dH = dev(cast(H[r0:r0 + p, c0:c0 + q]))
    ok = True
    out = []
    rng = np.random.default_rng(0)
    n = 37
    X = rng.standard_normal((N, n)) + (0 if real else 1j) * rng.standard_normal((N, n))
    Y0 = rng.standard_normal((N, n)) + (0 if real else 1j) * rng.standard_normal((N, n))
    if single:
        X, Y0 = cast(X).astype(np.complex128), cast(Y0).astype(np.complex128)
    ref = oracle.hemm_step(H, X, Y0, 0.7, -0.3, 0.45)
    # forward: X V-layout (rows c0..), Y W-layout (rows r0..)
    dY = dev(cast(Y0[r0:r0 + p]))
    ch.hemm_step(0, dH, dev(cast(X[c0:c0 + q])), dY, n, 0.7, -0.3, 0.45)
    e_f = np.linalg.norm(dY.cpu().numpy() - ref[r0:r0 + p]) / np.linalg.norm(ref[r0:r0 + p])
    dY = dev(cast(Y0[c0:c0 + q]))
    ch.hemm_step(1, dH, dev(cast(X[r0:r0 + p])), dY, n, 0.7, -0.3, 0.45)
    e_b = np.linalg.norm(dY.cpu().numpy() - ref[c0:c0 + q]) / np.linalg.norm(ref[c0:c0 + q])
    # filter
    degrees = np.sort(np.array([0, 2, 4, 8, 12, 20, 20, 36] + [20] * 20))
    V = oracle.random_block(9, 0, N, 0, len(degrees), 0)
    V = V.real.copy() if real else cast(V).astype(np.complex128)
    dV = dev(cast(V[c0:c0 + q]))
    dt = torch.float64 if real else (torch.complex64 if single else torch.complex128)
    dW = torch.zeros((len(degrees), p), dtype=dt, device="cuda").t()
    b_sup, mu_1, mu_ne = M.lam[-1] * 1.01, M.lam[0], M.lam[60]
    mv = ch.filter(dH, dV, dW, degrees, b_sup, mu_1, mu_ne)
    fref, _ = oracle.chebyshev_filter(H, V, degrees, b_sup, mu_1, mu_ne)
    e_filt = np.linalg.norm(dV.cpu().numpy() - fref[c0:c0 + q]) / np.linalg.norm(fref[c0:c0 + q])
    # pipelined filter (column chunks, all-reduce overlapped with the next chunk's GEMM)
    degrees2 = np.sort(np.concatenate([np.full(300, 8), np.full(500, 20), np.array([2, 4, 36, 36])]))
    V2 = oracle.random_block(11, 0, N, 0, len(degrees2), 0)
    V2 = V2.real.copy() if real else cast(V2).astype(np.complex128)
    dV2 = dev(cast(V2[c0:c0 + q]))
    dW2 = torch.zeros((len(degrees2), p), dtype=dt, device="cuda").t()
    ch.filter(dH, dV2, dW2, degrees2, b_sup, mu_1, mu_ne)
    fref2, _ = oracle.chebyshev_filter(H, V2, degrees2, b_sup, mu_1, mu_ne)
    e_filt2 = np.linalg.norm(dV2.cpu().numpy() - fref2[c0:c0 + q]) / np.linalg.norm(fref2[c0:c0 + q])
    e_filt = max(e_filt, e_filt2)
    # full solve
    vals, dvecs, rep, st = ch.solve(dH, nev, nex, deg=20, tol=tol)
    vecs_local = dvecs.cpu().numpy()[:, :nev].astype(float if real else complex)
    # assemble the V-layout eigenvectors (rows c0..c0+q) from the first row of ranks (i = 0)
    parts = [None] * world
    dist.all_gather_object(parts, (r0, p, c0, q, vecs_local, rank % grid[0]))
    errs = dict(fwd=e_f, bwd=e_b, filter=e_filt)
    errs = {k: max(v2 for v2 in [v]) for k, v in errs.items()}
    all_errs = [None] * world
    dist.all_gather_object(all_errs, (errs, vals.tolist(), st, rep["iterations"]))
    if rank == 0:
        normH = np.max(np.abs(M.lam))
        full = np.zeros((N, nev), dtype=float if real else complex)
        for (rr0, pp, cc0, qq, vl, i) in parts:
            if i == 0:
                full[cc0:cc0 + qq] = vl
        res = np.max(np.linalg.norm(H @ full - full * np.array(vals)[None, :], axis=0)) / normH
        e_eig = np.max(np.abs(np.array(vals) - M.lam[:nev])) / normH
        ov, _, orep = oracle.chase_solve(H, nev, nex, deg=20, tol=tol)
        same_vals = all(np.array_equal(np.array(a[1]), np.array(all_errs[0][1])) for a in all_errs)
        line = {"world": world, "grid": f"{grid[0]}x{grid[1]}", "N": N, "dtype": dtype,
                "max_step_rel_err": max(max(a[0]["fwd"], a[0]["bwd"]) for a in all_errs),
                "max_filter_rel_err": max(a[0]["filter"] for a in all_errs),
                "solve_status": [a[2] for a in all_errs], "iterations": [a[3] for a in all_errs],
                "oracle_iterations": orep.iterations, "eig_err_rel": e_eig, "resid_rel": res,
                "eig_vs_oracle": float(np.max(np.abs(np.array(vals) - ov)) / normH),
                "ritz_identical_on_all_ranks": same_vals,
                "orth": float(np.max(np.abs(full.conj().T @ full - np.eye(nev))))}
        # c64 bars (tests/test_gpu_c64.py): step 1e-5, filter 1e-4, eigenvalues 2e-5 ||H||, residual 1e-4
        t_step, t_filt, t_eig, t_res, t_orth = (1e-5, 1e-4, 2e-5, 1e-4, 1e-5) if single else \
            (1e-13, 1e-11, 1e-10, 1e-10, 1e-12)
        ok = (line["max_step_rel_err"] <= t_step and line["max_filter_rel_err"] <= t_filt and e_eig <= t_eig
              and res <= t_res and all(s == 0 for s in line["solve_status"]) and same_vals
              and line["orth"] <= t_orth)
        line["ok"] = bool(ok)
        print(json.dumps(line), flush=True)
    okt = [ok]
    dist.broadcast_object_list(okt, src=0)
    ch.close()
    dist.destroy_process_group()
    return 0 if okt[0] else 1


if __name__ == "__main__":
    sys.exit(main())
