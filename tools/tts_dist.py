"""Distributed time-to-solution (torchrun, one process per GPU): chase_solve on an r x c grid for a
BASELINE-style config, the shard generated on the device in column chunks (so complex-single
shards never need a complex-double copy).  Rank 0 prints one JSON line.
Usage: torchrun --nproc-per-node G tools/tts_dist.py N nev nex family dtype tol [max_iter]"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_02491_b200 as pkg  # noqa: E402
from paper_2205_02491_b200.dist import grid_shape, shard, broadcast_nccl_id, max_over_ranks  # noqa: E402
from chase_gen.dense import G2Matrix  # noqa: E402
from chase_gen.spectra import spectrum  # noqa: E402
from chase_gen.device import DeviceG2  # noqa: E402


def main():
    N, nev, nex = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    fam, dtype, tol = sys.argv[4], sys.argv[5], float(sys.argv[6])
    max_iter = int(sys.argv[7]) if len(sys.argv) > 7 else 0          # 0: auto (library default)
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    grid = grid_shape(world)
    r0, p, c0, q = shard(N, grid, rank)
    M = G2Matrix(spectrum(fam, N), seed=1)
    gen = DeviceG2(M)
    tdt = {"c128": torch.complex128, "c64": torch.complex64}[dtype]
    H = torch.empty((q, p), dtype=tdt, device="cuda").t()
    chunk = max(1, min(q, (4 << 30) // (16 * p)))
    for j in range(0, q, chunk):
        w = min(chunk, q - j)
        tmp = torch.empty((w, p), dtype=torch.complex128, device="cuda").t()
        gen.fill(tmp, r0, c0 + j)
        H[:, j:j + w].copy_(tmp)
        del tmp
    torch.cuda.synchronize()
    nid = broadcast_nccl_id(rank)
    ch = pkg.Chase(N, nev, nex, grid=grid, rank=rank, world_size=world, nccl_id=nid, device=local, dtype=dtype,
                   stream=torch.cuda.current_stream().cuda_stream)
    ch.set_option("max_iter", max_iter)
    if os.environ.get("CHASE_MIXED"):
        ch.set_option("mixed_filter", float(os.environ["CHASE_MIXED"]))
    vals, vecs, rep, st = ch.solve(H, nev, nex, deg=20, tol=tol)
    t_all = max_over_ranks(rep["t_all"])
    if rank == 0:
        lam = M.lam
        normH = float(np.max(np.abs(lam)))
        err = np.abs(vals - lam[:nev])
        print(json.dumps({"N": N, "nev": nev, "nex": nex, "family": fam, "dtype": dtype, "tol": tol,
                          "grid": f"{grid[0]}x{grid[1]}", "gpus": world, "status": st, "t_all_s": t_all,
                          "iterations": rep["iterations"], "locked": rep["locked"], "matvecs": rep["matvecs"],
                          "phases_rank0": {k: rep[k] for k in ("t_lanczos", "t_filter", "t_qr", "t_rr", "t_resid")},
                          "filter_tflops_per_gpu": 8.0 * N * N * rep["matvecs"] / world / max(rep["t_filter"], 1e-12) / 1e12,
                          "eig_err_rel_normH": float(np.max(err) / normH),
                          "eig_err_rel_max": float(np.max(err / np.maximum(np.abs(lam[:nev]), 1e-300))),
                          "mixed_filter": float(os.environ.get("CHASE_MIXED", "0")),
                          "options": "defaults (fp64_emulation 7 = Ozaki INT8 emulation for complex double, max_iter auto)"
                                     if max_iter == 0 and not os.environ.get("CHASE_MIXED") else f"max_iter {max_iter}"}),
              flush=True)
    ch.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
