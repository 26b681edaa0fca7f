"""Diagnostic: reported vs true (FP64) residuals of a c64 solve; and HQ accuracy of the c64 step."""
import sys, json
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2205_02491_b200 as pkg
from chase_gen.dense import G2Matrix
from chase_gen.spectra import spectrum
from chase_gen.device import device_matrix

N, nev, nex = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
tol = float(sys.argv[4]) if len(sys.argv) > 4 else 1e-4
M = G2Matrix(spectrum("uniform", N), seed=1)
H128 = torch.empty((N, N), dtype=torch.complex128, device="cuda").t()
device_matrix(M).fill(H128, 0, 0)
H = H128.to(torch.complex64)
Hr = H.to(torch.complex128)            # the c64 shard, exactly, in c128
ch = pkg.Chase(N, nev, nex, dtype="c64")
ch.set_option("max_iter", 30)
vals, vecs, rep, st = ch.solve(H, nev, nex, deg=20, tol=tol)
V = vecs[:, :nev].to(torch.complex128)
th = torch.tensor(vals, device="cuda", dtype=torch.float64)
R = Hr @ V - V * th[None, :]
nu = rep["nu"]
true_res = (torch.linalg.norm(R, dim=0) / nu).cpu().numpy()
orth = torch.linalg.norm(V.conj().T @ V - torch.eye(nev, device="cuda", dtype=torch.complex128)).item()
# HQ accuracy of the c64 forward step on orthonormal Q
Q, _ = torch.linalg.qr(torch.randn(N, 64, dtype=torch.complex128, device="cuda"))
Qf = Q.to(torch.complex64).t().contiguous().t()
W = torch.zeros((64, N), dtype=torch.complex64, device="cuda").t()
ch.hemm_step(0, H, Qf, W, 64, 1.0, 0.0, 0.0)
ref = Hr @ Qf.to(torch.complex128)
err = (torch.linalg.norm(W.to(torch.complex128) - ref, dim=0) / torch.linalg.norm(ref, dim=0)).max().item()
print(json.dumps({"N": N, "status": st, "iters": rep["iterations"], "max_resid_reported": rep["max_resid"],
                  "true_res_max": float(true_res.max()), "true_res_median": float(np.median(true_res)),
                  "orth": orth, "hq_col_relerr_max": err,
                  "eig_err": float(np.max(np.abs(vals - M.lam[:nev])) / np.max(np.abs(M.lam)))}))
