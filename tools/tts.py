"""Time-to-solution of chase_solve on one GPU for a BASELINE config (per-iteration trace with
CHASE_TRACE=1).  Usage: python tools/tts.py N nev nex family max_iter [c128|r64|c64] [tol]"""
import sys, time, json
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2205_02491_b200 as pkg
from chase_gen.dense import G2Matrix, R2Matrix
from chase_gen.spectra import spectrum
from chase_gen.device import device_matrix

N, nev, nex = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
fam = sys.argv[4] if len(sys.argv) > 4 else "uniform"
real = len(sys.argv) > 6 and sys.argv[6] == "r64"
single = len(sys.argv) > 6 and sys.argv[6] == "c64"
tol = float(sys.argv[7]) if len(sys.argv) > 7 else (1e-5 if single else 1e-10)
M = (R2Matrix if real else G2Matrix)(spectrum(fam, N), seed=1)
H = torch.empty((N, N), dtype=torch.float64 if real else torch.complex128, device="cuda").t()
device_matrix(M).fill(H, 0, 0)
if single:
    H = H.to(torch.complex64)
    torch.cuda.synchronize()
dtype = "r64" if real else ("c64" if single else "c128")
ch = pkg.Chase(N, nev, nex, dtype=dtype)
ch.set_option("max_iter", int(sys.argv[5]) if len(sys.argv) > 5 else 100)
import os
if os.environ.get("CHASE_MIXED"):
    ch.set_option("mixed_filter", float(os.environ["CHASE_MIXED"]))
vals, vecs, rep, st = ch.solve(H, nev, nex, deg=20, tol=tol)
normH = np.max(np.abs(M.lam))
print(json.dumps({"N": N, "nev": nev, "nex": nex, "family": fam, "status": st, "t_all": rep["t_all"],
                  "iterations": rep["iterations"], "matvecs": rep["matvecs"],
                  "phases": {k: rep[k] for k in ("t_lanczos", "t_filter", "t_qr", "t_rr", "t_resid")},
                  "dtype": dtype, "tol": tol, "mixed_filter": float(os.environ.get("CHASE_MIXED", "0")),
                  "filter_tflops": rep["filter_flops"] / max(rep["t_filter"], 1e-12) / 1e12,
                  "eig_err_rel": float(np.max(np.abs(vals - M.lam[:nev])) / normH),
                  "eig_err_relmax": float(np.max(np.abs(vals - M.lam[:nev]) / np.abs(M.lam[:nev])))}))
