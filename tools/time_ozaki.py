"""Time one complex-double fused step (forward and backward) at a bench shape with the FP64 DMMA
kernel and with the Ozaki INT8 emulation (fp64_emulation = S), and report the emulation's error
against the DMMA result.  Usage: python tools/time_ozaki.py [N] [ncols] [S ...] [nodmma] [r64] [crt]
(crt: Ozaki scheme II with 16 CRT moduli instead of S slices)"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2205_02491_b200 as pkg  # noqa: E402
from chase_gen.dense import G2Matrix, R2Matrix  # noqa: E402
from chase_gen.spectra import spectrum  # noqa: E402
from chase_gen.device import device_matrix  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 30000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
Ss = [int(x) for x in sys.argv[3:] if x.isdigit()] or [7]
skip_dmma = "nodmma" in sys.argv[3:]
real = "r64" in sys.argv[3:]
dt = torch.float64 if real else torch.complex128
M = (R2Matrix if real else G2Matrix)(spectrum("uniform", N), seed=1)
H = torch.empty((N, N), dtype=dt, device="cuda").t()
device_matrix(M).fill(H, 0, 0)
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn((n, N), dtype=dt, device="cuda", generator=g).t()
Y0 = torch.randn((n, N), dtype=dt, device="cuda", generator=g).t()
ch = pkg.Chase(N, n, 1, dtype="r64" if real else "c128")
fl = 2.0 if real else 8.0          # algorithmic flop per MAC
ch.set_option("fp64_emulation", 0)            # DMMA reference first


def run(direction, reps=3):
    Y = Y0.t().clone().t()
    ch.hemm_step(direction, H, X, Y, n, 0.7, -0.3, 0.45)     # warm-up (+ shard slices)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        ch.hemm_step(direction, H, X, Y, n, 0.7, -0.3, 0.45)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps * 1e-3
    Y = Y0.t().clone().t()
    ch.hemm_step(direction, H, X, Y, n, 0.7, -0.3, 0.45)
    return t, Y


out = {"N": N, "ncols": n}
ref = {}
for d in (0, 1):
    if skip_dmma:
        break
    t, Y = run(d)
    ref[d] = Y
    out[f"dmma_dir{d}"] = {"s": t, "tflops": fl * N * N * n / t / 1e12}
for S in Ss:
    ch.set_option("fp64_emulation", S)
    ch.set_option("oz_crt", 1 if "crt" in sys.argv[3:] else 0)
    for d in (0, 1):
        t, Y = run(d)
        err = (torch.linalg.norm(Y - ref[d]) / torch.linalg.norm(ref[d])).item() if d in ref else None
        out[f"ozaki{S}_dir{d}"] = {"s": t, "tflops": fl * N * N * n / t / 1e12, "rel_diff_vs_dmma": err}
    print(json.dumps(out), flush=True)
