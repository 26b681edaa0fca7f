"""Quick timing of one fused filter step (forward + backward) at a given shape on one B200."""
import sys, time, json
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2205_02491_b200 as pkg
from chase_gen import make_matrix
from chase_gen.device import DeviceG2

real = len(sys.argv) > 3 and sys.argv[3] == "r64"
single = len(sys.argv) > 3 and sys.argv[3] == "c64"
N = int(sys.argv[1]) if len(sys.argv) > 1 else 30000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
from chase_gen.device import device_matrix
dt = torch.float64 if real else (torch.complex64 if single else torch.complex128)
M = make_matrix("uniform", N, "r2" if real else "g2", seed=1)
H = torch.empty((N, N), dtype=torch.float64 if real else torch.complex128, device="cuda").t()
device_matrix(M).fill(H, 0, 0)
H = H.to(dt)
V = torch.randn((n, N), dtype=dt, device="cuda").t()
W = torch.zeros((n, N), dtype=dt, device="cuda").t()
ch = pkg.Chase(N, n - 10, 10, dtype="r64" if real else ("c64" if single else "c128"))
if not real and not single:
    ch.set_option("gemm3m", 1 if (len(sys.argv) <= 3 or sys.argv[3] == "3m") else 0)
for d in (0, 1):
    ch.hemm_step(d, H, V if d == 0 else W, W if d == 0 else V, n, 1e-3, 0.5, 0.3)
torch.cuda.synchronize()
for d in (0, 1):
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        ch.hemm_step(d, H, V if d == 0 else W, W if d == 0 else V, n, 1e-3, 0.5, 0.3)
        ts.append(time.perf_counter() - t)
    flops = (2.0 if real else 8.0) * N * N * n
    print(json.dumps({"algo": sys.argv[3] if len(sys.argv) > 3 else "3m", "dir": d, "N": N, "n": n, "s": min(ts), "tflops": flops / min(ts) / 1e12}))
