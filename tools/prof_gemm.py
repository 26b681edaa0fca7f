"""Profiling target: one forward and one backward fused filter step (zgemm_dmma_kernel) at
N x N H, ncols columns (default N=15000, ncols=3000) -- used under `ncu --set full`."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2205_02491_b200 as pkg
from chase_gen import make_matrix
from chase_gen.device import DeviceG2

N = int(sys.argv[1]) if len(sys.argv) > 1 else 15000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
M = make_matrix("uniform", N, "g2", seed=1)
H = torch.empty((N, N), dtype=torch.complex128, device="cuda").t()
DeviceG2(M).fill(H, 0, 0)
V = torch.randn((n, N), dtype=torch.complex128, device="cuda").t()
W = torch.zeros((n, N), dtype=torch.complex128, device="cuda").t()
ch = pkg.Chase(N, n - 10, 10)
ch.hemm_step(0, H, V, W, n, 1e-3, 0.5, 0.3)
ch.hemm_step(1, H, W, V, n, 1e-3, 0.5, 0.3)
torch.cuda.synchronize()
print("ok", N, n)
