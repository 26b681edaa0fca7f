"""Local (communication-free) fused-step rate at a grid shard's shape: emulated grid (world_size=1,
r x c > 1), rank 0's shard p x q of an N x N matrix, `n` columns.  Separates kernel speed from the
all-reduce when reading multi-GPU runs.  Usage: python tools/time_shard_step.py N n dtype r c"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2205_02491_b200 as pkg  # noqa: E402

N, n, dtype, r, c = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
tdt = {"c128": torch.complex128, "c64": torch.complex64}[dtype]
ch = pkg.Chase(N, n - 8, 8, grid=(r, c), rank=0, world_size=1, dtype=dtype)
r0, p, c0, q = ch.local_layout()
H = torch.randn((q, p), dtype=tdt, device="cuda").mul_(1e-3).t()
V = torch.randn((n, q), dtype=tdt, device="cuda").t()
W = torch.zeros((n, p), dtype=tdt, device="cuda").t()
for d in (0, 1):
    ch.hemm_step(d, H, V if d == 0 else W, W if d == 0 else V, n, 1e-3, 0.5, 0.3)
torch.cuda.synchronize()
for d in (0, 1):
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        ch.hemm_step(d, H, V if d == 0 else W, W if d == 0 else V, n, 1e-3, 0.5, 0.3)
        ts.append(time.perf_counter() - t)
    print(json.dumps({"dtype": dtype, "dir": d, "N": N, "grid": f"{r}x{c}", "p": p, "q": q, "n": n, "s": min(ts),
                      "tflops": 8.0 * p * q * n / min(ts) / 1e12}))
