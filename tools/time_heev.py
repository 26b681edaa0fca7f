"""Time the device block-Jacobi Hermitian eigensolver at size n (random Hermitian matrix)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2205_02491_b200 as pkg

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
rng = np.random.default_rng(0)
A = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
A = 0.5 * (A + A.conj().T)
ch = pkg.Chase(n, 1, 1)
dA = torch.from_numpy(np.asfortranarray(A)).t().contiguous().t().cuda()
th = torch.empty(n, dtype=torch.float64, device="cuda")
Z = torch.empty((n, n), dtype=torch.complex128, device="cuda").t()
for rep in range(2):
    G = dA.clone()
    torch.cuda.synchronize()
    t = time.perf_counter()
    sw = ch.heev(G, th, Z)
    torch.cuda.synchronize()
    el = time.perf_counter() - t
    print(f"n={n} sweeps={sw} time={el:.3f}s")
w = np.linalg.eigvalsh(A)
print("max eig err", np.max(np.abs(th.cpu().numpy() - w)) / np.linalg.norm(A, 2))
