"""Phase times of one ChASE iteration (bench.py's step: max_iter 1 from the same start) at the
config-2 shape on one GPU, for several option sets.

    python tools/time_iteration.py [N] "default" "oz_gemm_min=1e30" "fp64_emulation=0" ...
"""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2205_02491_b200 as pkg          # noqa: E402
from chase_gen.dense import G2Matrix         # noqa: E402
from chase_gen.spectra import spectrum       # noqa: E402
from chase_gen.device import DeviceG2        # noqa: E402

args = sys.argv[1:]
N = int(args.pop(0)) if args and args[0].isdigit() else 30000
specs = args or ["default"]
nev, nex, deg = (2250, 750, 20) if N == 30000 else (N // 40, N // 120, 20)
torch.cuda.set_device(0)
H = torch.empty((N, N), dtype=torch.complex128, device="cuda").t()
DeviceG2(G2Matrix(spectrum("uniform", N), seed=1)).fill(H, 0, 0)
vecs = torch.empty((nev + nex, N), dtype=torch.complex128, device="cuda").t()
for spec in specs:
    ch = pkg.Chase(N, nev, nex)
    ch.set_option("max_iter", 1)
    if spec != "default":
        for kv in spec.split(","):
            k, v = kv.split("=")
            ch.set_option(k, float(v))
    reps = []
    n_rep = int(os.environ.get("TI_REPS", "5"))          # TI_REPS=1: one solve (for ncu launch lists)
    for i in range(n_rep):
        _, _, rep, st = ch.solve(H, nev, nex, deg=deg, tol=1e-10, vectors=vecs)
        if i >= min(2, n_rep - 1):
            reps.append(rep)
    ph = {k: sum(r[k] for r in reps) / len(reps) for k in ("t_lanczos", "t_filter", "t_qr", "t_rr", "t_all")}
    print(json.dumps({"N": N, "spec": spec, **{k: round(v, 4) for k, v in ph.items()}}), flush=True)
    ch.close()
