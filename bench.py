#!/usr/bin/env python
"""Benchmark of the B200-native ChASE hot path.

Step = one ChASE subspace iteration on resident H (the paper's one-iteration protocol,
P:727-731): Lanczos bounds + filter (deg 20 on all nev+nex columns) + CholQR2 + Rayleigh-Ritz +
residuals + locking -- every SURVEY §8(a) row -- through the C ABI (chase_solve, max_iter = 1).

Workload (BASELINE.json configs[1]): complex double, Uniform spectrum (Table 1, d_max=1,
eps=1e-4), N = 30000, nev = 2250, nex = 750, deg = 20, on one B200.  For N>1 GPUs the paper's weak
scaling is used: N = 30000*sqrt(G) on an r x c grid (1x2, 2x2, 2x4), so the H shard per
GPU stays 14.4 GB and per-GPU filter work is fixed.

metric/value: filter TFLOP/s of the whole job = 8 N^2 matvecs / step time (max over ranks), with
the step time measured on the device (CUDA events inside the library, on its stream).

Launch:  python bench.py [--gpus N --steps K --warmup W]          (N = 1)
         torchrun --nproc-per-node N ... bench.py --gpus N ...     (N > 1)
         python bench.py --impl reference ...                      (the CPU oracle arm)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N1, NEV, NEX, DEG = 30000, 2250, 750, 20
METRIC = "filter TFLOP/s, one ChASE subspace iteration (P:727-731), complex double"
# Roofline denominators measured on a B200 by tools/microbench/peaks.cu (run_peaks.sh): FP64 DMMA
# (mma.sync.m8n8k4.f64) and tcgen05 kind::tf32, each as a burst (one ~60 ms launch after idle) and
# sustained (>= 6 s back to back, rate over the last 4 s) figure with the clocks recorded.  The
# timed regions here are seconds long, so the sustained figures are the denominators.
PEAKS_FILE = os.path.join(ROOT, "profiles", "r02_peaks.json")
FALLBACK_DMMA_TFLOPS = 37.12      # r01 short-run measurement (profiles/r01_fp64_peak.jsonl)
BF16_MEASURED_TFLOPS = 1644.0


def load_peaks():
    """(dmma_tflops, tf32_tflops, int8_tops, source) -- sustained measured figures, else labelled fallbacks."""
    try:
        d = json.load(open(PEAKS_FILE))
        return (d["dmma_f64"]["sustained_tflops"], d["tf32_tcgen05"]["sustained_tflops"],
                d["i8_tcgen05"]["sustained_tflops"],
                f"{os.path.relpath(PEAKS_FILE, ROOT)} (sustained, measured by tools/microbench/peaks.cu)")
    except Exception:
        try:
            bf16 = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("bf16_tflops", BF16_MEASURED_TFLOPS)
        except Exception:
            bf16 = BF16_MEASURED_TFLOPS
        return (FALLBACK_DMMA_TFLOPS, 0.5 * bf16, 2.0 * bf16,
                "fallback: r01 short-run DMMA figure; 1/2 and 2 x measured BF16 (nominal TF32 / INT8 ratios)")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="chase", choices=["chase", "reference"])
    ap.add_argument("--order", dest="n", type=int, default=N1, help="matrix order N on 1 GPU (weak-scaled for more)")
    ap.add_argument("--nev", type=int, default=NEV)
    ap.add_argument("--nex", type=int, default=NEX)
    ap.add_argument("--family", default="uniform")
    ap.add_argument("--tts", action="store_true", help="also run a full solve to convergence (time-to-solution); "
                    "default on 1 GPU")
    ap.add_argument("--no-tts", action="store_true", help="skip the time-to-solution solve")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c64", action="store_true", help="skip the complex-single filter sub-measurement")
    ap.add_argument("--no-config3", action="store_true", help="skip the config-3 (N=60000) one-GPU sub-line")
    ap.add_argument("--fp64", default="ozaki", choices=["ozaki", "dmma"],
                    help="complex-double products: ozaki = FP64 emulated on the INT8 tensor cores (library "
                         "default, fp64_emulation = 7), dmma = FP64 DMMA")
    ap.add_argument("--ref-seconds", type=float, default=None, help=argparse.SUPPRESS)   # tests: bound the oracle sample
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: N = n sqrt(G) (paper P:717-718, default); strong: N = n on every G (config 3)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- clocks sampler
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.gpus = set(gpus)
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                idx = int(f[0])
            except ValueError:
                continue
            if self.gpus and idx not in self.gpus:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for name, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        under_load = [s for s in sm if s > 300] or sm
        return {"sm_mhz": statistics.median(under_load) if under_load else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU oracle sample
def oracle_sample(N, seconds=12.0, rows=1024, ncols=64, family="uniform"):
    """The oracle's filter step (oracle.hemm_step, numpy complex128 on the host cores) on a
    bounded sample of the workload: a `rows` x N row panel of H (generated untimed from the same
    seeded G2 description) times a 64-column block, repeated for ~`seconds`.  Returns TFLOP/s."""
    import numpy as np
    import oracle
    from chase_gen.dense import G2Matrix
    from chase_gen.spectra import spectrum
    M = G2Matrix(spectrum(family, N), seed=1)
    Hp = M.block(0, rows, 0, N)
    X = oracle.random_block(2, 0, N, 0, ncols, 0)
    Y = np.zeros((rows, ncols), dtype=np.complex128)
    cores = len(os.sched_getaffinity(0))
    # torchrun exports OMP_NUM_THREADS=1; the oracle baseline runs on all host cores regardless
    try:
        from threadpoolctl import threadpool_limits, threadpool_info
        limiter = threadpool_limits(limits=cores)
        used = max([d.get("num_threads", 1) for d in threadpool_info()] or [1])
    except Exception:
        limiter, used = None, cores
    n, t0 = 0, time.perf_counter()
    while True:
        Y = oracle.hemm_step_rows(Hp, 0, X, Y, 0.5, -0.2, 0.3)
        n += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    if limiter is not None:
        limiter.restore_original_limits()
    cores = used
    flops = 8.0 * rows * N * ncols * n
    return flops / el / 1e12, cores, (f"{n} oracle filter steps (hemm_step, P:385-390) on a {rows} x {N} row panel of H "
                                      f"times {ncols} columns, numpy complex128; host CPU: {_cpu_model()}")


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _threads(n):
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=n)
    except Exception:
        return None


def config1_compare(pkg, gpu=True, runs=3):
    """BASELINE config 1 (N = 1000 complex double Uniform, G1 = Q diag(lambda) Q^H with Haar Q,
    nev 50, nex 25, deg 20, tol 1e-10): the oracle's full solve, best of `runs`, on 1 host thread
    and on all host threads, and the GPU solve (best of `runs`), with the
    eigenvalue agreement of the two."""
    import numpy as np
    import oracle
    from chase_gen import make_matrix
    N, nev, nex = 1000, 50, 25
    M = make_matrix("uniform", N, "g1", seed=1)
    H = M.dense()
    normH = float(np.max(np.abs(M.lam)))
    out = {"what": "BASELINE config 1: N=1000 complex double Uniform (G1), nev=50, nex=25, deg=20, tol=1e-10; best of %d" % runs}
    cores = len(os.sched_getaffinity(0))
    ovals = None
    for label, nthr in (("oracle_all_threads_s", cores), ("oracle_1_thread_s", 1)):
        lim = _threads(nthr)
        best = float("inf")
        for _ in range(runs):
            t0 = time.perf_counter()
            ovals, _, orep = oracle.chase_solve(H, nev, nex, deg=20, tol=1e-10)
            best = min(best, time.perf_counter() - t0)
        if lim is not None:
            lim.restore_original_limits()
        out[label] = best
    out["oracle_threads"] = cores
    out["oracle_iterations"] = orep.iterations
    out["oracle_eig_err_rel"] = float(np.max(np.abs(ovals - M.lam[:nev])) / normH)
    if gpu:
        import torch
        dH = torch.from_numpy(np.asfortranarray(H)).t().contiguous().t().cuda()
        ch = pkg.Chase(N, nev, nex)
        best, rep = float("inf"), None
        for _ in range(runs):
            vals, vecs, rep, st = ch.solve(dH, nev, nex, deg=20, tol=1e-10)
            best = min(best, rep["t_all"])
        V = vecs.cpu().numpy()[:, :nev]
        out.update(gpu_s=best, gpu_iterations=rep["iterations"], gpu_status=st,
                   gpu_eig_err_rel=float(np.max(np.abs(vals - M.lam[:nev])) / normH),
                   gpu_vs_oracle_eig_rel=float(np.max(np.abs(vals - ovals)) / normH),
                   gpu_resid_rel=float(np.max(np.linalg.norm(H @ V - V * vals[None, :], axis=0)) / normH),
                   speedup_vs_oracle_all_threads=out["oracle_all_threads_s"] / best)
        ch.close()
    return out


def projected_oracle_tts(rate_tflops, cases):
    """projected oracle time-to-solution for the large configs = (measured
    matvecs x 8 N^2 + iterations x the per-iteration QR / RR terms) / the oracle's measured rate.
    Per-iteration terms with n = nev + nex (an upper bound: locking shrinks n): RR's H Q 8 N^2 n,
    plus 40 N n^2 for Householder QR + its Q (16 N n^2), Q^H (HQ) (8), Q Z (8) and (HQ) Z (8)."""
    out = []
    for c in cases:
        N, n = float(c["N"]), float(c["nev"] + c["nex"])
        flops = 8.0 * N * N * c["matvecs"] + c["iterations"] * (8.0 * N * N * n + 40.0 * N * n * n)
        out.append(dict(c, projected_oracle_s=flops / (rate_tflops * 1e12), label="projected"))
    return out


def _recorded_tts():
    """Measured (matvecs, iterations) of the large configs from committed GPU runs (profiles/)."""
    cases = []
    for f, cfg in (("r02_config4_121_4gpu_tts.json", "config4 1-2-1"),
                   ("r02_config4_wilkinson_4gpu_tts.json", "config4 Wilkinson")):
        if not os.path.exists(os.path.join(ROOT, "profiles", f)):
            f = f.replace("r02_", "r01_")                     # round-1 (DMMA path) record
        try:
            lines = [ln for ln in open(os.path.join(ROOT, "profiles", f)) if ln.startswith("{")]
            d = json.loads(lines[-1])
            t = d.get("time_to_solution", d)
            cases.append({"config": cfg, "N": d.get("N", d.get("config", {}).get("N")),
                          "nev": d.get("nev", d.get("config", {}).get("nev")),
                          "nex": d.get("nex", d.get("config", {}).get("nex")),
                          "matvecs": t["matvecs"], "iterations": t["iterations"],
                          "gpu_s": t.get("t_all_s", t.get("s")), "gpus": d.get("gpus", d.get("n_gpus")),
                          "source": "profiles/" + f})
        except Exception:
            continue
    return cases


def run_reference(args, out):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    world = args.gpus
    from paper_2205_02491_b200.dist import weak_scaled_n, grid_shape
    N = weak_scaled_n(args.n, world) if args.scaling == "weak" else args.n
    per = max(3.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    if args.ref_seconds:
        per = args.ref_seconds
    for _ in range(args.warmup):
        oracle_sample(N, seconds=per / 3, family=args.family)
    vals, cores, sample = [], 0, ""
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v, cores, sample = oracle_sample(N, seconds=per, family=args.family)
        vals.append(v)
    wall = time.perf_counter() - t0
    v = statistics.mean(vals)
    r, c = grid_shape(world)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall / args.steps * 1e3,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "c128",
            "data": "synthetic (seeded G2 generator, Table 1 spectrum)",
            "config": {"workload": f"config2 (weak-scaled): N={N} complex double {args.family}, nev={args.nev}, nex={args.nex}, deg={DEG}; oracle filter-step sample",
                       "N": N, "grid": f"{r}x{c}"},
            "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), file=out, flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU arm
def _json_out():
    """Keep stdout for the single JSON line: libraries (NCCL's version banner, CUDA) write to fd 1,
    so fd 1 is pointed at stderr for the run and the result goes to the saved descriptor."""
    saved = os.dup(1)
    os.dup2(2, 1)
    return os.fdopen(saved, "w")


def main():
    args = parse()
    out = _json_out()
    if args.impl == "reference":
        return run_reference(args, out)
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2205_02491_b200 as pkg
    from paper_2205_02491_b200.dist import grid_shape, weak_scaled_n, shard, broadcast_nccl_id, max_over_ranks
    from chase_gen.dense import G2Matrix
    from chase_gen.spectra import spectrum
    from chase_gen.device import DeviceG2

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE", file=sys.stderr)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    grid = grid_shape(world)
    N = weak_scaled_n(args.n, world) if args.scaling == "weak" else args.n
    nev, nex = args.nev, args.nex
    row0, p, col0, q = shard(N, grid, rank)

    # ---- input: H shard generated on the device from the seeded G2 description (untimed)
    M = G2Matrix(spectrum(args.family, N), seed=1)
    H = torch.empty((q, p), dtype=torch.complex128, device="cuda").t()        # p x q column-major
    DeviceG2(M).fill(H, row0, col0)
    torch.cuda.synchronize()
    nccl_id = broadcast_nccl_id(rank) if world > 1 else None
    stream = torch.cuda.current_stream().cuda_stream
    ch = pkg.Chase(N, nev, nex, grid=grid, rank=rank, world_size=world, nccl_id=nccl_id, device=local,
                   stream=stream)
    assert ch.local_layout() == (row0, p, col0, q)
    ch.set_option("max_iter", 1)
    EMU = 7 if args.fp64 == "ozaki" else 0
    ch.set_option("fp64_emulation", EMU)
    vecs = torch.empty((nev + nex, q), dtype=torch.complex128, device="cuda").t()

    def step():
        vals, _, rep, st = ch.solve(H, nev, nex, deg=DEG, tol=1e-10, vectors=vecs)
        return rep

    for _ in range(max(3, args.warmup)):
        step()
    # ---- timed region
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
    ids = [int(x) for x in vis.split(",") if x.strip().isdigit()] if vis else list(range(world))
    sampler = ClockSampler(ids[:world] if ids else [])
    sampler.start()
    time.sleep(0.3)
    l0 = pkg.kernel_launches()
    t_wall0 = time.perf_counter()
    reps = [step() for _ in range(args.steps)]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_wall = time.perf_counter() - t_wall0
    launches = pkg.kernel_launches() - l0
    clocks = sampler.stop()
    dev_s = sum(r["t_all"] for r in reps)
    filt_s = sum(r["t_filter"] for r in reps)
    matvecs = sum(r["matvecs"] for r in reps)
    flops = 8.0 * N * N * matvecs
    dev_s_max = max_over_ranks(dev_s)
    filt_s_max = max_over_ranks(filt_s)
    value = flops / dev_s_max / 1e12
    phases = {k: max_over_ranks(sum(r[k] for r in reps)) / args.steps
              for k in ("t_lanczos", "t_filter", "t_qr", "t_rr", "t_resid", "t_all")}

    # ---- end-to-end through the C ABI with HOST buffers: chase_solve reads the shard from pinned
    #      host memory and writes the eigenvectors to host memory; the copies run inside the call,
    #      every step, and the whole call is timed (wall clock around a synchronous call)
    e2e = None
    if not args.no_e2e:
        try:
            Hh = torch.empty((q, p), dtype=torch.complex128, pin_memory=True).t()
            vh = torch.empty((nev, q), dtype=torch.complex128, pin_memory=True).t()
            pinned = True
        except RuntimeError:                     # host cannot pin this much: pageable buffers
            Hh = torch.empty((q, p), dtype=torch.complex128).t()
            vh = torch.empty((nev, q), dtype=torch.complex128).t()
            pinned = False
        Hh.copy_(H)
        ch.solve(Hh, nev, nex, deg=DEG, tol=1e-10, vectors=vh)          # warm-up (staging buffer)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        mv = 0
        for _ in range(args.steps):
            vals, _, rep, st = ch.solve(Hh, nev, nex, deg=DEG, tol=1e-10, vectors=vh)
            mv += rep["matvecs"]
        e2e_s = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": 8.0 * N * N * mv / e2e_s / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": 16 * p * q, "d2h_bytes_per_step": 16 * q * nev + 8 * nev,
               "steps": args.steps, "pinned_host": pinned,
               "how": "chase_solve(H_shard in host memory, ritz_vectors in host memory): the C-ABI call copies "
                      "the shard H2D and the eigenvectors D2H itself; wall time of the synchronous calls, max over ranks"}
        del Hh, vh

    # ---- roofline of the dominant kernel: algorithmic FLOPs / measured filter time
    per_launch_flops = 8.0 * p * q * (nev + nex)        # first iteration: every column at every degree step
    launches_filter = DEG * args.steps
    achieved = flops / world / filt_s_max / 1e12
    dmma_peak, tf32_peak, i8_peak, peak_src = load_peaks()
    traffic = None
    scheme = int(ch.get_option("ozaki_scheme")) if EMU else 0     # 2 = CRT (scheme II), 1 = slices
    prof = os.path.join(ROOT, "profiles", {2: "r02_ncu_ozaki_crt_step.json", 1: "r02_ncu_ozaki_step.json"}.get(
        scheme, "r01_ncu_filter_gemm.json"))
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_step" if scheme else "dram_bytes_per_launch")
        except Exception:
            traffic = None

    def emu_peak(sch):
        # int8 GEMMs per complex MAC: 3 real products (3M) x 16 moduli (scheme II) or x S(S+1)/2
        # slice pairs (S = 7: 28); 2 int8 ops per int8 MAC, 8 algorithmic flop per complex MAC
        prods = 16 if sch == 2 else EMU * (EMU + 1) // 2
        return i8_peak * 8.0 / (2.0 * 3 * prods), 2 * 3 * prods

    if scheme:
        peak_c, ops = emu_peak(scheme)
        what = ("Ozaki scheme II: residues of the 52-bit scaled operands modulo 16 coprime moduli, one int8 GEMM "
                "per modulus, exact CRT reconstruction" if scheme == 2 else f"Ozaki scheme, {EMU} slices")
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak_c, "unit": "TFLOP/s", "frac": achieved / peak_c,
                "traffic": traffic,
                "kernel": "oz_gemm_kernel (filter step: FP64 complex product emulated on INT8 tcgen05 MMAs, "
                          f"{what}, 3M; + residue / reconstruction kernels, all inside the timed filter phase)",
                "per_launch_flops": per_launch_flops, "launches": launches_filter, "unit_of_launch": "one fused filter step",
                "int8_pipe_frac": achieved / peak_c,
                "peak_source": f"INT8 tcgen05 peak {i8_peak:.0f} TOPS ({peak_src}) x 8 / {ops} "
                               "(int8 ops per algorithmic complex flop)"}
    else:
        roof = {"bound": "tensor", "achieved": achieved, "peak": dmma_peak * 4.0 / 3.0, "unit": "TFLOP/s",
                "frac": achieved / (dmma_peak * 4.0 / 3.0), "traffic": traffic,
                "kernel": "zgemm3m_dmma_kernel (filter step: 3M complex product on FP64 DMMA.8x8x4, TMA-staged)",
                "per_launch_flops": per_launch_flops, "launches": launches_filter,
                "dmma_pipe_frac": achieved * 0.75 / dmma_peak,
                "peak_source": f"4/3 x the FP64 DMMA.8x8x4 peak {dmma_peak:.2f} TFLOP/s ({peak_src}): 3M spends 3 real "
                               "DMMA MACs per complex MAC; MEASURED_PEAKS.json has no FP64 entry"}
    # ---- the other complex-double product path on the same H, one iteration (context)
    other = None
    if world == 1 and not args.no_c64:
        ch.set_option("fp64_emulation", 0 if EMU else 7)
        _, _, ro, _ = ch.solve(H, nev, nex, deg=DEG, tol=1e-10, vectors=vecs)
        ch.set_option("fp64_emulation", EMU)
        fo = 8.0 * N * N * ro["matvecs"]
        other = {"what": ("FP64 DMMA" if EMU else "Ozaki INT8 emulation (fp64_emulation = 7)")
                 + " complex-double products, one iteration on the same H (context for the main line)",
                 "value": fo / ro["t_all"] / 1e12, "filter_tflops": fo / ro["t_filter"] / 1e12,
                 "ms_per_step": ro["t_all"] * 1e3, "unit": "TFLOP/s"}
    # ---- complex-single filter on the same workload shape: H rounded to
    #      complex64 once (untimed), chase_filter with every column at degree 20 (20 fused steps)
    c64 = None
    if world == 1 and not args.no_c64:
        peak64 = tf32_peak / 3.0
        H32 = H.to(torch.complex64)
        ch32 = pkg.Chase(N, nev, nex, dtype="c64", device=local, stream=stream)
        V32 = (vecs[:, :nev + nex]).to(torch.complex64)
        W32 = torch.empty((nev + nex, p), dtype=torch.complex64, device="cuda").t()
        degs = [DEG] * (nev + nex)
        lam = M.lam
        b_sup, mu_1, mu_ne = float(lam[-1]) * 1.05, float(lam[0]), float(lam[nev + nex])
        ch32.filter(H32, V32, W32, degs, b_sup, mu_1, mu_ne)          # warm-up (+ H_lo, formats)
        reps64 = 3
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        mv64 = 0
        for _ in range(reps64):
            mv64 += ch32.filter(H32, V32, W32, degs, b_sup, mu_1, mu_ne)
        e1.record()
        torch.cuda.synchronize()
        t64 = e0.elapsed_time(e1) * 1e-3
        a64 = 8.0 * N * N * mv64 / t64 / 1e12
        c64 = {"what": "chase_filter in complex single (CHASE_C64: tcgen05 kind::tf32 3xTF32 on CTA pairs), "
                       f"N={N}, {nev + nex} columns at degree {DEG}, same Uniform H rounded to complex64",
               "tflops": a64, "peak": peak64, "frac": a64 / peak64, "unit": "TFLOP/s", "s_per_filter": t64 / reps64,
               "peak_source": f"TF32 tcgen05 peak {tf32_peak:.1f} TFLOP/s ({peak_src}) / 3 MMAs per real product (3xTF32)"}
        ch32.close()
        del H32, V32, W32
        torch.cuda.empty_cache()
    tts = None
    if (args.tts or world == 1) and not args.no_tts:
        ch.set_option("max_iter", 0)          # default: auto (iterate while converging)
        t0 = time.perf_counter()
        vals, _, rep, st = ch.solve(H, nev, nex, deg=DEG, tol=1e-10, vectors=vecs)
        lam = M.lam[:nev]
        tts = {"what": "chase_solve to tol 1e-10 (default options: max_iter auto) on the same H, library device time, max over ranks",
               "s": max_over_ranks(rep["t_all"]), "status": st, "iterations": rep["iterations"],
               "matvecs": rep["matvecs"], "filter_tflops_per_gpu": 8.0 * N * N * rep["matvecs"] / world / max(rep["t_filter"], 1e-12) / 1e12,
               "max_abs_eig_err_rel": float(np.max(np.abs(vals - lam)) / np.max(np.abs(M.lam)))}
    ch.close()
    del H, vecs
    torch.cuda.empty_cache()

    # ---- BASELINE config 3 on one GPU (N = 60000 Geometric, nev 1000, nex 300; the largest
    #      single-GPU BASELINE config): one subspace iteration, 1 warm-up + 1 timed
    cfg3 = None
    if world == 1 and not args.no_config3 and (args.n, nev, nex) == (N1, NEV, NEX):
        N3, nev3, nex3 = 60000, 1000, 300
        M3 = G2Matrix(spectrum("geometric", N3), seed=1)
        H3 = torch.empty((N3, N3), dtype=torch.complex128, device="cuda").t()
        DeviceG2(M3).fill(H3, 0, 0)
        torch.cuda.synchronize()
        ch3 = pkg.Chase(N3, nev3, nex3, device=local, stream=stream)
        ch3.set_option("max_iter", 1)
        ch3.set_option("fp64_emulation", EMU)
        v3 = torch.empty((nev3 + nex3, N3), dtype=torch.complex128, device="cuda").t()
        ch3.solve(H3, nev3, nex3, deg=DEG, tol=1e-10, vectors=v3)
        _, _, r3, _ = ch3.solve(H3, nev3, nex3, deg=DEG, tol=1e-10, vectors=v3)
        f3 = 8.0 * N3 * N3 * r3["matvecs"]
        scheme3 = int(ch3.get_option("ozaki_scheme")) if EMU else 0
        peak3 = emu_peak(scheme3)[0] if scheme3 else dmma_peak * 4.0 / 3.0
        cfg3 = {"workload": f"config3: N={N3} complex double geometric, nev={nev3}, nex={nex3}, deg={DEG}, one subspace "
                            "iteration (P:727-731), 1x1; 1 warm-up + 1 timed iteration; same product path as the main line",
                "value": f3 / r3["t_all"] / 1e12, "unit": "TFLOP/s", "ms_per_step": r3["t_all"] * 1e3,
                "filter_tflops": f3 / r3["t_filter"] / 1e12,
                "roofline_frac": f3 / r3["t_filter"] / 1e12 / peak3,
                "fp64_products": {0: "FP64 DMMA", 1: "Ozaki slices (the residues of the 57.6 GB shard do not fit)",
                                  2: "Ozaki scheme II"}[scheme3],
                "phases_s": {k: r3[k] for k in ("t_lanczos", "t_filter", "t_qr", "t_rr", "t_resid", "t_all")}}
        ch3.close()
        del H3, v3
        torch.cuda.empty_cache()
    cfg1 = None
    if world == 1 and not args.no_cpu:
        cfg1 = config1_compare(pkg)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": dev_s_max / args.steps * 1e3,
                "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
                "dtype": ("c128 (products: int8 residues -> int32 -> exact CRT -> f64)" if scheme == 2 else
                          "c128 (products: int8 slices -> int32 -> f64)" if scheme == 1 else "c128"),
                "data": f"synthetic (seeded G2 generator: H = Phi P C P^H Phi^H with the Table 1 {args.family} spectrum, d_max=1, eps=1e-4)",
                "config": {"workload": ({(N1, NEV, NEX): "config2", (60000, 1000, 300): "config3",
                                         (115000, 1200, 400): "config4"}.get((args.n, nev, nex), "custom")
                                        + (" (weak-scaled)" if world > 1 and args.scaling == "weak" else ""))
                           + f": N={N} complex double {args.family}, nev={nev}, nex={nex}, deg={DEG}, one subspace iteration (P:727-731)",
                           "N": N, "nev": nev, "nex": nex, "deg": DEG, "grid": f"{grid[0]}x{grid[1]}",
                           "l2": "inputs larger than L2 (H shard %.1f GB >> 126 MB)" % (16e-9 * p * q)},
                "wall_ms_per_step": t_wall / args.steps * 1e3,
                "phases_s_per_step": phases,
                "filter_tflops_per_gpu": achieved,
                "roofline": roof,
                "fp64_products": {2: "Ozaki scheme II on INT8 tensor cores (16 CRT moduli, exact integer products, one "
                                     "FP64 rounding; step error ~9e-15 vs FP64 DMMA; SURVEY f4)",
                                  1: "Ozaki-scheme emulation on INT8 tensor cores (7 slices, step error ~1e-14 vs FP64 "
                                     "DMMA; SURVEY f4)", 0: "FP64 DMMA"}[scheme],
                "clocks": clocks, "gpu_launches": launches, "e2e": e2e}
        if other:
            line["c128_dmma_iteration" if EMU else "c128_ozaki_iteration"] = other
        if tts:
            line["time_to_solution"] = tts
        if c64:
            line["c64_filter"] = c64
        if cfg3:
            line["config3_1gpu"] = cfg3
        if world == 1 and not args.no_cpu:
            v, cores, sample = oracle_sample(N, seconds=12.0, family=args.family)
            lim = _threads(1)
            v1, _, _ = oracle_sample(N, seconds=6.0, family=args.family)
            if lim is not None:
                lim.restore_original_limits()
            cases = _recorded_tts()
            if tts:
                cases.insert(0, {"config": "config2", "N": N, "nev": nev, "nex": nex, "matvecs": tts["matvecs"],
                                 "iterations": tts["iterations"], "gpu_s": tts["s"], "gpus": 1,
                                 "source": "this run's time_to_solution"})
            line["cpu_baseline"] = {"value": v, "unit": "TFLOP/s", "cores": cores, "kind": "oracle", "sample": sample,
                                    "value_1_thread": v1, "config1_full_solve": cfg1,
                                    "projected_time_to_solution": projected_oracle_tts(v, cases)}
        print(json.dumps(line), file=out, flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
