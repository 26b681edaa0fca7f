"""Build the in-tree CUDA libraries for sm_100a with nvcc (no JIT cache; the .so files travel with
the repo snapshot to the GPU box).

  libchase_b200.so   the product library (C ABI in include/chase.h)
  libchase_gen.so    device twin of the seeded input generator (chase_gen/csrc/gen.cu)
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec and spec.submodule_search_locations:
        base = list(spec.submodule_search_locations)[0]
        return os.path.join(base, "include"), os.path.join(base, "lib")
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _stale(out, srcs):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


def build_lib(out, srcs, deps, extra, force=False, verbose=False):
    if not force and not _stale(out, srcs + deps):
        return out
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-Xptxas", "-v" if verbose else "-O3", "-o", out, *srcs, *extra]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed building {os.path.basename(out)}")
    if verbose:
        sys.stderr.write(r.stderr)
    return out


def build(force=False, verbose=False):
    inc, lib = _nccl_dirs()
    csrc = os.path.join(HERE, "csrc")
    srcs = sorted(glob.glob(os.path.join(csrc, "*.cu")))
    deps = sorted(glob.glob(os.path.join(csrc, "*.h")) + glob.glob(os.path.join(csrc, "*.cuh"))
                  + [os.path.join(ROOT, "include", "chase.h")])
    build_lib(os.path.join(HERE, "libchase_b200.so"), srcs, deps,
              [f"-I{inc}", f"-I{os.path.join(ROOT, 'include')}", f"-L{lib}", "-l:libnccl.so.2",
               f"-Xlinker", f"-rpath={lib}"], force, verbose)
    gsrc = os.path.join(ROOT, "chase_gen", "csrc")
    gsrcs = sorted(glob.glob(os.path.join(gsrc, "*.cu")))
    if gsrcs:
        build_lib(os.path.join(ROOT, "chase_gen", "libchase_gen.so"), gsrcs, [], [], force, verbose)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print("built")
