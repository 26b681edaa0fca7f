"""Multi-GPU parity through torchrun + NCCL + the fused peer all-reduce, when the
box exposes at least two GPUs (skipped otherwise).  Runs tools/mgpu_check.py, which compares the
distributed fused steps, filter and chase_solve against the oracle / exact spectrum on rank 0."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("dtype", ["c128", "c128-ozaki", "c64", "c64-fused", "r64", "r64-ozaki"])
def test_two_gpu_grid(dtype):
    if _ngpu() < 2:
        pytest.skip("needs >= 2 GPUs")
    env = dict(os.environ, MG_DTYPE=dtype.split("-")[0], CHASE_DEBUG_PEER="1")
    if dtype == "c64-fused":
        env["MG_FUSED_C64"] = "1"
    if dtype.endswith("-ozaki"):
        env["MG_OZAKI"] = "7"          # Ozaki INT8 emulation of the FP64 products + NCCL all-reduce
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29531", os.path.join(ROOT, "tools", "mgpu_check.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert r.returncode == 0 and lines, r.stdout[-2000:] + r.stderr[-2000:]
    res = json.loads(lines[-1])
    assert res["ok"], res
    if dtype in ("c128", "r64"):   # the filter ran through the fused peer all-reduce (f1)
        assert "fused peer all-reduce ready" in r.stderr
    if dtype == "c64-fused":
        assert "fused peer all-reduce ready for complex single" in r.stderr
