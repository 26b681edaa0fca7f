"""Host-side plumbing for one-process-per-GPU runs (torch.distributed is the control plane only;
every data-path collective is the library's own NCCL call inside libchase_b200.so).

  grid_shape(G)        r x c "as square as possible" with r <= c
  weak_scaled_n(N1, G) matrix order keeping N^2/G fixed (paper's weak scaling)
  block_range(n, k, i) ledger #19 block partition (first n mod k blocks one longer)
  shard(N, grid, rank) (row0, p, col0, q) of rank = i + j*r
  broadcast_nccl_id    rank 0 draws the ncclUniqueId through the library, everyone receives it
  max_over_ranks(x)    float max over the process group (timing rule: max over ranks)
  run_colocated(G, fn) G ranks as threads of one process on one GPU (chase_init_args.colocated)
"""
from __future__ import annotations

import math


def grid_shape(world: int):
    r = int(math.isqrt(world))
    while r > 1 and world % r:
        r -= 1
    return r, world // r


def weak_scaled_n(n1: int, world: int) -> int:
    return int(round(n1 * math.sqrt(world)))


def block_range(n: int, parts: int, idx: int):
    base, rem = divmod(n, parts)
    return idx * base + min(idx, rem), base + (1 if idx < rem else 0)


def shard(N: int, grid, rank: int):
    r, c = grid
    i, j = rank % r, rank // r
    row0, p = block_range(N, r, i)
    col0, q = block_range(N, c, j)
    return row0, p, col0, q


def broadcast_nccl_id(rank: int, make_id=None):
    """Rank 0 creates the 128-byte id (make_id(), default: the library's ncclGetUniqueId) and
    broadcasts it over the default process group."""
    import torch.distributed as dist
    obj = [None]
    if rank == 0:
        if make_id is None:
            from ._lib import nccl_unique_id
            make_id = nccl_unique_id
        obj[0] = bytes(make_id())
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def max_over_ranks(x: float) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_colocated(world: int, fn, device: int = 0, timeout: float = 900.0):
    """Run fn(rank) for rank = 0..world-1 on `world` threads of this process (the co-located mode
    of chase_init_args.colocated: every rank's handle on `device`, communicators in-process).
    Returns the per-rank results; re-raises the first rank's exception.  Each rank's collective
    library calls block until all ranks make them, so the threads must run concurrently (ctypes
    releases the GIL inside the library)."""
    import threading
    results, errors = [None] * world, [None] * world

    def body(rank):
        try:
            import torch
            torch.cuda.set_device(device)
            results[rank] = fn(rank)
        except BaseException as e:     # noqa: BLE001 -- re-raised on the caller's thread
            errors[rank] = e

    threads = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout)
    if any(t.is_alive() for t in threads):
        raise TimeoutError(f"co-located ranks did not finish within {timeout} s")
    for e in errors:
        if e is not None:
            raise e
    return results
