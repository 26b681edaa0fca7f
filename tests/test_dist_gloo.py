"""Host-side multi-process logic on CPU (gloo, world_size 2): grid shape, shard partition,
nccl-id broadcast and max-over-ranks timing reduction used by bench.py / tools/mgpu_check.py."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from chase_gen import block_partition
from paper_2205_02491_b200.dist import grid_shape, shard, weak_scaled_n, block_range


def test_grid_shape_square_as_possible():
    assert [grid_shape(g) for g in (1, 2, 4, 8, 6, 9)] == [(1, 1), (1, 2), (2, 2), (2, 4), (2, 3), (3, 3)]


def test_shard_matches_block_partition():
    for N in (10, 1001, 30000):
        for g in (1, 2, 4, 6, 8):
            r, c = grid_shape(g)
            rows, cols = block_partition(N, r), block_partition(N, c)
            cover = set()
            for rank in range(g):
                r0, p, c0, q = shard(N, (r, c), rank)
                assert (r0, p) == rows[rank % r] and (c0, q) == cols[rank // r]
                cover.add((r0, c0))
            assert len(cover) == g
    assert block_range(10, 3, 0) == (0, 4)


def test_weak_scaling_keeps_shard_size():
    for g in (1, 2, 4, 8):
        n = weak_scaled_n(30000, g)
        assert abs(n * n / g - 30000 ** 2) / 30000 ** 2 < 1e-3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2205_02491_b200.dist import broadcast_nccl_id, max_over_ranks
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nid = broadcast_nccl_id(rank, make_id=lambda: bytes(range(128)))
    m = max_over_ranks(1.5 + rank)
    q.put((rank, nid == bytes(range(128)), m))
    dist.destroy_process_group()


def test_gloo_two_ranks_id_broadcast_and_max():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == [(0, True, 2.5), (1, True, 2.5)]
