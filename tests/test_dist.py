"""Multi-process (gloo, world size 2, CPU) checks of the DP / TP partitioning
used by bench.py: every request / head is owned by exactly one rank, and the
TP all-gather reassembles the full [B, H, 512] output in head order."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_10718_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B, H, Dd = 5, 8, 512
        full = torch.arange(B * H * Dd, dtype=torch.float32).view(B, H, Dd)
        lo, hi = D.tp_range(H, world, rank)
        got = D.tp_gather_heads(full[:, lo:hi].contiguous())
        ok_tp = bool(torch.equal(got, full))
        # DP: ranks cover every request exactly once
        lo, hi = D.dp_range(B, world, rank)
        mine = torch.zeros(B, dtype=torch.int64)
        mine[lo:hi] = 1
        dist.all_reduce(mine)
        ok_dp = bool(torch.all(mine == 1))
        # max-over-ranks timing reduction used by bench.py
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        q.put((rank, ok_tp, ok_dp, float(t)))
    finally:
        dist.destroy_process_group()


def test_tp_gather_and_dp_partition_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok_tp, ok_dp, tmax in res:
        assert ok_tp and ok_dp, rank
        assert tmax == float(world)


@pytest.mark.parametrize("B,W", [(64, 8), (5, 2), (1, 4), (128, 3)])
def test_dp_range_covers(B, W):
    seen = []
    for r in range(W):
        lo, hi = D.dp_range(B, W, r)
        seen += list(range(lo, hi))
    assert seen == list(range(B))


def test_tp_range_requires_divisible():
    assert D.tp_range(128, 8, 3) == (48, 64)
    with pytest.raises(ValueError):
        D.tp_range(10, 4, 0)
