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


# ---- DP x TP hybrid (NEXT-4(c)): world 4 = DP2 x TP2, gloo on CPU
def _hybrid_worker(rank, world, tp, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B, H, Dd = 6, 8, 512
        full = torch.arange(B * H * Dd, dtype=torch.float32).view(B, H, Dd)
        d, t = D.dptp_coords(world, tp, rank)
        group = D.dptp_groups(world, tp)
        b0, b1 = D.dp_range(B, world // tp, d)
        h0, h1 = D.tp_range(H, tp, t)
        got = D.tp_gather_heads(full[b0:b1, h0:h1].contiguous(), group=group)
        ok_gather = bool(torch.equal(got, full[b0:b1]))
        # every (request, head) computed by exactly one rank
        own = torch.zeros(B, H, dtype=torch.int64)
        own[b0:b1, h0:h1] = 1
        dist.all_reduce(own)
        D.stream_barrier(group=group)
        q.put((rank, ok_gather, bool(torch.all(own == 1))))
    finally:
        dist.destroy_process_group()


def test_dptp_hybrid_gloo():
    world, tp = 4, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_hybrid_worker, args=(r, world, tp, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok_gather, ok_own in res:
        assert ok_gather and ok_own, rank


def test_dptp_coords():
    assert [D.dptp_coords(8, 2, r) for r in range(4)] == [(0, 0), (0, 1), (1, 0), (1, 1)]
    assert D.dptp_coords(8, 8, 5) == (0, 5)
    with pytest.raises(ValueError):
        D.dptp_coords(6, 4, 0)
