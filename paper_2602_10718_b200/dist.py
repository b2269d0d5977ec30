"""Multi-GPU partitioning of the decode step (the paper's DP / TP
deployments).  One process per GPU, torch.distributed for the
plumbing.

DP  (batch partition): rank r owns requests [r*B/W, (r+1)*B/W) with its own
    pools and block table; no collective on the data path.
TP  (head partition): rank r owns heads [r*H/W, (r+1)*H/W); MLA's latent is
    shared by all heads, so every rank holds (and appends) the full KV cache;
    one all-gather of the BF16 output [B, H/W, 512] per step.
"""
import torch
import torch.distributed as dist


def dp_range(batch, world, rank):
    """Requests [lo, hi) of `rank` when `batch` requests are split over `world` ranks
    (the first batch % world ranks get one extra)."""
    base, extra = divmod(batch, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def tp_range(num_heads, world, rank):
    """Heads [lo, hi) of `rank`; num_heads must divide evenly."""
    if num_heads % world:
        raise ValueError(f"num_heads={num_heads} not divisible by world={world}")
    per = num_heads // world
    return rank * per, (rank + 1) * per


def tp_gather_heads(out_local, group=None, gathered=None):
    """All-gather the head-partitioned output [B, H/W, D] of every rank into
    [B, H, D] (rank-major heads).  `gathered` [W, B, H/W, D] may be preallocated."""
    world = dist.get_world_size(group)
    if gathered is None:
        gathered = torch.empty((world,) + tuple(out_local.shape), dtype=out_local.dtype, device=out_local.device)
    dist.all_gather_into_tensor(gathered.view(-1), out_local.contiguous().view(-1), group=group)
    w, b, hl, d = gathered.shape
    return gathered.permute(1, 0, 2, 3).reshape(b, w * hl, d)
