"""Multi-GPU partitioning of the decode step (the paper's DP / TP
deployments).  One process per GPU, torch.distributed for the
plumbing.

DP  (batch partition): rank r owns requests [r*B/W, (r+1)*B/W) with its own
    pools and block table; no collective on the data path.
TP  (head partition): rank r owns heads [r*H/W, (r+1)*H/W); MLA's latent is
    shared by all heads, so every rank holds (and appends) the full KV cache;
    one all-gather of the BF16 output [B, H/W, 512] per step -- NCCL
    (tp_gather_heads) or fused into the combine epilogue as peer stores
    (mla_combine_gather over symmetric-memory buffers, NEXT-4(c)).
DPxTP (hybrid, the paper's DP4/TP2-style deployments): world = D x T;
    rank r = d * T + t owns requests dp_range(B, D, d) and heads
    tp_range(H, T, t); the T ranks of a DP replica (consecutive ranks) form
    the TP group that gathers heads.
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


def dptp_coords(world, tp, rank):
    """(dp index, tp index) of `rank` in a world = (world // tp) x tp grid; TP groups are
    consecutive ranks."""
    if tp < 1 or world % tp:
        raise ValueError(f"world={world} not divisible by tp={tp}")
    return rank // tp, rank % tp


def dptp_groups(world, tp):
    """Create the TP subgroups {d*tp, ..., d*tp + tp - 1} (a collective: every rank calls it
    with the same arguments) and return this rank's group."""
    groups = [dist.new_group(list(range(d * tp, (d + 1) * tp))) for d in range(world // tp)]
    return groups[dist.get_rank() // tp]


def symmetric_gather_output(shape, group, device):
    """A bf16 output buffer of `shape` in symmetric memory on every rank of `group`, and the
    device pointers of all ranks' copies (rank order) for mla_combine_gather's peer stores."""
    import torch.distributed._symmetric_memory as symm_mem
    buf = symm_mem.empty(*shape, dtype=torch.bfloat16, device=device)
    hdl = symm_mem.rendezvous(buf, group)
    return buf, [int(p) for p in hdl.buffer_ptrs]


def stream_barrier(group=None, device=None):
    """Stream-ordered barrier (one-element all-reduce): peer stores issued before it on
    every rank are visible to every rank after it."""
    t = torch.zeros(1, dtype=torch.int32, device=device)
    dist.all_reduce(t, group=group)
