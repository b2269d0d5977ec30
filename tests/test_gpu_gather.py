"""NEXT-4(c): mla_combine_gather (the TP all-gather fused into the combine epilogue as peer
stores), exercised on one GPU with `world` local buffers standing in for the peer-mapped
outputs.  Every virtual rank decodes its head slice; after all ranks' fused combines,
every buffer must equal, bit for bit, the concatenation over ranks of the plain per-rank
mla_combine outputs -- and, when the per-rank and full-head decodes share the split plan
(same number of 64-row head tiles), the full-head decode itself."""
import numpy as np
import pytest
import torch

from gpu_cases import Case, parity_stats
from paper_2602_10718_b200 import ops

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("H,world", [(64, 4), (64, 2), (128, 8), (128, 2), (32, 2), (16, 1)])
def test_fused_gather_equals_per_rank_combine(H, world):
    case = Case([700, 1, 65, 4096 + 3, 0], H, seed=600 + H + world)
    cache = case.gpu_cache()
    dev = "cuda"
    B, Hl = case.B, H // world
    bt = torch.from_numpy(case.bt).to(dev)
    sl = torch.from_numpy(case.lens.astype(np.int32)).to(dev)
    q = case.q.to(dev)
    outs = [torch.full((B, H, 512), float("nan"), dtype=torch.bfloat16, device=dev) for _ in range(world)]
    plain = []
    for r in range(world):
        qr = q[:, r * Hl:(r + 1) * Hl].contiguous()
        ws = torch.empty(ops.mla_decode_workspace_bytes(B, Hl), dtype=torch.uint8, device=dev)
        ops.mla_decode_fp8(qr, cache.kv_fp8, cache.kv_rope, cache.kv_scale, bt, sl, case.scale, ws)
        o = torch.empty(B, Hl, 512, dtype=torch.bfloat16, device=dev)
        lse_plain = torch.empty(B, Hl, dtype=torch.float32, device=dev)
        ops.mla_combine(ws, B, Hl, o, lse_plain)
        lse_g = torch.empty(B, Hl, dtype=torch.float32, device=dev)
        ops.mla_combine_gather(ws, B, Hl, outs, r, lse_g)
        torch.cuda.synchronize()
        assert torch.equal(lse_plain.view(torch.int32), lse_g.view(torch.int32))
        plain.append(o)
    ref = torch.cat(plain, dim=1)
    for r in range(world):
        assert torch.equal(outs[r].view(torch.int16), ref.view(torch.int16)), f"buffer of rank {r}"
    if (Hl + 63) // 64 == (H + 63) // 64:   # same split plan as the full-head decode
        full, _ = case.gpu_decode(cache)
        if (Hl <= 16) == (H <= 16):         # ... and the same kernel (rows <= 16: swapped-operand, §7.11)
            assert np.array_equal(full.astype(np.float32), ref.float().cpu().numpy())
        else:                                # different kernels: both within the O7 gate, so close
            mx, mn = parity_stats(full.astype(np.float32).reshape(-1, 512),
                                  ref.float().cpu().numpy().reshape(-1, 512))
            assert mx <= 2e-2 and mn <= 2e-3, (mx, mn)


def test_fused_gather_rejects_bad_args():
    case = Case([65], 16, seed=650)
    dev = "cuda"
    ws = torch.empty(ops.mla_decode_workspace_bytes(1, 16), dtype=torch.uint8, device=dev)
    outs = [torch.empty(1, 16 * 9, 512, dtype=torch.bfloat16, device=dev) for _ in range(9)]
    with pytest.raises(RuntimeError, match="UNSUPPORTED"):
        ops.mla_combine_gather(ws, 1, 16, outs, 0)       # world > 8
    two = [torch.empty(1, 32, 512, dtype=torch.bfloat16, device=dev) for _ in range(2)]
    with pytest.raises(RuntimeError, match="SHAPE"):
        ops.mla_combine_gather(ws, 1, 16, two, 2)        # rank >= world
