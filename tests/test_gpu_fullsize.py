"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(one decode over the whole workload: same batch, heads, context, plan and grid), on
sampled outputs the oracle computes one request at a time:
  * the GPU cache bytes / scales / RoPE of the sampled requests == oracle append_quant
    of their inputs (bit-exact), and
  * the decode output of sampled (request, head) rows == the O7 closed form
    (north_star gate, reading R23: fp32 result max-abs <= 2e-2 RMS, mean-abs <= 2e-3 RMS;
    LSE within 1e-3).
Inputs: seeded torch.Generator on the GPU (synth.torch_latent / torch_queries, the bench's
generators), random page permutation."""
import numpy as np
import pytest
import torch

from gpu_cases import parity_stats
from oracle import snapmla as O
from paper_2602_10718_b200 import ops, synth

pytestmark = pytest.mark.gpu

CONFIGS = {   # BASELINE.json configs[1..3] per-GPU shapes (bench.py WORKLOADS)
    "dsr1": (64, 128, 32768),
    "longcat": (128, 64, 131072),
    "dsr1_tp8": (256, 16, 65536),
}


@pytest.mark.parametrize("name", sorted(CONFIGS))
def test_full_size_sampled(name):
    B, H, L = CONFIGS[name]
    dev = torch.device("cuda")
    gen = torch.Generator(device=dev)
    gen.manual_seed(900 + B)
    ppr = L // 64
    cache = ops.PagedMLACache(B * ppr, dev)
    bt = torch.randperm(B * ppr, generator=gen, device=dev).to(torch.int32).view(B, ppr).contiguous()
    samples = [0, B // 2 + 1, B - 1]
    kept = {}
    chunk = 1 << 20
    for s in range(0, B * L, chunk):
        idx = torch.arange(s, min(s + chunk, B * L), device=dev)
        req, pos = idx // L, idx % L
        c, r = synth.torch_latent(idx.numel(), gen, dev)
        cache.append(c, r, bt[req, pos // 64].view(-1, 1).contiguous(), (pos % 64 + 1).to(torch.int32))
        for b in samples:   # keep the sampled requests' inputs for the oracle
            m = req == b
            if bool(m.any()):
                kept.setdefault(b, []).append((c[m].cpu(), r[m].cpu()))
    q = synth.torch_queries(B * H, gen, dev).view(B, H, 576)
    sl = torch.full((B,), L, dtype=torch.int32, device=dev)
    scale = synth.DEFAULT_SOFTMAX_SCALE
    out, lse = ops.decode_step(q, cache, bt, sl, scale, f32_out=True)
    torch.cuda.synchronize()
    heads = np.unique(np.array([0, 1, H // 2, H - 1]))
    bt_np = bt.cpu().numpy()
    refs, gots, lerr = [], [], 0.0
    for b in samples:
        c = torch.cat([x[0] for x in kept[b]]).float().numpy()
        r = torch.cat([x[1] for x in kept[b]]).float().numpy()
        kc, sk, kr = O.append_quant(c, r)
        slots = bt_np[b][np.arange(L) // 64].astype(np.int64) * 64 + np.arange(L) % 64
        ts = torch.from_numpy(slots).to(dev)
        assert np.array_equal(cache.kv_fp8.view(-1, 512)[ts].cpu().numpy(), kc), f"codes of request {b}"
        assert np.array_equal(cache.kv_scale.view(-1)[ts].cpu().numpy().view(np.uint32), sk.view(np.uint32))
        assert np.array_equal(cache.kv_rope.view(-1, 64)[ts].view(torch.int16).cpu().numpy().view(np.uint16), kr)
        qc, sq, qr = O.q_quant(q[b, heads].float().cpu().numpy())
        o7, l7 = O.decode_o7(qc, sq, qr, kc, sk, kr, scale)
        refs.append(o7)
        gots.append(out[b, heads].cpu().numpy())
        lerr = max(lerr, float(np.abs(lse[b, heads].cpu().numpy() - l7).max()))
    mx, mn = parity_stats(np.concatenate(gots), np.concatenate(refs))
    msg = f"{name}: max/rms={mx:.2e} mean/rms={mn:.2e} lse={lerr:.2e}"
    print(msg)
    assert mx <= 2e-2 and mn <= 2e-3 and lerr <= 1e-3, msg


@pytest.mark.parametrize("name", ["dsr1", "longcat"])
def test_full_size_sampled_bf16_baseline(name):
    """NEXT-2 baseline at the full sizes: BF16 cache bytes of sampled requests == their inputs
    (a copy), sampled rows of mla_decode_bf16 vs O8 (decode gate)."""
    B, H, L = CONFIGS[name]
    dev = torch.device("cuda")
    gen = torch.Generator(device=dev)
    gen.manual_seed(950 + B)
    ppr = L // 64
    cache = ops.PagedMLACacheBF16(B * ppr, dev)
    bt = torch.randperm(B * ppr, generator=gen, device=dev).to(torch.int32).view(B, ppr).contiguous()
    samples = [1, B - 2]
    kept = {}
    chunk = 1 << 20
    for s in range(0, B * L, chunk):
        idx = torch.arange(s, min(s + chunk, B * L), device=dev)
        req, pos = idx // L, idx % L
        c, r = synth.torch_latent(idx.numel(), gen, dev)
        cache.append(c, r, bt[req, pos // 64].view(-1, 1).contiguous(), (pos % 64 + 1).to(torch.int32))
        for b in samples:
            m = req == b
            if bool(m.any()):
                kept.setdefault(b, []).append((c[m].cpu(), r[m].cpu()))
    q = synth.torch_queries(B * H, gen, dev).view(B, H, 576)
    sl = torch.full((B,), L, dtype=torch.int32, device=dev)
    scale = synth.DEFAULT_SOFTMAX_SCALE
    out, lse = ops.decode_step(q, cache, bt, sl, scale, f32_out=True)
    torch.cuda.synchronize()
    heads = np.unique(np.array([0, H // 3, H - 1]))
    bt_np = bt.cpu().numpy()
    refs, gots, lerr = [], [], 0.0
    for b in samples:
        c = torch.cat([x[0] for x in kept[b]])
        r = torch.cat([x[1] for x in kept[b]])
        slots = torch.from_numpy(bt_np[b][np.arange(L) // 64].astype(np.int64) * 64 + np.arange(L) % 64).to(dev)
        assert torch.equal(cache.kv_c.view(-1, 512)[slots].cpu().view(torch.int16), c.view(torch.int16))
        assert torch.equal(cache.kv_rope.view(-1, 64)[slots].cpu().view(torch.int16), r.view(torch.int16))
        o8, l8 = O.attn_o8(q[b, heads].float().cpu().numpy(), c.float().numpy(), r.float().numpy(), scale)
        refs.append(o8)
        gots.append(out[b, heads].cpu().numpy())
        lerr = max(lerr, float(np.abs(lse[b, heads].cpu().numpy() - l8).max()))
    mx, mn = parity_stats(np.concatenate(gots), np.concatenate(refs))
    msg = f"bf16 {name}: max/rms={mx:.2e} mean/rms={mn:.2e} lse={lerr:.2e}"
    print(msg)
    assert mx <= 2e-2 and mn <= 2e-3 and lerr <= 1e-3, msg
