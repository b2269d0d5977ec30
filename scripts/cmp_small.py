"""Decode time of the two kernels for rows <= 32 (mla_debug_set_small: 0 single-CTA with heads padded to
M = 64, -1 the swapped-operand kernel) on TP8-shape points (heads per rank H): median of 20 timed decodes
(CUDA events, one stream) after a 1 s load phase per point, and the fraction of the measured HBM roofline.
  python scripts/cmp_small.py [H]"""
import json, os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from paper_2602_10718_b200 import ops, synth

H = int(sys.argv[1]) if len(sys.argv) > 1 else 16
points = [(256, 65536), (64, 32768), (1, 32768), (8, 32768), (64, 4096), (512, 4096), (8, 131072)]
dev = torch.device("cuda")
lib = ops.lib()
for B, L in points:
    gen = torch.Generator(device=dev); gen.manual_seed(0)
    ppr = L // 64
    cache = ops.PagedMLACache(B * ppr, dev)
    bt = torch.randperm(B * ppr, generator=gen, device=dev).to(torch.int32).view(B, ppr).contiguous()
    for s in range(0, B * L, 1 << 21):
        idx = torch.arange(s, min(s + (1 << 21), B * L), device=dev)
        req, pos = idx // L, idx % L
        c, r = synth.torch_latent(idx.numel(), gen, dev)
        cache.append(c, r, bt[req, pos // 64].view(-1, 1).contiguous(), (pos % 64 + 1).to(torch.int32))
    q = synth.torch_queries(B * H, gen, dev).view(B, H, 576)
    sl = torch.full((B,), L, dtype=torch.int32, device=dev)
    ws = torch.empty(ops.mla_decode_workspace_bytes(B, H), dtype=torch.uint8, device=dev)
    row = {"batch": B, "context": L, "heads": H}
    outs = {}
    for kk in (0, -1):
        lib.mla_debug_set_small(kk)
        f = lambda: ops.mla_decode_fp8(q, cache.kv_fp8, cache.kv_rope, cache.kv_scale, bt, sl, synth.DEFAULT_SOFTMAX_SCALE, ws)
        outs[kk] = ops.decode_step(q, cache, bt, sl, synth.DEFAULT_SOFTMAX_SCALE, f32_out=True)[0].clone()
        t0 = time.time()
        while time.time() - t0 < 1.0:
            for _ in range(10): f()
            torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); f(); e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        byts = B * L * 644 + B * H * 1152
        name = "single" if kk == 0 else "swapped"
        row[f"{name}_ms"] = round(ms, 4)
        row[f"{name}_frac"] = round(byts / (ms / 1e3) / 1e9 / 6553.6, 4)
    lib.mla_debug_set_small(-1)
    d = (outs[0] - outs[-1]).abs().max().item() / outs[0].pow(2).mean().sqrt().item()
    row["max_diff_over_rms"] = float(f"{d:.3e}")
    print(json.dumps(row), flush=True)
    del cache
    torch.cuda.empty_cache()
