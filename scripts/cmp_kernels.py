"""Decode time of the kernels for 64 < rows <= 128 (mla_debug_set_pair: 0 single-CTA, 1 block-pair) over DeepSeek-R1-shape points (128 heads): median of 20 timed decodes (CUDA
events, one stream) after a 1 s load phase per point.  python scripts/cmp_kernels.py [kernels]"""
import json, os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from paper_2602_10718_b200 import ops, synth

kernels = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else "0,1".split(","))]
points = [(1, 32768), (8, 32768), (64, 4096), (512, 4096), (32, 16384), (8, 131072), (64, 32768), (1, 4096)]
dev = torch.device("cuda")
lib = ops.lib()
res = []
for B, L in points:
    gen = torch.Generator(device=dev); gen.manual_seed(0)
    ppr = L // 64
    cache = ops.PagedMLACache(B * ppr, dev)
    bt = torch.randperm(B * ppr, generator=gen, device=dev).to(torch.int32).view(B, ppr).contiguous()
    for s in range(0, B * L, 1 << 20):
        idx = torch.arange(s, min(s + (1 << 20), B * L), device=dev)
        req, pos = idx // L, idx % L
        c, r = synth.torch_latent(idx.numel(), gen, dev)
        cache.append(c, r, bt[req, pos // 64].view(-1, 1).contiguous(), (pos % 64 + 1).to(torch.int32))
    q = synth.torch_queries(B * 128, gen, dev).view(B, 128, 576)
    sl = torch.full((B,), L, dtype=torch.int32, device=dev)
    ws = torch.empty(ops.mla_decode_workspace_bytes(B, 128), dtype=torch.uint8, device=dev)
    row = {"batch": B, "context": L}
    for kk in kernels:
        lib.mla_debug_set_pair(kk)
        f = lambda: ops.mla_decode_fp8(q, cache.kv_fp8, cache.kv_rope, cache.kv_scale, bt, sl, synth.DEFAULT_SOFTMAX_SCALE, ws)
        t0 = time.time()
        while time.time() - t0 < 1.0:
            for _ in range(20): f()
            torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); f(); e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        byts = B * L * 644 + B * 128 * 1152
        row[f"k{kk}_ms"] = round(ms, 4)
        row[f"k{kk}_frac"] = round(byts / (ms / 1e3) / 1e9 / 6553.6, 4)
    lib.mla_debug_set_pair(-1)
    print(json.dumps(row), flush=True)
    del cache
    torch.cuda.empty_cache()
