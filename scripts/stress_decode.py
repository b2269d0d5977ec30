"""Run decode on a list of (B, H, L) configs and report CUDA errors / NaNs (debug aid)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
from paper_2602_10718_b200 import ops, synth

dev = torch.device("cuda")
for spec in sys.argv[1:]:
    B, H, L = map(int, spec.split("x"))
    gen = torch.Generator(device=dev); gen.manual_seed(0)
    ppr = (L + 63) // 64
    cache = ops.PagedMLACache(B * ppr, dev)
    bt = torch.randperm(B * ppr, generator=gen, device=dev).to(torch.int32).view(B, ppr).contiguous()
    n_tok = B * L
    for s in range(0, n_tok, 1 << 18):
        idx = torch.arange(s, min(s + (1 << 18), n_tok), device=dev)
        req, pos = idx // L, idx % L
        c, r = synth.torch_latent(idx.numel(), gen, dev)
        cache.append(c, r, bt[req, pos // 64].view(-1, 1).contiguous(), (pos % 64 + 1).to(torch.int32))
    q = synth.torch_queries(B * H, gen, dev).view(B, H, 576)
    sl = torch.full((B,), L, dtype=torch.int32, device=dev)
    try:
        out, lse = ops.decode_step(q, cache, bt, sl, synth.DEFAULT_SOFTMAX_SCALE, f32_out=True)
        torch.cuda.synchronize()
        print(spec, "ok", "nan" if torch.isnan(out).any().item() else "finite", float(out.abs().max()), flush=True)
    except Exception as e:
        print(spec, "FAIL", e, flush=True)
        break
