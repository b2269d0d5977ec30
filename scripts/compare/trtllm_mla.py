"""Context measurement (not our hot path): FlashInfer's TRT-LLM-gen MLA decode on
B200 for the same shapes, BF16 cache (1152 B/token) and per-tensor FP8 cache
(576 B/token).  Usage: python scripts/compare/trtllm_mla.py [B H L]"""
import json
import sys

import torch

B, H, L = (int(x) for x in sys.argv[1:4]) if len(sys.argv) >= 4 else (64, 128, 32768)
dev = "cuda"
torch.manual_seed(0)
import flashinfer
from flashinfer.mla import trtllm_batch_decode_with_kv_cache_mla

page = 64
ppr = (L + page - 1) // page
num_pages = B * ppr
bt = torch.randperm(num_pages, device=dev, dtype=torch.int32).view(B, ppr).contiguous()
seq = torch.full((B,), L, dtype=torch.int32, device=dev)
res = {"shape": dict(batch=B, heads=H, context=L, page=page)}
for name, dt in (("bf16", torch.bfloat16), ("fp8_per_tensor", torch.float8_e4m3fn)):
    try:
        kv = (torch.randn(num_pages, page, 576, device=dev) * 0.5).to(dt)
        q = (torch.randn(B, 1, H, 576, device=dev) * 0.5).to(dt)
        ws = torch.zeros(128 * 1024 * 1024, dtype=torch.int8, device=dev)
        out = torch.empty(B, 1, H, 512, dtype=torch.bfloat16, device=dev)
        def run():
            return trtllm_batch_decode_with_kv_cache_mla(q, kv, ws, 128, 512, 64, bt, seq, L, out=out,
                                                         bmm1_scale=1.0 / (192 ** 0.5), bmm2_scale=1.0)
        for _ in range(5):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 30
        e0.record()
        for _ in range(n):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        nbytes = B * L * (1152 if dt == torch.bfloat16 else 576)
        res[name] = dict(ms=round(ms, 4), tokens_per_s=round(B / (ms / 1e3), 1),
                         gbs=round(nbytes / (ms / 1e3) / 1e9, 1), frac_of_6452=round(nbytes / (ms / 1e3) / 1e9 / 6452.8, 4))
        del kv, q, ws, out
        torch.cuda.empty_cache()
    except Exception as ex:   # cubins unavailable offline, unsupported shape, ...
        res[name] = {"error": f"{type(ex).__name__}: {str(ex)[:300]}"}
print(json.dumps(res))
