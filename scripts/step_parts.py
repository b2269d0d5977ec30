"""Per-kernel time of one decode step at a small shape (append, plan + decode, combine), eager and as a
CUDA graph: mean over 200 back-to-back repetitions of each part.  python scripts/step_parts.py [B H L]"""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
from paper_2602_10718_b200 import ops, synth

B, H, L = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (1, 128, 4096)))
dev = torch.device("cuda")
gen = torch.Generator(device=dev); gen.manual_seed(0)
ppr = L // 64
cache = ops.PagedMLACache(B * ppr, dev)
bt = torch.randperm(B * ppr, generator=gen, device=dev).to(torch.int32).view(B, ppr).contiguous()
q = synth.torch_queries(B * H, gen, dev).view(B, H, 576)
c, r = synth.torch_latent(B, gen, dev)
sl = torch.full((B,), L, dtype=torch.int32, device=dev)
ws = torch.empty(ops.mla_decode_workspace_bytes(B, H), dtype=torch.uint8, device=dev)
out = torch.empty(B, H, 512, dtype=torch.bfloat16, device=dev)
lse = torch.empty(B, H, dtype=torch.float32, device=dev)
S = synth.DEFAULT_SOFTMAX_SCALE
parts = {
    "append": lambda: cache.append(c, r, bt, sl),
    "plan+decode": lambda: ops.mla_decode_fp8(q, cache.kv_fp8, cache.kv_rope, cache.kv_scale, bt, sl, S, ws),
    "combine": lambda: ops.mla_combine(ws, B, H, out, lse),
}
parts["step"] = lambda: (parts["append"](), parts["plan+decode"](), parts["combine"]())
for name, f in parts.items():
    for mode in ("eager", "graph"):
        for _ in range(5): f()
        torch.cuda.synchronize()
        run = f
        if mode == "graph":
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                f()
            run = g.replay
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(200): run()
        e1.record(); torch.cuda.synchronize()
        t_host = time.perf_counter()
        for _ in range(200): run()
        host_us = (time.perf_counter() - t_host) / 200 * 1e6
        torch.cuda.synchronize()
        print(f"{name:12s} {mode:5s} {e0.elapsed_time(e1) / 200 * 1e3:8.1f} us/iter (host enqueue {host_us:6.1f} us/iter)", flush=True)
