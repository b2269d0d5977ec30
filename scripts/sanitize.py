"""One small decode step (append -> decode -> combine) for compute-sanitizer runs.
  compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python scripts/sanitize.py <case> <kernel>
case:   tiny   (1 request x 256 tokens, 16 heads)
        ragged (2 requests of 77 and 300 tokens + an empty one, 128 heads: two head tiles, tail blocks,
                a half pair in the block-pair kernel, a zero-length request)
kernel: single | bp (forced through mla_debug_set_pair) | bf16 (the NEXT-2 baseline decode)"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from paper_2602_10718_b200 import ops, synth

case, kernel = sys.argv[1], sys.argv[2]
lens, H = ([256], 16) if case == "tiny" else ([77, 300, 0], 128)
dev = torch.device("cuda")
rng = np.random.default_rng(5)
bt_np, num_pages = synth.paged_layout(rng, lens, extra_pages=2)
n_tok = sum(lens)
c, r = synth.latent_tokens(rng, n_tok)
q = synth.queries(rng, len(lens) * H).reshape(len(lens), H, 576).to(dev)
bt = torch.from_numpy(bt_np).to(dev)
req = np.repeat(np.arange(len(lens)), lens)
pos = np.concatenate([np.arange(L) for L in lens])
page = bt_np[req, pos // 64]
bt_v = torch.from_numpy(page.astype(np.int32)[:, None]).to(dev)
sl_v = torch.from_numpy((pos % 64 + 1).astype(np.int32)).to(dev)
sl = torch.tensor(lens, dtype=torch.int32, device=dev)
lib = ops.lib()
if kernel == "bf16":
    cache = ops.PagedMLACacheBF16(num_pages, dev)
    cache.append(c.to(dev), r.to(dev), bt_v, sl_v)
    ws = torch.empty(ops.mla_decode_workspace_bytes(len(lens), H), dtype=torch.uint8, device=dev)
    ops.mla_decode_bf16(q, cache.kv_c, cache.kv_rope, bt, sl, synth.DEFAULT_SOFTMAX_SCALE, ws)
    out = torch.empty(len(lens), H, 512, dtype=torch.bfloat16, device=dev)
    lse = torch.empty(len(lens), H, dtype=torch.float32, device=dev)
    ops.mla_combine(ws, len(lens), H, out, lse)
else:
    lib.mla_debug_set_pair({"single": 0, "bp": 1}[kernel])
    cache = ops.PagedMLACache(num_pages, dev)
    cache.append(c.to(dev), r.to(dev), bt_v, sl_v)
    out, lse = ops.decode_step(q, cache, bt, sl, synth.DEFAULT_SOFTMAX_SCALE)
torch.cuda.synchronize()
o = out.float().cpu().numpy()
assert np.isfinite(o).all()
print(f"sanitize case={case} kernel={kernel} ok, |o|max={np.abs(o).max():.3g}")
