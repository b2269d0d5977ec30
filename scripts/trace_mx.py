"""CTA-0 event timeline of the MX kernel (SNAPMLA_TRACE build), DS-R1 shape; events per block n of
the CTA pair (own blocks: even n).  SNAPMLA_LIB=paper_2602_10718_b200/libsnapmla_trace.so python scripts/trace_mx.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from paper_2602_10718_b200 import ops, synth

B, H, L = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (64, 128, 32768)))
dev = torch.device("cuda")
gen = torch.Generator(device=dev); gen.manual_seed(0)
ppr = L // 64
cache = ops.PagedMLACache(B * ppr, dev)
bt = torch.randperm(B * ppr, generator=gen, device=dev).to(torch.int32).view(B, ppr).contiguous()
for s in range(0, B * L, 1 << 18):
    idx = torch.arange(s, min(s + (1 << 18), B * L), device=dev)
    req, pos = idx // L, idx % L
    c, r = synth.torch_latent(idx.numel(), gen, dev)
    cache.append(c, r, bt[req, pos // 64].view(-1, 1).contiguous(), (pos % 64 + 1).to(torch.int32))
q = synth.torch_queries(B * H, gen, dev).view(B, H, 576)
sl = torch.full((B,), L, dtype=torch.int32, device=dev)
lib = ops.lib()
tr = torch.zeros(16 * 256 + 2 * 1024, dtype=torch.int64, device=dev)
lib.mla_debug_set_trace.argtypes = [ctypes.c_void_p]
for i in range(3):
    if i == 2:
        lib.mla_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
    ops.decode_step(q, cache, bt, sl, synth.DEFAULT_SOFTMAX_SCALE, mx=True)
torch.cuda.synchronize()
lib.mla_debug_set_trace(None)
t = tr.cpu().numpy()[:16 * 256].reshape(16, 256).astype(np.int64)
N = dict(TMA=0, QK=1, PVL=2, SM_in=4, SM_out=5, S3=10, S4=11, C1=14, C2=15)
own = np.arange(0, 256, 2)
lo, hi = 10, 180
def per(ev, idx):
    v = t[N[ev]][idx]; v = v[v > 0]
    return int(np.median(np.diff(v[lo // 2:hi // 2]))) if len(v) > 20 else None
print("own-block period:", {e: per(e, own) for e in ("QK", "SM_in", "SM_out", "C1")}, " all-block PV period:", per("PVL", np.arange(256)))
def gap(a, b, idx):
    d = (t[N[b]] - t[N[a]])[idx][lo // 2:hi // 2]
    return int(np.median(d))
print("own blocks: C1->QK", gap("C1", "QK", own), "QK->SM_in", gap("QK", "SM_in", own), "SM_in->S3", gap("SM_in", "S3", own),
      "S3->S4", gap("S3", "S4", own), "S4->SM_out", gap("S4", "SM_out", own), "SM_out->PVL", gap("SM_out", "PVL", own))
