"""CTA-0 (leader) event timeline of the 2-SM kernel (SNAPMLA_TRACE build), DS-R1 shape.
   SNAPMLA_LIB=paper_2602_10718_b200/libsnapmla_trace.so python scripts/trace_2sm.py"""
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
lib.mla_debug_set_pair(int(os.environ.get("V", "2")))
tr = torch.zeros(16 * 256 + 2 * 1024, dtype=torch.int64, device=dev)
lib.mla_debug_set_trace.argtypes = [ctypes.c_void_p]
for i in range(3):
    if i == 2:
        lib.mla_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
    ops.decode_step(q, cache, bt, sl, synth.DEFAULT_SOFTMAX_SCALE)
torch.cuda.synchronize()
lib.mla_debug_set_trace(None)
t = tr.cpu().numpy()[:16 * 256].reshape(16, 256).astype(np.int64)
names = ["TMA", "QK", "PV_L", "PV_R", "SM_in", "SM_out", "C_L", "C_R", "SMsc", "QKkvq", "SMsoft", "SMpemp", "PVpp", "C0", "C1", "C2"]
nv = int((t[1] > 0).sum())
def per(e):
    return np.median(np.diff(t[e][20:min(nv, 200)]))
print("blocks", nv, "periods:", {names[e]: per(e) for e in (0, 1, 2, 4, 5, 6)})
def med(a, b):
    return np.median((t[b] - t[a])[20:min(nv, 200)])
print("QKkvq-TMA", med(0, 9), "QK-QKkvq", med(9, 1), "SM_in-QK", med(1, 4), "SMsc-SM_in", med(4, 8),
      "SMsoft-SMsc", med(8, 10), "SMpemp-SMsoft", med(10, 11), "SM_out-SMpemp", med(11, 5),
      "PVpp-SM_out", med(5, 12), "PV_L-PVpp", med(12, 2), "C0-SM_out", med(5, 13), "C_L-PV_L", med(2, 6), "C_R-C_L", med(6, 7))

ct = tr.cpu().numpy()[16 * 256:].reshape(-1, 2).astype(np.int64)
ok = ct[:, 0] > 0
if ok.any():
    d = (ct[ok, 1] - ct[ok, 0]) / 1e3
    print("CTA durations us: min/median/max", d.min(), np.median(d), d.max(), "span", (ct[ok, 1].max() - ct[ok, 0].min()) / 1e3)
rel = t - t[0][0]
print("first blocks (TMA, QK, PV_L, SM_in, SM_out, C_L):")
for n in range(min(nv, 6)):
    print(n, [int(rel[e][n]) for e in (0, 1, 2, 4, 5, 6)])
