"""CTA-0 timeline of the BF16 baseline decode (mla_decode_kernel<true>, SNAPMLA_TRACE build), DS-R1 shape."""
import ctypes, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from paper_2602_10718_b200 import ops, synth

B, H, L = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (64, 128, 32768)))
dev = torch.device("cuda")
gen = torch.Generator(device=dev); gen.manual_seed(0)
ppr = L // 64
cache = ops.PagedMLACacheBF16(B * ppr, dev)
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
    ops.decode_step(q, cache, bt, sl, synth.DEFAULT_SOFTMAX_SCALE)
torch.cuda.synchronize()
lib.mla_debug_set_trace(None)
t = tr.cpu().numpy()[:16 * 256].reshape(16, 256).astype(np.int64)
names = ["TMA", "QK", "PV_L", "PV_R", "SM_in", "SM_out", "C_L", "C_R", "S1", "S2", "S3", "S4", "S5", "C0", "C1", "C2"]
nv = int((t[1] > 0).sum())
lo, hi = 20, min(nv, 200)
print("blocks", nv, "periods:", {names[e]: float(np.median(np.diff(t[e][lo:hi]))) for e in (0, 1, 2, 4, 5, 6)})
def med(a, b):
    return float(np.median((t[b] - t[a])[lo:hi]))
print("QK-TMA", med(0, 1), "SM_in-QK", med(1, 4), "SM_out-SM_in", med(4, 5), "PV_L-SM_out", med(5, 2),
      "C_L-PV_L", med(2, 6), "C_R-C_L", med(6, 7), "S5-S4(p_empty wait)", med(11, 12))
rel = t - t[0][0]
for n in range(24, 30):
    print(n, [int(rel[e][n]) for e in range(8)])
