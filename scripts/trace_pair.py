"""CTA-0 event timeline of the CTA-pair decode kernel (SNAPMLA_TRACE build), DS-R1 shape by default.
   SNAPMLA_LIB=paper_2602_10718_b200/libsnapmla_trace.so python scripts/trace_pair.py [B H L]"""
import ctypes
import os
import sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from paper_2602_10718_b200 import ops, synth

B, H, L = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (64, 128, 32768)))
dev = torch.device("cuda")
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
# untraced timing of the same decode (plan + decode + combine), 20 back-to-back calls
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3):
    ops.decode_step(q, cache, bt, sl, synth.DEFAULT_SOFTMAX_SCALE)
e0.record()
for _ in range(20):
    ops.decode_step(q, cache, bt, sl, synth.DEFAULT_SOFTMAX_SCALE)
e1.record()
torch.cuda.synchronize()
print("untraced decode_step ms:", e0.elapsed_time(e1) / 20)
if os.environ.get("TIME_ONLY") == "1":
    sys.exit(0)
NEV = 16
tr = torch.zeros(NEV * 256 + 2 * 1024, dtype=torch.int64, device=dev)
lib = ops.lib()
lib.mla_debug_set_trace.argtypes = [ctypes.c_void_p]
for i in range(3):
    if i == 2:
        lib.mla_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
    ops.decode_step(q, cache, bt, sl, synth.DEFAULT_SOFTMAX_SCALE)
torch.cuda.synchronize()
lib.mla_debug_set_trace(None)
allt = tr.cpu().numpy().astype(np.int64)
t = allt[:NEV * 256].reshape(NEV, 256)
ct = allt[NEV * 256:].reshape(-1, 2)
ct = ct[ct[:, 0] > 0]
dur = (ct[:, 1] - ct[:, 0]) / 1e3
allct = allt[NEV * 256:].reshape(-1, 2)
t0g = ct[:, 0].min()
print('CTAs', len(ct), 'duration us min/median/max', dur.min(), np.median(dur), dur.max(),
      'start spread us', (ct[:, 0].max() - t0g) / 1e3, 'span us', (ct[:, 1].max() - t0g) / 1e3)
d_all = np.where(allct[:, 0] > 0, (allct[:, 1] - allct[:, 0]) / 1e3, -1)[:148]
print('per-CTA duration (us), blockIdx order:', np.round(d_all, 0).astype(int).tolist())
print('per-CTA start offset (us):', np.round((allct[:148, 0] - t0g) / 1e3, 0).astype(int).tolist())
names = ["TMA", "QK", "PV_L", "PV_R", "SM_in", "SM_out", "C_L", "C_R", "SMkvl", "QKkvq", "SMB_in", "SMdone",
         "SMpemp", "C0", "C1", "SMB_out"]
t0 = t[0][0]
rel = np.where(t > 0, t - t0, 0)
print("pair events (index np): TMA QKkvq QK SM_in SMkvl SMdone SMpemp SM_out SMB_in SMB_out")
pe = [0, 9, 1, 4, 8, 11, 12, 5, 10, 15]
for n in list(range(0, 8)) + list(range(60, 66)):
    print(f"{n:3d} " + " ".join(f"{rel[e][n]:7d}" for e in pe))
print("block events (index n): PV_L PV_R C0 C1 C_L C_R")
be = [2, 3, 13, 14, 6, 7]
for n in list(range(0, 12)) + list(range(120, 128)):
    print(f"{n:3d} " + " ".join(f"{rel[e][n]:7d}" for e in be))
def per(e, a=20, b=100):
    return np.median(np.diff(t[e][a:b]))
print("periods (median): pair TMA", per(0), "QK", per(1), "SM_in", per(4), "| block PV_L", per(2, 40, 200), "C_L", per(6, 40, 200))
def med(a, b, lo=20, hi=100):
    return np.median((t[b] - t[a])[lo:hi])
print("pair: QKkvq-TMA", med(0, 9), "QK-QKkvq", med(9, 1), "SM_in-QK", med(1, 4), "SMkvl-SM_in", med(4, 8),
      "SMdone-SMkvl", med(8, 11), "SMpemp-SMdone", med(11, 12), "SM_out-SMpemp", med(12, 5))
