"""Record and summarise the CTA-0 event timeline of mla_decode_fp8 (debug build hook)."""
import ctypes
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from paper_2602_10718_b200 import ops, synth

B, H, L = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
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
NEV = 16
tr = torch.zeros(NEV * 256 + 2 * 1024, dtype=torch.int64, device=dev)
lib = ops.lib()  # use SNAPMLA_LIB=...libsnapmla_trace.so (SNAPMLA_TRACE build)
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
t0g = ct[:, 0].min()
dur = (ct[:, 1] - ct[:, 0]) / 1e3
print('CTAs', len(ct), 'start spread us', (ct[:, 0].max() - t0g) / 1e3, 'duration us min/median/max', dur.min(), np.median(dur), dur.max(), 'kernel span us', (ct[:, 1].max() - t0g) / 1e3)
print('durations sorted (us):', np.round(np.sort(dur)[::10], 1)); print('slowest 12 CTAs (us):', ' '.join(f'{x:.1f}' for x in np.sort(dur)[-12:]), '| ids', ' '.join(str(i) for i in np.argsort(dur)[-12:]))
names = ["TMA", "QK", "PV_L", "PV_R", "SM_in", "SM_out", "C_L", "C_R", "S1", "S2", "S3", "S4", "S5", "C0", "C1", "C2"]
valid = t[1] > 0
nv = int(valid.sum())
t0 = t[0][0]
rel = np.where(t > 0, t - t0, 0)
print("blocks traced:", nv)
print("  n " + " ".join(f"{nm:>7}" for nm in names))
for n in list(range(0, 12)) + list(range(100, 108)):
    if n < nv:
        print(f"{n:3d} " + " ".join(f"{rel[e][n]:7d}" for e in range(NEV)))
d = np.diff(t[1][:nv])
print("QK issue period: median", np.median(d[10:]), "mean", d[10:].mean())
for e in range(NEV):
    dd = np.diff(t[e][20:nv])
    print(f"{names[e]:>7} period median {np.median(dd):.0f}")
print("SM_out - SM_in median", np.median((t[5] - t[4])[20:nv]))
print("C_L - SM_out median", np.median((t[6] - t[5])[20:nv]))
print("PV_L - C_L median", np.median((t[2] - t[6])[20:nv]))
print("C_R - C_L median", np.median((t[7] - t[6])[20:nv]))
print("SM_in - QK median", np.median((t[4] - t[1])[20:nv]))
print("QK(n) - TMA(n) median", np.median((t[1] - t[0])[20:nv]))

def med(a, b):
    return np.median((t[b] - t[a])[20:nv])
print("softmax: S1-SM_in", med(4, 8), "S2-S1", med(8, 9), "S3-S2", med(9, 10), "S4-S3", med(10, 11), "S5-S4", med(11, 12), "SM_out-S5", med(12, 5))
print("corr: C0-prevC_R", np.median((t[13][21:nv] - t[7][20:nv-1])), "C1-C0", med(13, 14), "C_L-C1", med(14, 6), "C2-C_L", med(6, 15), "C_R-C2", med(15, 7))

pro = tr.cpu().numpy()[15 * 256 + 250: 15 * 256 + 255].astype(np.int64)
qq = tr.cpu().numpy()[15 * 256 + 245: 15 * 256 + 248].astype(np.int64)
if pro[0] > 0 and qq[0] > 0:
    print("Q-quant (cycles from kernel entry): start", qq[0] - pro[0], "amax done", qq[1] - pro[0], "codes in TMEM", qq[2] - pro[0])
if pro[0] > 0:
    print("prologue (cycles from kernel entry): setup done", pro[1] - pro[0], "plan visible", pro[2] - pro[0],
          "Q-quant done", pro[3] - pro[0], "QK sees q_full", pro[4] - pro[0],
          "first TMA", int(t[0][0] - pro[0]), "first QK", int(t[1][0] - pro[0]), "first SM_in", int(t[4][0] - pro[0]))

if nv > 30:
    sl = slice(20, nv)
    print("softmax tail: C2-S5 (stats + P' stores)", np.median((t[15] - t[12])[sl]), "SM_out-C2 (fence.proxy.async + arrive)", np.median((t[5] - t[15])[sl]))
if nv > 30:
    sl = slice(20, nv)
    print("swapped-PV acc (if built): C0->C1 (t_full wait, half L)", np.median((t[14] - t[13])[sl]), "C1->C_L (consume L)", np.median((t[6] - t[14])[sl]),
          "PVL->C1", np.median((t[14] - t[2])[sl]), "SM_out->PVL", np.median((t[2] - t[5])[sl]))
