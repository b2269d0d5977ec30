"""CTA-0 (leader) event timeline of the block-pair 2-SM kernel (SNAPMLA_TRACE build), DS-R1 shape.
   SNAPMLA_LIB=paper_2602_10718_b200/libsnapmla_trace.so python scripts/trace_bp.py [B H L]
Events are indexed by the CTA's n-th block PAIR; prints the median per-pair period and the
median gap between consecutive stages of one pair."""
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
lib.mla_debug_set_pair(int(os.environ.get("V", "1")))
tr = torch.zeros(16 * 256 + 2 * 1024, dtype=torch.int64, device=dev)
lib.mla_debug_set_trace.argtypes = [ctypes.c_void_p]
for i in range(3):
    if i == 2:
        lib.mla_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
    ops.decode_step(q, cache, bt, sl, synth.DEFAULT_SOFTMAX_SCALE)
torch.cuda.synchronize()
lib.mla_debug_set_trace(None)
t = tr.cpu().numpy()[:16 * 256].reshape(16, 256).astype(np.int64)
N = dict(TMA=0, QK=1, PVL=2, PVR=3, SM_in=4, SM_out=5, C_L=6, C_R=7, S1=8, S2=9, S3=10, S4=11, S5=12, C0=13, C1=14, C2=15)
nv = int((t[N["QK"]] > 0).sum())
lo, hi = 10, min(nv, 200)
print("pairs", nv)
print("period (median diff):", {k: int(np.median(np.diff(t[v][lo:hi]))) for k, v in N.items() if (t[v][lo:hi] > 0).all()})
chain = ["TMA", "C1", "QK", "SM_in", "S1", "S2", "S3", "S4", "SM_out", "S5", "C2", "PVL", "C_L", "C_R"]
print("stage gaps (median over pairs):")
for a, b in zip(chain[:-1], chain[1:]):
    d = (t[N[b]] - t[N[a]])[lo:hi]
    print(f"  {a:>6} -> {b:<6} {int(np.median(d)):8d}")
print("  SM_out -> C0", int(np.median((t[N["C0"]] - t[N["SM_out"]])[lo:hi])))
ct = tr.cpu().numpy()[16 * 256:].reshape(-1, 2).astype(np.int64)
ok = ct[:, 0] > 0
if ok.any():
    d = (ct[ok, 1] - ct[ok, 0]) / 1e3
    t0 = ct[ok, 0].min()
    print("CTA durations us: min/median/max", d.min(), np.median(d), d.max(), "span", (ct[ok, 1].max() - t0) / 1e3)
    print("CTA start offsets us: median/max", np.median((ct[ok, 0] - t0) / 1e3), ((ct[ok, 0] - t0) / 1e3).max())
    ends = np.sort((ct[ok, 1] - t0) / 1e3)
    print("CTA end times us (sorted, every 16th):", [round(x, 1) for x in ends[::16]], "last", round(ends[-1], 1))
    ws = torch.zeros(8, dtype=torch.int32)
    hdr = None
    try:
        nsm = torch.cuda.get_device_properties(0).multi_processor_count
        print("SMs", nsm, "CTAs traced", int(ok.sum()))
    except Exception as e:
        print(e)
rel = t - t[N["TMA"]][0]
print("first pairs (TMA, QK, SM_in, SM_out, PVL, C_L):")
for n in range(min(nv, 6)):
    print(n, [int(rel[N[e]][n]) for e in ("TMA", "QK", "SM_in", "SM_out", "PVL", "C_L")])
# untraced decode time of the same call (trace buffer off)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(3):
    ops.decode_step(q, cache, bt, sl, synth.DEFAULT_SOFTMAX_SCALE)
e0.record()
for i in range(20):
    ops.decode_step(q, cache, bt, sl, synth.DEFAULT_SOFTMAX_SCALE)
e1.record(); torch.cuda.synchronize()
print("untraced decode_step ms (mean of 20):", round(e0.elapsed_time(e1) / 20, 4))
