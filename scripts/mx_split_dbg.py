"""Debug: compare every split partial (o_part, lse_part) of the MX decode with oracle.decode_mx
over that split's key blocks (lens,H,seed)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import numpy as np, torch
from gpu_cases import Case
from oracle import snapmla as O
from paper_2602_10718_b200 import ops
lens = [int(x) for x in sys.argv[1].split(",")]; H = int(sys.argv[2]); seed = int(sys.argv[3])
case = Case(lens, H, seed=seed)
cache = case.gpu_cache()
bt = torch.from_numpy(case.bt).cuda(); sl = torch.from_numpy(case.lens.astype(np.int32)).cuda()
B = len(lens)
ws = torch.zeros(ops.mla_decode_workspace_bytes(B, H), dtype=torch.uint8, device="cuda")
ops.mla_decode_fp8_mx(case.q.cuda(), cache.kv_fp8, cache.kv_rope, cache.kv_scale, bt, sl, case.scale, ws)
torch.cuda.synchronize()
w = ws.cpu().numpy()
hdr = w[:64].view(np.int32)
total, per, groups, nht = hdr[0], hdr[1], hdr[2], hdr[3]
sms = 148
# workspace layout (snapmla_internal.h ws_layout)
def al(x, a): return (x + a - 1) // a * a
cum_off = 64; first = al(cum_off + (B + 1) * 4, 16); groups_ws = sms // nht
lse_off = al(first + (groups_ws + 1) * 4, 256); slots = B + groups_ws
o_off = al(lse_off + slots * nht * 64 * 4, 256)
lse_p = w[lse_off:lse_off + slots * nht * 64 * 4].view(np.float32).reshape(slots, nht, 64)
o_p = w[o_off:o_off + slots * nht * 64 * 512 * 4].view(np.float32).reshape(slots, nht, 64, 512)
cum = np.concatenate([[0], np.cumsum([(L + 63) // 64 for L in lens])])
pools = case.oracle_pools()
for b in range(B):
    if lens[b] == 0: continue
    qc, sq, qr = O.q_quant(case.q[b].float().numpy())
    kc, sk, kr = O.gather_request(pools, case.bt[b], lens[b])
    for g in range(groups):
        lo, hi = max(g * per, cum[b]), min((g + 1) * per, cum[b + 1])
        if lo >= hi: continue
        j0, j1 = (lo - cum[b]) * 64, min((hi - cum[b]) * 64, lens[b])
        om, lm = O.decode_mx(qc, sq, qr, kc[j0:j1], sk[j0:j1], kr[j0:j1], case.scale)
        got = o_p[b + g].reshape(nht * 64, 512)[:H]; gl = lse_p[b + g].reshape(-1)[:H]
        rms = np.sqrt(np.mean(om ** 2))
        err = np.abs(got - om).max(axis=1) / rms
        if err.max() > 1e-3 or np.abs(gl - lm).max() > 1e-3:
            bad = np.nonzero(err > 1e-3)[0]
            print(f"req {b} split g={g} blocks [{lo - cum[b]},{hi - cum[b]}) max/rms={err.max():.2e} bad rows {bad.tolist()[:10]} lse_err={np.abs(gl-lm).max():.2e}")
            for rr in bad[:2]:
                ratio = got[rr] / np.where(np.abs(om[rr]) > 1e-9, om[rr], np.nan)
                print("   row", rr, "ratio median %.6f p1 %.6f p99 %.6f" % (np.nanmedian(ratio), np.nanpercentile(ratio, 1), np.nanpercentile(ratio, 99)),
                      "dims 0-255 vs 256-511 ratio medians %.6f %.6f" % (np.nanmedian(ratio[:256]), np.nanmedian(ratio[256:])))
                for bb in range(lo, hi):   # per-block oracle partial for this row
                    jj0, jj1 = (bb - cum[b]) * 64, min((bb - cum[b] + 1) * 64, lens[b])
                    ob, lb = O.decode_mx(qc[rr:rr+1], sq[rr:rr+1], qr[rr:rr+1], kc[jj0:jj1], sk[jj0:jj1], kr[jj0:jj1], case.scale)
                    print("     block", bb - cum[b], "lse %.3f" % lb[0], "resid fit:", float(np.dot(got[rr] - om[rr], ob[0]) / np.dot(ob[0], ob[0])))
print("done")
