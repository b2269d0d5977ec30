"""Debug helper: one MX decode on a given case (lens,H) -> per-request / per-row error vs oracle.decode_mx."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import numpy as np, torch
from gpu_cases import Case
from paper_2602_10718_b200 import ops
lens = [int(x) for x in sys.argv[1].split(",")]
H = int(sys.argv[2])
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 1
case = Case(lens, H, seed=seed)
cache = case.gpu_cache()
bt = torch.from_numpy(case.bt).cuda(); sl = torch.from_numpy(case.lens.astype(np.int32)).cuda()
out, lse = ops.decode_step(case.q.cuda(), cache, bt, sl, case.scale, f32_out=True, mx=True)
torch.cuda.synchronize()
out = out.cpu().numpy(); lse = lse.cpu().numpy()
pools = case.oracle_pools()
for b in range(case.B):
    if lens[b] == 0: continue
    om, lm = case.oracle_request(pools, b, mx=True)
    rms = np.sqrt(np.mean(om ** 2))
    err = np.abs(out[b] - om).max(axis=1) / rms
    bad = np.nonzero(err > 1e-3)[0]
    print(f"req {b} L={lens[b]} max/rms={err.max():.2e} bad rows={bad.tolist()[:20]} n_bad={len(bad)} lse_err={np.abs(lse[b]-lm).max():.2e}")
    if len(bad):
        r = bad[0]; d = np.abs(out[b, r] - om[r]) / rms
        print("  row", r, "bad dims", np.nonzero(d > 1e-3)[0][:40].tolist())
