"""Diagnostic: per-head parity of the CUDA decode vs O7 / O6 (fp32 combine output)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
from gpu_cases import Case, parity_stats
from oracle import snapmla as O

for (lens, H, seed, dist) in [([256], 16, 0, "mla"), ([256], 16, 0, "iid"), ([4096], 16, 1, "mla"), ([700, 64, 1, 2049], 64, 2, "mla")]:
    case = Case(lens, H, seed=seed, dist=dist)
    cache = case.gpu_cache()
    out32, lse32 = case.gpu_decode(cache, f32_out=True)
    outb, _ = case.gpu_decode(cache)
    pools = case.oracle_pools()
    for b in range(case.B):
        o7, l7 = case.oracle_request(pools, b)
        o6, l6 = case.oracle_request(pools, b, which="o6")
        rms = np.sqrt(np.mean(o7**2))
        d = np.abs(out32[b] - o7) / rms
        db = np.abs(outb[b] - o7) / rms
        d76 = np.abs(o7 - o6) / rms
        print(f"lens={lens} H={H} {dist} b={b} L={case.lens[b]}: f32 max {d.max():.2e} mean {d.mean():.2e} | bf16 max {db.max():.2e} mean {db.mean():.2e} | O7-O6 max {d76.max():.2e} | lse {np.abs(lse32[b]-l7).max():.2e}")
        print("   per-head f32 max:", np.array2string(d.max(1)[:16], precision=1))
        print("   max|o|/rms", np.abs(o7).max()/rms)
