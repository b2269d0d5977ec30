import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
from gpu_cases import Case, parity_stats
from paper_2602_10718_b200 import ops
ops.lib().mla_debug_set_pair(2)
for lens in ([2], [31], [32], [33], [63], [64], [65], [128], [2, 63], [700]):
    case = Case(lens, 128, seed=5)
    cache = case.gpu_cache()
    out, lse = case.gpu_decode(cache, f32_out=True)
    pools = case.oracle_pools()
    errs = []
    for b in range(case.B):
        o7, l7 = case.oracle_request(pools, b)
        mx, mn = parity_stats(out[b], o7)
        rows_bad = np.where(np.abs(out[b] - o7).max(axis=1) > 1e-2 * np.abs(o7).max())[0]
        errs.append((round(mx, 4), round(float(np.abs(lse[b] - l7).max()), 4), rows_bad[:8].tolist(), len(rows_bad)))
    print(lens, errs)
