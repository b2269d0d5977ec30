import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
from gpu_cases import Case
from paper_2602_10718_b200 import ops
ops.lib().mla_debug_set_pair(int(os.environ.get("V", "2")))
case = Case([int(x) for x in os.environ.get("LENS", "1").split(",")], 128, seed=5)
cache = case.gpu_cache()
try:
    out, lse = case.gpu_decode(cache, f32_out=True)
    print("ok", np.abs(out).max())
except Exception as e:
    print("ERR", e)
    torch.cuda.synchronize()
