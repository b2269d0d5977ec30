import os, sys, ctypes
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
from gpu_cases import Case
from oracle import snapmla as O, codec as C
from paper_2602_10718_b200 import ops
L = ops.lib()
L.mla_debug_set_pair(2)
case = Case([64], 128, seed=5)
cache = case.gpu_cache()
dump = torch.zeros(128 * 64, dtype=torch.float32, device="cuda")
L.mla_debug_set_trace.argtypes = [ctypes.c_void_p]
L.mla_debug_set_trace(ctypes.c_void_p(dump.data_ptr()))
case.gpu_decode(cache, f32_out=True)
L.mla_debug_set_trace(None)
S = dump.view(128, 64).cpu().numpy()
pools = case.oracle_pools()
qc, sq, qr = O.q_quant(case.q[0].float().numpy())
kc, sk, kr = O.gather_request(pools, case.bt[0], 64)
dq = C.decode_e4m3(qc).astype(np.float64); dk = C.decode_e4m3(kc).astype(np.float64)
bq = C.bf16_bits_to_f64(qr).astype(np.float64) if hasattr(C, "bf16_bits_to_f64") else None
print([n for n in dir(C) if not n.startswith("_")])
ref = dq @ dk.T
if bq is not None:
    ref = ref + bq @ C.bf16_bits_to_f64(kr).astype(np.float64).T
for half in (0, 1):
    d = np.abs(S[:, 32 * half:32 * half + 32] - ref[:, 32 * half:32 * half + 32])
    print("half", half, "max abs diff", d.max(), "rel", d.max() / np.abs(ref).max())
print("S[0,30:36]", S[0, 30:36]); print("ref[0,30:36]", ref[0, 30:36])
print("S[70,30:36]", S[70, 30:36]); print("ref[70,30:36]", ref[70, 30:36])
rc = dq @ dk.T
rr = bq @ C.bf16_bits_to_f64(kr).astype(np.float64).T
h = slice(32, 64)
for name, guess in [("content only", rc[:, h]), ("rope only", rr[:, h]), ("content + rope of tokens 0-31", (rc + rr)[:, 0:32]),
                    ("content(32-63)+rope(0-31)", rc[:, h] + rr[:, 0:32]), ("content(0-31)+rope(32-63)", rc[:, 0:32] + rr[:, h])]:
    d = np.abs(S[:, h] - guess)
    print(f"{name:35s} max rel {d.max() / np.abs(guess).max():.3e}")
