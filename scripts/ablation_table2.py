"""NEXT-4(a): Table 2 / Fig. 5 numerical-accuracy ablation on synthetic MLA-like
data (the paper uses real LongCat-Flash-Thinking activations, which are not
available here).  For each "layer" (a seeded synthetic cache of the given context
and distribution) and each KV-cache quantization configuration of Table 2, the
attention output vs the BF16 ground truth (O8, fp64 over the unquantized inputs):
RMSE, cosine difference, relative L2.  Rows:
  snapmla_kv / A / B / C / D   exact softmax over the dequantized cache (KV-only)
  snapmla_full                 the full SnapMLA decode (O7: + Q quant, + block P quant)
  full_mx32 / full_mx64        NEXT-4(b) variant: the same with MX power-of-two P scales per
                               32 / 64 tokens instead of sigma_p = M/448 (not the method)
  python scripts/ablation_table2.py [context] [heads] [n_layers] > profiles/...json
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from oracle import snapmla as O  # noqa: E402
from paper_2602_10718_b200 import synth  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
H = int(sys.argv[2]) if len(sys.argv) > 2 else 64
N_LAYERS = int(sys.argv[3]) if len(sys.argv) > 3 else 4
SCALE = synth.DEFAULT_SOFTMAX_SCALE
CONFIGS = ["snapmla", "A", "B", "C", "D"]

t0 = time.time()
layers = []
for li in range(N_LAYERS):
    dist = "mla" if li % 2 == 0 else "iid"
    rng = np.random.default_rng(1000 + li)
    c, r = synth.latent_tokens(rng, L, dist)
    q = synth.queries(rng, H, dist)
    c, r, q = c.float().numpy(), r.float().numpy(), q.float().numpy()
    o8, _ = O.attn_o8(q, c, r, SCALE)
    row = {"layer": li, "dist": dist}
    for cfg in CONFIGS:
        cq, rq = O.kv_quant_config(c, r, cfg)
        o, _ = O.attn_dequantized(q, cq, rq, SCALE)
        m = O.error_metrics(o, o8)
        row[cfg] = {k: m[k] for k in ("rmse", "cos_diff", "rel_l2")}
    kc, sk, kr = O.append_quant(c, r)
    qc, sq, qr = O.q_quant(q)
    o7, _ = O.decode_o7(qc, sq, qr, kc, sk, kr, SCALE)
    m = O.error_metrics(o7, o8)
    row["snapmla_full"] = {k: m[k] for k in ("rmse", "cos_diff", "rel_l2")}
    for g in (32, 64):
        om, _ = O.decode_o7(qc, sq, qr, kc, sk, kr, SCALE, p_mx_group=g)
        m = O.error_metrics(om, o8)
        row[f"full_mx{g}"] = {k: m[k] for k in ("rmse", "cos_diff", "rel_l2")}
    layers.append(row)

summary = {}
for cfg in CONFIGS + ["snapmla_full", "full_mx32", "full_mx64"]:
    summary[cfg] = {k: float(np.mean([lay[cfg][k] for lay in layers])) for k in ("rmse", "cos_diff", "rel_l2")}
print(json.dumps({"what": "Table 2 configurations vs BF16 ground truth (O8), synthetic MLA-like caches",
                  "context": L, "heads": H, "layers": N_LAYERS, "softmax_scale": SCALE,
                  "mean_over_layers": summary, "per_layer": layers, "cpu_seconds": round(time.time() - t0, 1)}))
