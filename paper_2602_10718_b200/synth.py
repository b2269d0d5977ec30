"""Seeded synthetic inputs shared by tests, bench and smoke.

Holds NONE of the method's arithmetic: it only draws BF16 inputs (latent
c_kv, post-RoPE k_pe, absorbed q), paged block tables and sequence lengths.
The recipe follows the paper's description of the MLA cache:
the RoPE part "spans a significantly wider dynamic range (reaching +-10^3),
exhibiting distinct outlier tails, while the content component is tightly
concentrated around zero (within +-10^1)".

  latent  c[t,i] = mu_i + s_i z,  mu_i ~ N(0, 0.5^2), s_i ~ logN(0, 0.5^2),
          1% outlier tokens x5
  rope    N(0, 30^2) with a 1% x20 tail, clipped to +-1e3
  q       q_c ~ N(0, 1), q_r ~ N(0, 0.1^2)   (logit std ~2 at scale 1/sqrt(192))
  "iid"   variant: everything N(0, 1) (zero-mean, parity-suite stress case)

numpy PCG64 for the CPU-sized cases, torch.Generator on the device for the
bench-sized caches.  BF16 rounding of the draws is done by torch's cast.
"""
import numpy as np
import torch

D_C, D_R, PAGE = 512, 64, 64
DEFAULT_SOFTMAX_SCALE = 1.0 / np.sqrt(192.0)   # DeepSeek qk_head_dim 192 (reading R8)


def _bf16(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16)


def latent_tokens(rng, n, dist="mla"):
    """(c_kv [n,512], k_pe [n,64]) as torch.bfloat16 CPU tensors."""
    if dist == "iid":
        return _bf16(rng.standard_normal((n, D_C))), _bf16(rng.standard_normal((n, D_R)))
    mu = rng.normal(0.0, 0.5, D_C)
    sc = np.exp(rng.normal(0.0, 0.5, D_C))
    c = mu[None, :] + sc[None, :] * rng.standard_normal((n, D_C))
    out = rng.random(n) < 0.01
    c[out] *= 5.0
    r = rng.normal(0.0, 30.0, (n, D_R))
    tail = rng.random((n, D_R)) < 0.01
    r[tail] *= 20.0
    r = np.clip(r, -1e3, 1e3)
    return _bf16(c), _bf16(r)


def queries(rng, rows, dist="mla"):
    """q [rows,576] torch.bfloat16 (absorbed q_nope | q_pe)."""
    if dist == "iid":
        return _bf16(rng.standard_normal((rows, D_C + D_R)))
    qc = rng.standard_normal((rows, D_C))
    qr = rng.normal(0.0, 0.1, (rows, D_R))
    return _bf16(np.concatenate([qc, qr], axis=1))


def paged_layout(rng, seq_lens, extra_pages=0, max_pages_per_seq=None):
    """Random page permutation: returns (block_table int32 [B, maxp], num_pages).
    Every request gets ceil(L/64) distinct pages drawn from a shuffled pool."""
    seq_lens = np.asarray(seq_lens, dtype=np.int64)
    need = (seq_lens + PAGE - 1) // PAGE
    maxp = int(max(1, need.max())) if max_pages_per_seq is None else int(max_pages_per_seq)
    num_pages = int(need.sum()) + int(extra_pages)
    perm = rng.permutation(num_pages)
    bt = np.zeros((len(seq_lens), maxp), dtype=np.int32)
    k = 0
    for b, n in enumerate(need):
        bt[b, :n] = perm[k:k + n]
        k += n
    return bt, num_pages


def torch_latent(n, gen, device):
    """Device-side draw for bench-sized caches (same recipe as latent_tokens)."""
    mu = torch.randn(D_C, generator=gen, device=device) * 0.5
    sc = torch.exp(torch.randn(D_C, generator=gen, device=device) * 0.5)
    c = mu + sc * torch.randn(n, D_C, generator=gen, device=device)
    out = torch.rand(n, generator=gen, device=device) < 0.01
    c = torch.where(out[:, None], c * 5.0, c)
    r = torch.randn(n, D_R, generator=gen, device=device) * 30.0
    tail = torch.rand(n, D_R, generator=gen, device=device) < 0.01
    r = torch.clamp(torch.where(tail, r * 20.0, r), -1e3, 1e3)
    return c.to(torch.bfloat16), r.to(torch.bfloat16)


def torch_queries(rows, gen, device):
    qc = torch.randn(rows, D_C, generator=gen, device=device)
    qr = torch.randn(rows, D_R, generator=gen, device=device) * 0.1
    return torch.cat([qc, qr], dim=1).to(torch.bfloat16)
