"""a1 parity: the CUDA quantize-on-append must match the oracle bit-exactly on
all three cache planes (codes, BF16 pre-scaled RoPE, fp32 scales)."""
import numpy as np
import pytest
import torch

from gpu_cases import Case, cache_to_numpy
from oracle import snapmla as O
from paper_2602_10718_b200 import ops

pytestmark = pytest.mark.gpu


def _assert_pools_equal(a, b):
    for k in ("kv_fp8", "kv_rope", "kv_scale"):
        x, y = a[k], b[k]
        if k == "kv_scale":
            x, y = x.view(np.uint32), y.view(np.uint32)
        bad = np.flatnonzero((x != y).ravel())
        assert bad.size == 0, f"{k}: {bad.size} mismatches, first at {bad[:5]}"


def test_append_tiny_bitexact():
    c = Case([256], 16, seed=0)
    _assert_pools_equal(cache_to_numpy(c.gpu_cache()), c.oracle_pools())


@pytest.mark.parametrize("dist", ["mla", "iid"])
def test_append_100k_tokens_page_crossings(dist):
    rng = np.random.default_rng(1)
    lens = rng.integers(1, 3000, 70)
    c = Case(lens, 16, seed=2, dist=dist)
    assert c.lens.sum() > 90000
    _assert_pools_equal(cache_to_numpy(c.gpu_cache()), c.oracle_pools())


def test_append_special_values_bitexact():
    """signed zeros, all-zero latent (sigma clamp), tiny / huge amax, outlier
    tokens, subnormal BF16 RoPE, every BF16 bit pattern as content."""
    c = Case([64 * 40], 16, seed=3, extra_pages=0)
    cv = c.c_kv.clone()
    kp = c.k_pe.clone()
    n = cv.shape[0]
    cv[0] = 0.0
    cv[1] = -0.0
    cv[2, ::2] = -0.0
    cv[3] *= 1e-30                   # amax far below 448 * 2^-24: clamp
    cv[4] *= 1e30                    # huge amax
    cv[5, 7] = 3e38                  # single outlier dominates the scale
    kp[0:8] = torch.tensor(1e-40).to(torch.bfloat16)    # subnormal rope
    kp[8] = -0.0
    # all finite BF16 patterns, 512 per token
    allbits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    vals = torch.from_numpy(allbits.view(np.int16)).view(torch.bfloat16)
    vals = vals[torch.isfinite(vals)]
    k = vals.numel() // 512
    cv[16:16 + k] = vals[:k * 512].reshape(k, 512)
    # same patterns scaled so that every token has a different sigma
    cv[16 + k:16 + 2 * k] = (vals[:k * 512].float().reshape(k, 512) * 2.0 ** -40).to(torch.bfloat16)
    assert 16 + 2 * k < n
    c.c_kv, c.k_pe = cv, kp
    _assert_pools_equal(cache_to_numpy(c.gpu_cache()), c.oracle_pools())


def test_append_sequential_steps_match_oracle():
    """decode-style appends: one token per request per call, seq_lens growing."""
    rng = np.random.default_rng(4)
    B, steps = 8, 70
    c = Case([steps] * B, 16, seed=5)
    dev = "cuda"
    cache = ops.PagedMLACache(c.num_pages, dev)
    bt = torch.from_numpy(c.bt).to(dev)
    cv = c.c_kv.reshape(B, steps, 512)
    kp = c.k_pe.reshape(B, steps, 64)
    for t in range(steps):
        sl = torch.full((B,), t + 1, dtype=torch.int32, device=dev)
        cache.append(cv[:, t].contiguous().to(dev), kp[:, t].contiguous().to(dev), bt, sl)
    torch.cuda.synchronize()
    _assert_pools_equal(cache_to_numpy(cache), c.oracle_pools())


def test_append_cvt_rounding_sweep():
    """x / sigma sweeps the whole E4M3 range incl. ties and subnormals: tokens
    whose amax element is 448 * 2^e and whose other elements are BF16 grid
    points between 2^-12 and 448 in that token's scale."""
    rng = np.random.default_rng(6)
    n = 4096
    e = rng.integers(-30, 30, n)
    mant = rng.integers(0, 128, (n, 511))
    ex = rng.integers(-12, 9, (n, 511))
    sign = rng.choice([-1.0, 1.0], (n, 511))
    body = sign * (1 + mant / 128.0) * np.exp2(ex) * np.exp2(e)[:, None]
    body = np.clip(body, -448 * np.exp2(e)[:, None], 448 * np.exp2(e)[:, None])
    cvals = np.concatenate([448 * np.exp2(e)[:, None], body], axis=1)
    c = Case([n], 16, seed=7, extra_pages=0)
    c.c_kv = torch.from_numpy(cvals.astype(np.float32)).to(torch.bfloat16)
    _assert_pools_equal(cache_to_numpy(c.gpu_cache()), c.oracle_pools())
