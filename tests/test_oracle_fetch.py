"""Pins of the oracle's Fused-Fetch-Dequant (NEXT-3, §3.3; SPEC
fused_fetch_dequant; reading R26: fp32 RNE product, then RNE to BF16)."""
import numpy as np
import torch

from oracle import snapmla as O
from paper_2602_10718_b200 import synth


def _pools(L, seed, pow2=False):
    rng = np.random.default_rng(seed)
    bt, npages = synth.paged_layout(rng, [L], extra_pages=1)
    c, r = synth.latent_tokens(rng, L)
    c, r = c.float().numpy(), r.float().numpy()
    if pow2:   # content amax a power of two times 448 -> sigma is a power of two
        c = c / np.abs(c).max(axis=1, keepdims=True) * (448.0 * 2.0 ** rng.integers(-6, 4, size=(L, 1)))
        c = torch.from_numpy(c).to(torch.bfloat16).float().numpy()
    pools = dict(kv_fp8=np.zeros((npages, 64, 512), np.uint8), kv_rope=np.zeros((npages, 64, 64), np.uint16),
                 kv_scale=np.zeros((npages, 64), np.float32))
    for t in range(L):
        O.append_to_pools(pools, c[t:t + 1], r[t:t + 1], bt, np.array([t + 1]))
    return pools, bt[0], c, r


def test_fetch_vs_torch_dequant():
    """independent dequantization: torch float8_e4m3fn decode, fp32 multiply, torch BF16 cast."""
    pools, bt, _, _ = _pools(150, seed=1)
    cb, rb = O.fetch_dequant(pools, bt, 10, 120)
    slots = np.array([O.slot_of(bt, 10 + i) for i in range(120)])
    codes = torch.from_numpy(pools["kv_fp8"].reshape(-1, 512)[slots]).view(torch.float8_e4m3fn).float()
    rope = torch.from_numpy(pools["kv_rope"].reshape(-1, 64)[slots].view(np.int16)).view(torch.bfloat16).float()
    sig = torch.from_numpy(pools["kv_scale"].reshape(-1)[slots])[:, None]
    c_ref = (codes * sig).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    r_ref = (rope * sig).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    np.testing.assert_array_equal(cb, c_ref)
    np.testing.assert_array_equal(rb, r_ref)


def test_fetch_pow2_scales_recover_rope_exactly():
    """SPEC example: power-of-two sigma -> k_r / sigma and * sigma are exact."""
    pools, bt, c, r = _pools(70, seed=2, pow2=True)
    sig = pools["kv_scale"].reshape(-1)[[O.slot_of(bt, i) for i in range(70)]]
    assert np.all(np.log2(sig) == np.round(np.log2(sig)))
    _, rb = O.fetch_dequant(pools, bt, 0, 70)
    r_bits = torch.from_numpy(r).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    np.testing.assert_array_equal(rb, r_bits)


def test_fetch_content_round_trip_bound():
    """|fetch(append(c)) - c| <= max(2^-4 |c|, 2^-10 sigma) (E4M3) + BF16 output rounding."""
    pools, bt, c, _ = _pools(130, seed=3)
    cb, _ = O.fetch_dequant(pools, bt, 0, 130)
    got = O.bf16_bits_to_f64(cb)
    sig = pools["kv_scale"].reshape(-1)[[O.slot_of(bt, i) for i in range(130)]].astype(np.float64)[:, None]
    bound = np.maximum(2.0 ** -4 * np.abs(c), 2.0 ** -10 * sig)
    err = np.abs(got - c)
    assert np.all(err <= bound * (1 + 2.0 ** -8) + 2.0 ** -8 * np.abs(got) + 1e-30)


def test_fetch_composes_across_page_boundaries():
    pools, bt, _, _ = _pools(200, seed=4)
    whole = O.fetch_dequant(pools, bt, 30, 150)
    a = O.fetch_dequant(pools, bt, 30, 34)       # ends exactly at the page boundary 64
    b = O.fetch_dequant(pools, bt, 64, 116)
    np.testing.assert_array_equal(whole[0], np.concatenate([a[0], b[0]]))
    np.testing.assert_array_equal(whole[1], np.concatenate([a[1], b[1]]))
