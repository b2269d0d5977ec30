"""Pins of the Table-2 KV quantization configurations (NEXT-4(a), P:413-429;
granularities of Appendix A)."""
import numpy as np
import torch

from oracle import snapmla as O
from paper_2602_10718_b200 import synth


def _data(L=200, seed=0):
    rng = np.random.default_rng(seed)
    c, r = synth.latent_tokens(rng, L)
    return c.float().numpy().astype(np.float64), r.float().numpy().astype(np.float64)


def _torch_fp8(x):   # torch's own E4M3 RNE cast (satfinite inputs only)
    return torch.from_numpy(np.asarray(x, np.float32)).to(torch.float8_e4m3fn).to(torch.float64).numpy()


def test_config_b_is_plain_e4m3_cast():
    c, r = _data(seed=1)
    cq, rq = O.kv_quant_config(c, r, "B")
    np.testing.assert_array_equal(cq, _torch_fp8(c))
    np.testing.assert_array_equal(rq, r)


def test_config_c_scale_is_global_amax():
    c, r = _data(seed=2)
    cq, _ = O.kv_quant_config(c, r, "C")
    s = np.abs(c).max() / 448.0
    np.testing.assert_array_equal(cq, _torch_fp8((c / s).astype(np.float32)) * s)
    assert np.isclose(np.abs(cq).max(), np.abs(c).max(), rtol=2.0 ** -4)


def test_config_d_blocks_are_independent():
    c, r = _data(L=130, seed=3)
    cq, _ = O.kv_quant_config(c, r, "D", block=64)
    for i in (0, 64, 128):
        for j in (0, 256, 448):
            blk = c[i:i + 64, j:j + 64]
            s = np.abs(blk).max() / 448.0
            np.testing.assert_array_equal(cq[i:i + 64, j:j + 64], _torch_fp8((blk / s).astype(np.float32)) * s)


def test_config_a_quantizes_rope_and_snapmla_keeps_it():
    c, r = _data(seed=4)
    _, ra = O.kv_quant_config(c, r, "A")
    _, rs = O.kv_quant_config(c, r, "snapmla")
    err_a = np.abs(ra - r).max() / np.abs(r).max()
    err_s = np.abs(rs - r).max() / np.abs(r).max()
    assert err_s <= 2.0 ** -8 + 1e-12          # BF16 of r / sigma, times sigma
    assert err_a > 4 * err_s                   # RoPE-unaware per-token FP8 loses the RoPE precision


def test_snapmla_config_matches_append_quant():
    c, r = _data(seed=5)
    cq, rq = O.kv_quant_config(c, r, "snapmla")
    codes, sig, rbits = O.append_quant(c.astype(np.float32), r.astype(np.float32))
    np.testing.assert_array_equal(cq, O.decode_e4m3(codes) * sig.astype(np.float64)[:, None])


def test_attn_dequantized_identity_is_o8():
    c, r = _data(L=90, seed=6)
    q = synth.queries(np.random.default_rng(7), 8).float().numpy()
    o1, l1 = O.attn_dequantized(q, c, r, 0.07)
    o2, l2 = O.attn_o8(q, c, r, 0.07)
    np.testing.assert_allclose(o1, o2, rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(l1, l2, rtol=1e-13)
