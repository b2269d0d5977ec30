"""Pins of the Table-2 KV quantization configurations (NEXT-4(a), P:413-429;
granularities of Appendix A)."""
import pytest
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


# ---- NEXT-4(b): MX-style power-of-two P scales (a variant, not the method)
@pytest.mark.parametrize("group", [32, 64])
def test_p_quant_mx_vs_torch_cast(group):
    """p_quant_mx against torch's own E4M3 cast (an independent implementation): per (row,
    group) the scale is the power of two 2^ceil(log2(max / 448)) and the codes are
    float8_e4m3fn(w / scale)."""
    rng = np.random.default_rng(group)
    w = rng.exponential(size=(7, 150)) * np.exp(rng.normal(size=(7, 1)) * 3)
    w[2, 40:80] = 0.0   # an all-zero group
    A = O.p_quant_mx(w, group)
    for r in range(w.shape[0]):
        for g0 in range(0, w.shape[1], group):
            blk = w[r, g0:g0 + group]
            M = blk.max()
            if M == 0:
                assert np.all(A[r, g0:g0 + group] == 0)
                continue
            sig = 2.0 ** np.ceil(np.log2(M / 448.0))
            assert M / 448.0 <= sig < 2 * M / 448.0
            ref = torch.from_numpy((blk / sig).astype(np.float32)).to(torch.float8_e4m3fn).double().numpy() * sig
            np.testing.assert_array_equal(A[r, g0:g0 + group], ref)


def test_mx_variant_loses_the_exact_block_max():
    """Why the paper's sigma_p = M/448 matters: it maps each block's largest weight to
    448, which E4M3 represents exactly, so the dominant term of a peaked softmax is exact.  A
    power-of-two MX scale leaves M/sigma in (224, 448], rounded to 3 mantissa bits.  Both stay
    within the E4M3 bound (relative 2^-4 per weight), but on MLA-like logits the MX decode
    error is far larger than the paper's."""
    rng = np.random.default_rng(5)
    c, r = synth.latent_tokens(rng, 700)
    q = synth.queries(rng, 8)
    kc, sk, kr = O.append_quant(c.float().numpy(), r.float().numpy())
    qc, sq, qr = O.q_quant(q.float().numpy())
    s = O.logits(qc, sq, qr, kc, sk, kr, 0.07)
    w = np.exp(s - s.max(axis=1, keepdims=True)) * sk[None, :].astype(np.float64)
    A = O.p_quant_mx(w, 32)
    big = w > 2.0 ** -6 * w.max()            # normal range of E4M3 after scaling
    assert (np.abs(A - w) / w)[big].max() <= 2.0 ** -4
    o_id, _ = O.decode_o7(qc, sq, qr, kc, sk, kr, 0.07, p_quant=False)
    o_p, _ = O.decode_o7(qc, sq, qr, kc, sk, kr, 0.07)
    o_mx, _ = O.decode_o7(qc, sq, qr, kc, sk, kr, 0.07, p_mx_group=32)
    e_p = O.error_metrics(o_p, o_id)["rel_l2"]
    e_mx = O.error_metrics(o_mx, o_id)["rel_l2"]
    assert e_p < 1e-3 and e_mx > 10 * e_p and e_mx < 0.1
