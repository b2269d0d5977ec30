"""Pins for the oracle decode: O7 (gate), Algorithm-1 recurrence, O6, O8, combine.

Independent anchors: torch SDPA / logsumexp in fp64 with torch's own FP8 and
BF16 dequantization; special cases with exact answers; the E4M3 rounding
bound on |O7 - O6|; split invariance; the paper's Eq.7 worked value.
"""
import json
import math
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import snapmla as O
from paper_2602_10718_b200 import synth

SCALE = synth.DEFAULT_SOFTMAX_SCALE
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def _case(L, H=16, seed=0, dist="mla"):
    rng = np.random.default_rng(seed)
    c, r = synth.latent_tokens(rng, L, dist)
    q = synth.queries(rng, H, dist)
    c, r, q = c.float().numpy(), r.float().numpy(), q.float().numpy()
    kc, sk, kr = O.append_quant(c, r)
    qc, sq, qr = O.q_quant(q)
    return dict(c=c, r=r, q=q, kc=kc, sk=sk, kr=kr, qc=qc, sq=sq, qr=qr)


def _args(d):
    return d["qc"], d["sq"], d["qr"], d["kc"], d["sk"], d["kr"]


def _torch_deq(codes, sigma, rope_bits):
    """dequantize with torch's own FP8 / BF16 types (independent of oracle.codec)."""
    cd = torch.from_numpy(codes).view(torch.float8_e4m3fn).to(torch.float64)
    rd = torch.from_numpy(rope_bits.view(np.int16)).view(torch.bfloat16).to(torch.float64)
    s = torch.from_numpy(sigma.astype(np.float64))[:, None]
    return torch.cat([cd, rd], dim=1) * s, cd * s


def _sdpa(q, k, v, scale):
    o = F.scaled_dot_product_attention(q[None, None], k[None, None], v[None, None], scale=scale)[0, 0]
    lse = torch.logsumexp(scale * (q @ k.T), dim=1)
    return o.numpy(), lse.numpy()


@pytest.mark.parametrize("L", [1, 5, 64, 300])
def test_o6_vs_torch_sdpa(L):
    d = _case(L, seed=L)
    qd, _ = _torch_deq(d["qc"], d["sq"], d["qr"])
    kd, vd = _torch_deq(d["kc"], d["sk"], d["kr"])
    o_ref, lse_ref = _sdpa(qd, kd, vd, SCALE)
    o, lse = O.attn_o6(*_args(d), SCALE)
    np.testing.assert_allclose(o, o_ref, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(lse, lse_ref, rtol=1e-12, atol=1e-12)


def test_o8_vs_torch_sdpa():
    d = _case(200, seed=11)
    q = torch.from_numpy(d["q"].astype(np.float64))
    k = torch.from_numpy(np.concatenate([d["c"], d["r"]], 1).astype(np.float64))
    v = torch.from_numpy(d["c"].astype(np.float64))
    o_ref, lse_ref = _sdpa(q, k, v, SCALE)
    o, lse = O.attn_o8(d["q"], d["c"], d["r"], SCALE)
    np.testing.assert_allclose(o, o_ref, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(lse, lse_ref, rtol=1e-12)


@pytest.mark.parametrize("L", [1, 64, 129, 700])
def test_o7_identity_rounding_equals_o6(L):
    d = _case(L, seed=100 + L)
    o7, l7 = O.decode_o7(*_args(d), SCALE, p_quant=False)
    o6, l6 = O.attn_o6(*_args(d), SCALE)
    np.testing.assert_allclose(o7, o6, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(l7, l6, rtol=1e-13)


@pytest.mark.parametrize("L", [1, 63, 64, 65, 100, 128, 192, 1000, 1024])
@pytest.mark.parametrize("dist", ["mla", "iid"])
def test_o7_equals_algorithm1_recurrence(L, dist):
    d = _case(L, seed=L + 7, dist=dist)
    o7, l7 = O.decode_o7(*_args(d), SCALE)
    oa, la = O.decode_alg1(*_args(d), SCALE)
    rms = np.sqrt(np.mean(o7 ** 2))
    assert np.max(np.abs(o7 - oa)) <= 1e-12 * rms
    np.testing.assert_allclose(l7, la, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("L", [64, 257, 2000])
def test_o7_within_e4m3_bound_of_o6(L):
    """Each P' carries at most half an E4M3 ulp of relative error (2^-4), or
    2^-10 of the block scale in the subnormal range, so
    |O7 - O6| <= sum_j max(2^-4 w_j, 2^-10 M_b/448) |dec(kc_j)| / sum_j e_j."""
    d = _case(L, seed=L)
    o7, _ = O.decode_o7(*_args(d), SCALE)
    o6, _ = O.attn_o6(*_args(d), SCALE)
    s = O.logits(*_args(d), SCALE)
    e = np.exp(s - s.max(1, keepdims=True))
    w = e * d["sk"][None].astype(np.float64)
    Mb = np.repeat(np.stack([w[:, i:i + 64].max(1) for i in range(0, L, 64)], 1), 64, axis=1)[:, :L]
    err_w = np.maximum(2.0 ** -4 * w, 2.0 ** -10 * Mb / 448)
    bound = (err_w @ np.abs(O.decode_e4m3(d["kc"]))) / e.sum(1, keepdims=True)
    assert np.all(np.abs(o7 - o6) <= bound * (1 + 1e-9))
    assert np.max(np.abs(o7 - o6)) > 0      # P quantization really happened


def test_single_token():
    d = _case(1, seed=3)
    o7, l7 = O.decode_o7(*_args(d), SCALE)
    v = O.decode_e4m3(d["kc"][0]) * np.float64(d["sk"][0])
    np.testing.assert_array_equal(o7, np.broadcast_to(v, o7.shape))   # P' = 448 exactly
    np.testing.assert_allclose(l7, O.logits(*_args(d), SCALE)[:, 0], rtol=1e-15)


def test_duplicated_tokens_lse_plus_ln2():
    d = _case(1, seed=4)
    d2 = dict(d, kc=np.repeat(d["kc"], 2, 0), sk=np.repeat(d["sk"], 2), kr=np.repeat(d["kr"], 2, 0))
    o1, l1 = O.decode_o7(*_args(d), SCALE)
    o2, l2 = O.decode_o7(*_args(d2), SCALE)
    np.testing.assert_allclose(l2, l1 + math.log(2.0), rtol=1e-14)
    np.testing.assert_allclose(o2, o1, rtol=1e-14)


def test_constant_logits_equal_scales_give_mean():
    """q = 0 -> all logits 0; tokens built with equal sigma_K inside each block
    -> every P' = 448 and O7 is the plain mean of V_deq."""
    L = 150
    rng = np.random.default_rng(12)
    c = rng.uniform(-1, 1, (L, 512)).astype(np.float32)
    blk_amax = np.repeat(np.array([3.0, 0.5, 7.0]), 64)[:L].astype(np.float32)
    c[:, 0] = blk_amax
    c = np.clip(c, -blk_amax[:, None], blk_amax[:, None])
    c = torch.from_numpy(c).to(torch.bfloat16).float().numpy()
    r = synth.latent_tokens(rng, L)[1].float().numpy()
    kc, sk, kr = O.append_quant(c, r)
    qc, sq, qr = O.q_quant(np.zeros((4, 576), np.float32))
    o7, l7 = O.decode_o7(qc, sq, qr, kc, sk, kr, SCALE)
    mean = (O.decode_e4m3(kc) * sk[:, None].astype(np.float64)).mean(0)
    np.testing.assert_allclose(o7, np.broadcast_to(mean, o7.shape), rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(l7, math.log(L), rtol=1e-14)


@pytest.mark.parametrize("cut", [1, 3, 6])
def test_block_aligned_split_plus_combine_equals_unsplit(cut):
    d = _case(7 * 64 - 5, seed=cut)
    o, l = O.decode_o7(*_args(d), SCALE)
    pa = O.decode_o7(*_args(d), SCALE, block_range=(0, cut))
    pb = O.decode_o7(*_args(d), SCALE, block_range=(cut, 7))
    oc, lc = O.combine(np.stack([pa[0], pb[0]]), np.stack([pa[1], pb[1]]))
    np.testing.assert_allclose(oc, o, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(lc, l, rtol=1e-13)


def test_combine_special_cases():
    rng = np.random.default_rng(0)
    o = rng.standard_normal((3, 512))
    lse = rng.standard_normal(3)
    oc, lc = O.combine(o[None], lse[None])
    np.testing.assert_array_equal(oc, o)
    np.testing.assert_array_equal(lc, lse)
    oc, lc = O.combine(np.stack([o, o]), np.stack([lse, lse]))
    np.testing.assert_allclose(oc, o, rtol=1e-15)
    np.testing.assert_allclose(lc, lse + math.log(2), rtol=1e-15)
    # weights e^{L_s - L}: a split with lse -inf-like contributes nothing
    oc, lc = O.combine(np.stack([o, 5 * o]), np.stack([lse, lse - 800]))
    np.testing.assert_allclose(oc, o, rtol=1e-15)


def test_request_from_pools_matches_gathered():
    rng = np.random.default_rng(13)
    L = 200
    bt, npages = synth.paged_layout(rng, [L], extra_pages=2)
    c, r = synth.latent_tokens(rng, L)
    q = synth.queries(rng, 16).float().numpy()
    pools = dict(kv_fp8=np.zeros((npages, 64, 512), np.uint8),
                 kv_rope=np.zeros((npages, 64, 64), np.uint16),
                 kv_scale=np.zeros((npages, 64), np.float32))
    c, r = c.float().numpy(), r.float().numpy()
    for t in range(L):
        O.append_to_pools(pools, c[t:t + 1], r[t:t + 1], bt, np.array([t + 1]))
    o, l = O.decode_request(q, pools, bt[0], L, SCALE)
    kc, sk, kr = O.append_quant(c, r)
    qc, sq, qr = O.q_quant(q)
    o2, l2 = O.decode_o7(qc, sq, qr, kc, sk, kr, SCALE)
    np.testing.assert_array_equal(o, o2)


def test_eq7_effective_peak():
    g = GOLD["eq7_effective_peak_tflops"]
    assert round(O.effective_peak(GOLD["eq7_bf16_peak_tflops"]["value"]), g["digits"]) == g["value"]


def test_error_metrics_definitions():
    ref = np.array([3.0, 4.0])
    m = O.error_metrics(ref * 2, ref)
    assert m["rel_l2"] == pytest.approx(1.0)
    assert m["cos_diff"] == pytest.approx(0.0, abs=1e-15)
    assert m["rmse"] == pytest.approx(np.sqrt((9 + 16) / 2))


# ---- MTP (NEXT-1, reading R25): the causal mask convention pinned against torch SDPA
@pytest.mark.parametrize("L,T", [(5, 2), (64, 2), (130, 3), (1, 2)])
def test_o8_mtp_vs_torch_masked_sdpa(L, T):
    rng = np.random.default_rng(31 + L)
    H = 3
    c = rng.normal(size=(L, 512))
    r = rng.normal(size=(L, 64))
    q = rng.normal(size=(T, H, 576))
    o, lse = O.attn_o8_mtp(q, c, r, SCALE)
    k = torch.from_numpy(np.concatenate([c, r], 1))
    v = torch.from_numpy(c)
    qt = torch.from_numpy(q.reshape(T * H, 576))
    tok = np.repeat(np.arange(T), H)
    visible = torch.from_numpy(np.arange(L)[None, :] <= (L - T + tok)[:, None])   # key j visible to row
    for row in range(T * H):
        t, h = divmod(row, H)
        if not visible[row].any():
            assert np.all(o[t, h] == 0) and lse[t, h] == -np.inf
            continue
        o_ref = F.scaled_dot_product_attention(qt[row][None, None, None], k[None, None], v[None, None],
                                               attn_mask=visible[row][None, None, None], scale=SCALE)[0, 0, 0]
        s = SCALE * (qt[row] @ k.T)
        lse_ref = torch.logsumexp(s[visible[row]], dim=0)
        np.testing.assert_allclose(o[t, h], o_ref.numpy(), rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(lse[t, h], lse_ref.item(), rtol=1e-12)


def _pools_for(d):
    """the case's tokens in a fresh paged pool (identity page order)."""
    L = len(d["c"])
    npages = (L + 63) // 64
    pools = dict(kv_fp8=np.zeros((npages, 64, 512), np.uint8), kv_rope=np.zeros((npages, 64, 64), np.uint16),
                 kv_scale=np.zeros((npages, 64), np.float32))
    slots = np.arange(L)
    pools["kv_fp8"].reshape(-1, 512)[slots] = d["kc"]
    pools["kv_rope"].reshape(-1, 64)[slots] = d["kr"]
    pools["kv_scale"].reshape(-1)[slots] = d["sk"]
    return pools, np.arange(npages)


def test_mtp_last_token_is_single_token_decode():
    d = _case(200, seed=41)
    pools, bt = _pools_for(d)
    q2 = np.stack([d["q"], d["q"][::-1].copy()])               # [2, H, 576]
    o2, l2 = O.decode_request_mtp(q2, pools, bt, 200, SCALE)
    o1, l1 = O.decode_request(q2[1], pools, bt, 200, SCALE)
    o0, l0 = O.decode_request(q2[0], pools, bt, 199, SCALE)
    np.testing.assert_array_equal(o2[1], o1)
    np.testing.assert_array_equal(o2[0], o0)
    np.testing.assert_array_equal(l2[0], l0)
