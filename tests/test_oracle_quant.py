"""Pins for oracle per-token quantization (a1 append, a2 q-quant) and paging.

Against: ml_dtypes / torch casts (independent codec), closed-form invariants
(power-of-two invariance, amax -> 448, round-trip bound, Eq.6 recovery) and
brute-force page accounting.
"""
import ml_dtypes
import numpy as np
import torch

from oracle import snapmla as O
from oracle.codec import bf16_bits_to_f64, decode_e4m3
from paper_2602_10718_b200 import synth


def _tokens(n, seed=0, dist="mla"):
    rng = np.random.default_rng(seed)
    c, r = synth.latent_tokens(rng, n, dist)
    return c.float().numpy(), r.float().numpy()


def test_append_vs_independent_libraries():
    c, r = _tokens(2000)
    codes, sig, rope = O.append_quant(c, r)
    # sigma: amax / 448 in fp32, via torch
    amax = torch.from_numpy(c).abs().amax(dim=1)
    sig_t = torch.clamp(amax / 448.0, min=2.0 ** -24).numpy()
    np.testing.assert_array_equal(sig, sig_t)
    # codes: fp32 division then ml_dtypes E4M3 cast (RNE; no saturation needed below 464)
    q = (c / sig[:, None]).astype(np.float32)
    assert np.abs(q).max() < 464.0     # amax/sigma may round a hair above 448; RNE still gives 448
    np.testing.assert_array_equal(codes, q.astype(ml_dtypes.float8_e4m3fn).view(np.uint8))
    # rope': fp32 division then torch bf16 cast
    rr = torch.from_numpy((r / sig[:, None]).astype(np.float32)).to(torch.bfloat16)
    np.testing.assert_array_equal(rope, rr.view(torch.int16).numpy().view(np.uint16))


def test_amax_element_encodes_to_448():
    c, r = _tokens(3000, seed=1)
    c = c * np.exp2(np.random.default_rng(5).integers(-20, 12, (3000, 1))).astype(np.float32)
    c = torch.from_numpy(c).to(torch.bfloat16).float().numpy()
    codes, sig, _ = O.append_quant(c, r)
    unclamped = np.abs(c).max(axis=1) >= 448 * 2.0 ** -24
    am = np.argmax(np.abs(c), axis=1)
    top = codes[np.arange(len(c)), am]
    assert np.all((top[unclamped] & 0x7F) == 0x7E)
    # clamped rows: sigma = 2^-24, so the top code is just E4M3(amax * 2^24) (< 448 unless amax rounds up)
    assert np.all(sig[~unclamped] == np.float32(2.0 ** -24))
    assert np.all(decode_e4m3(top[~unclamped]) <= 448.0)


def test_power_of_two_invariance():
    c, r = _tokens(500, seed=2)
    codes, sig, rope = O.append_quant(c, r)
    for k in (-7, -1, 3, 9):
        c2 = (c * np.float32(2.0 ** k)).astype(np.float32)
        codes2, sig2, rope2 = O.append_quant(c2, r)
        np.testing.assert_array_equal(codes2, codes)
        np.testing.assert_array_equal(sig2, (sig * np.float32(2.0 ** k)).astype(np.float32))


def test_round_trip_bound():
    c, r = _tokens(2000, seed=3, dist="iid")
    codes, sig, _ = O.append_quant(c, r)
    deq = decode_e4m3(codes) * sig[:, None].astype(np.float64)
    bound = np.maximum(2.0 ** -4 * np.abs(c), 2.0 ** -10 * sig[:, None]) * (1 + 2.0 ** -20)
    assert np.all(np.abs(c - deq) <= bound)
    # unclamped sigma: every element within 2^-4 amax
    assert np.all(np.abs(c - deq) <= 2.0 ** -4 * np.abs(c).max(axis=1, keepdims=True) * (1 + 2.0 ** -20))


def test_rope_prescale_recovery_eq6():
    c, r = _tokens(2000, seed=4)
    codes, sig, rope = O.append_quant(c, r)
    rec = bf16_bits_to_f64(rope) * sig[:, None]
    assert np.all(np.abs(rec - r) <= 2.0 ** -8 * np.abs(r) * (1 + 1e-6) + 1e-30)
    # power-of-two scale -> exact recovery
    c2 = np.zeros_like(c)
    c2[:, 0] = 448.0 * 2.0 ** np.random.default_rng(6).integers(-10, 5, len(c))
    _, sig2, rope2 = O.append_quant(c2, r)
    assert np.all(np.log2(sig2) == np.round(np.log2(sig2)))
    np.testing.assert_array_equal(bf16_bits_to_f64(rope2) * sig2[:, None], r)


def test_zero_latent_clamp():
    r = _tokens(4, seed=7)[1]
    codes, sig, rope = O.append_quant(np.zeros((4, 512), np.float32), r)
    assert np.all(codes == 0) and np.all(sig == np.float32(2.0 ** -24))
    assert np.all(np.isfinite(bf16_bits_to_f64(rope)))
    np.testing.assert_array_equal(bf16_bits_to_f64(rope), r * 2.0 ** 24)


def test_q_quant_is_per_row_with_content_only_amax():
    rng = np.random.default_rng(8)
    q = synth.queries(rng, 64).float().numpy()
    qc, sq, qr = O.q_quant(q)
    np.testing.assert_array_equal(sq, np.maximum(np.abs(q[:, :512]).max(1) / np.float32(448), np.float32(2.0 ** -24)).astype(np.float32))
    q2 = q.copy()
    q2[:, 512:] *= 1000   # RoPE part never enters the amax
    q2 = torch.from_numpy(q2).to(torch.bfloat16).float().numpy()
    _, sq2, _ = O.q_quant(q2)
    np.testing.assert_array_equal(sq2, sq)


def test_paging_accounting_and_gather_order():
    rng = np.random.default_rng(9)
    L = 65
    bt, npages = synth.paged_layout(rng, [L], extra_pages=3)
    assert (bt[0] >= 0).all() and len(set(bt[0][:2])) == 2
    pools = dict(kv_fp8=np.zeros((npages, 64, 512), np.uint8),
                 kv_rope=np.zeros((npages, 64, 64), np.uint16),
                 kv_scale=np.zeros((npages, 64), np.float32))
    c, r = _tokens(L, seed=10)
    for t in range(L):     # 65 sequential appends
        O.append_to_pools(pools, c[t:t + 1], r[t:t + 1], bt, np.array([t + 1]))
    used = np.flatnonzero(pools["kv_scale"].reshape(npages, -1).any(axis=1))
    assert len(used) == 2                                 # 65 tokens -> 2 pages
    kc, sk, kr = O.gather_request(pools, bt[0], L)
    codes, sig, rope = O.append_quant(c, r)
    np.testing.assert_array_equal(kc, codes)
    np.testing.assert_array_equal(sk, sig)
    np.testing.assert_array_equal(kr, rope)
