"""Pins for oracle.decode_mx, the NEXT-4(b) MX variant the B200 kernel mla_decode_fp8_mx
implements (not the paper's method, reading R28).  Checked against:
  * O6 (exact attention over the dequantized cache): identity P rounding gives O6 exactly;
  * the E4M3 rounding bound: |decode_mx - O6| within the worst-case relative P error;
  * invariance: shifting every logit of a row by k ln 2 (k integer) leaves o unchanged and
    moves lse by k ln 2 (the codes do not depend on the integer references);
  * the existing p_quant_mx (power-of-two scale per 64 tokens) inside decode_o7 when the row
    maximum is made an integer in log2 units: then both definitions quantize identically;
  * torch SDPA (fp64) for lse with identity rounding."""
import numpy as np
import pytest
import torch

from oracle import snapmla as O
from paper_2602_10718_b200 import synth


def _case(L=700, H=8, seed=0, dist="mla"):
    rng = np.random.default_rng(seed)
    c, r = synth.latent_tokens(rng, L, dist)
    q = synth.queries(rng, H, dist)
    kc, sk, kr = O.append_quant(c.float().numpy(), r.float().numpy())
    qc, sq, qr = O.q_quant(q.float().numpy())
    return qc, sq, qr, kc, sk, kr


@pytest.mark.parametrize("L", [1, 63, 64, 65, 700])
def test_identity_rounding_equals_o6(L):
    qc, sq, qr, kc, sk, kr = _case(L)
    o, lse = O.decode_mx(qc, sq, qr, kc, sk, kr, synth.DEFAULT_SOFTMAX_SCALE, p_quant=False)
    o6, lse6 = O.attn_o6(qc, sq, qr, kc, sk, kr, synth.DEFAULT_SOFTMAX_SCALE)
    assert np.allclose(o, o6, rtol=1e-12, atol=1e-12 * np.abs(o6).max())
    assert np.allclose(lse, lse6, rtol=0, atol=1e-12)


def test_lse_matches_torch_logsumexp():
    qc, sq, qr, kc, sk, kr = _case(333)
    s = O.logits(qc, sq, qr, kc, sk, kr, synth.DEFAULT_SOFTMAX_SCALE)
    _, lse = O.decode_mx(qc, sq, qr, kc, sk, kr, synth.DEFAULT_SOFTMAX_SCALE)
    assert np.allclose(lse, torch.logsumexp(torch.from_numpy(s), dim=1).numpy(), atol=1e-12)


def test_within_e4m3_bound_of_o6():
    """each P' code is within 2^-4 relative of its value (E4M3 RNE, |w / 2^e| in (224, 448]
    for the block max, subnormal floor below): |o - o6| <= 2^-4 * sum_j a_j |V_j| / sum_j a_j
    with a_j the exact (unrounded) weights -- checked loosely as 2^-4 * max |V_deq|."""
    qc, sq, qr, kc, sk, kr = _case(1000, seed=3)
    o, _ = O.decode_mx(qc, sq, qr, kc, sk, kr, synth.DEFAULT_SOFTMAX_SCALE)
    o6, _ = O.attn_o6(qc, sq, qr, kc, sk, kr, synth.DEFAULT_SOFTMAX_SCALE)
    vmax = np.abs(O.decode_e4m3(kc)).max()
    assert np.abs(o - o6).max() <= 2.0 ** -4 * vmax
    assert np.abs(o - o6).max() > 0   # the rounding is really applied


def test_integer_log2_shift_invariance():
    qc, sq, qr, kc, sk, kr = _case(500, seed=5)
    scale = synth.DEFAULT_SOFTMAX_SCALE
    o, lse = O.decode_mx(qc, sq, qr, kc, sk, kr, scale)
    # scaling sigma_q by 2 doubles every logit; instead shift logits by k ln 2 through the
    # closed form directly: add k ln 2 to s by re-running with a wrapped logits function
    orig = O.logits
    try:
        O.logits = lambda *a: orig(*a) + 3 * np.log(2.0)
        o2, lse2 = O.decode_mx(qc, sq, qr, kc, sk, kr, scale)
    finally:
        O.logits = orig
    assert np.allclose(o2, o, rtol=1e-13, atol=1e-13 * np.abs(o).max())
    assert np.allclose(lse2 - lse, 3 * np.log(2.0), atol=1e-12)


def test_equals_p_quant_mx_when_row_max_is_integer_in_log2():
    """decode_o7(p_mx_group=64) quantizes w = exp(s - m) sigma_K; when m log2 e is an integer
    that is w scaled by an exact power of two relative to decode_mx's w, so the codes agree."""
    qc, sq, qr, kc, sk, kr = _case(640, H=4, seed=7)
    scale = synth.DEFAULT_SOFTMAX_SCALE
    orig = O.logits
    s0 = orig(qc, sq, qr, kc, sk, kr, scale)
    m2 = s0.max(axis=1) / np.log(2.0)
    shift = (np.ceil(m2) - m2) * np.log(2.0)          # makes each row's max an integer in log2
    try:
        O.logits = lambda *a: orig(*a) + shift[:, None]
        o_mx, _ = O.decode_mx(qc, sq, qr, kc, sk, kr, scale)
        o_g, _ = O.decode_o7(qc, sq, qr, kc, sk, kr, scale, p_mx_group=64)
    finally:
        O.logits = orig
    assert np.allclose(o_mx, o_g, rtol=1e-10, atol=1e-10 * np.abs(o_g).max())
