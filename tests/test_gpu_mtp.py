"""NEXT-1 parity: multi-token prediction (MTP) through mla_decode_fp8_ex.

q [B, q_len, H, 576]: rows (t, h) share the paged cache; query token t attends
causally to keys 0 .. L - q_len + t (reading R25).  Same gates as
test_gpu_decode (BASELINE north_star tolerance vs the oracle's O7 per token).
"""
import numpy as np
import pytest
import torch

from gpu_cases import Case, parity_stats

pytestmark = pytest.mark.gpu

GATE_MAX, GATE_MEAN, DIAG_MAX, LSE_ABS = 2e-2, 2e-3, 1e-3, 1e-3


def _check_mtp(case):
    cache = case.gpu_cache()
    out32, lse32 = case.gpu_decode(cache, f32_out=True)
    out16, _ = case.gpu_decode(cache)
    pools = case.oracle_pools()
    refs, gots, lref, lgot, empty = [], [], [], [], []
    for b in range(case.B):
        o7, l7 = case.oracle_request_mtp(pools, b)
        vis = np.isfinite(l7)
        empty.append((out32[b][~vis], lse32[b][~vis]))
        refs.append(o7[vis])
        gots.append(out32[b][vis])
        lref.append(l7[vis])
        lgot.append(lse32[b][vis])
    for o, l in empty:   # a query token that sees no key -> o = 0, lse = -inf
        assert np.all(o == 0) and np.all(np.isneginf(l))
    ref, got = np.concatenate(refs), np.concatenate(gots)
    mx, mn = parity_stats(got, ref)
    lerr = float(np.max(np.abs(np.concatenate(lgot) - np.concatenate(lref))))
    rne = torch.from_numpy(out32.astype(np.float32)).to(torch.bfloat16).float().numpy()
    assert np.array_equal(rne, out16), "bf16 output is not RNE(fp32 output)"
    msg = f"f32 max/rms={mx:.2e} mean/rms={mn:.2e} lse={lerr:.2e}"
    print(msg)
    assert mx <= GATE_MAX and mn <= GATE_MEAN and mx <= DIAG_MAX, msg
    assert lerr <= LSE_ABS, msg


@pytest.mark.parametrize("H", [16, 64, 128])
@pytest.mark.parametrize("lens", [[1, 2, 64, 65], [129, 4096 + 1], [148 * 64 * 2 + 1]])
def test_mtp2(H, lens):
    _check_mtp(Case(lens, H, seed=200 + H + len(lens), q_len=2))


@pytest.mark.parametrize("q_len,H", [(3, 16), (4, 64), (2, 96)])
def test_mtp_other_lengths(q_len, H):
    _check_mtp(Case([1, 3, 63, 64, 65, 700], H, seed=300 + q_len, q_len=q_len))


def test_mtp1_ex_equals_plain_decode():
    """mla_decode_fp8_ex with q_len = 1 is mla_decode_fp8 bit for bit."""
    case1 = Case([700, 65, 1], 64, seed=401)
    case2 = Case([700, 65, 1], 64, seed=401)
    case2.q = case1.q[:, None].clone()
    cache = case1.gpu_cache()
    o1, l1 = case1.gpu_decode(cache, f32_out=True)
    o2, l2 = case2.gpu_decode(cache, f32_out=True)
    assert np.array_equal(o1.view(np.uint32), o2[:, 0].view(np.uint32))
    assert np.array_equal(l1, l2[:, 0])
