"""NEXT-2 baseline parity: the unquantized BF16 decode (mla_kv_append_bf16 + mla_decode_bf16 +
combine, the same kernel skeleton as the FP8 path) vs the oracle's O8 = fp64 absorbed-MLA
attention over the unquantized BF16 inputs (oracle.snapmla.attn_o8, pinned in
test_oracle_decode.py).  The kernel rounds the softmax weights p to BF16 for the PV product
(relative 2^-9 per weight, reading R27), so the gate is the decode gate of
test_gpu_decode.py (max-abs <= 2e-2 RMS, mean-abs <= 2e-3 RMS on the fp32 result) plus an
element-wise bound that follows from that rounding alone: with p~_j = p_j (1 + d_j),
|d_j| <= 2^-9, |o~_d - o_d| = |sum_j p_j d_j c_jd| / l <= 2^-9 max_j |c_jd| (plus 1e-4 RMS
for fp32 accumulation).  The append is a copy: bit-exact."""
import numpy as np
import pytest
import torch

from gpu_cases import PAGE, Case, parity_stats
from oracle import snapmla as O
from paper_2602_10718_b200 import ops

pytestmark = pytest.mark.gpu

GATE_MAX, GATE_MEAN, LSE_ABS = 2e-2, 2e-3, 1e-3


def bf16_cache(case):
    cache = ops.PagedMLACacheBF16(case.num_pages, "cuda")
    if len(case.tok_pos):
        bt_v = torch.from_numpy(case.tok_page.astype(np.int32)[:, None]).cuda()
        sl_v = torch.from_numpy((case.tok_pos % PAGE + 1).astype(np.int32)).cuda()
        cache.append(case.c_kv.cuda(), case.k_pe.cuda(), bt_v, sl_v)
    torch.cuda.synchronize()
    return cache


def decode(case, cache, f32_out):
    bt = torch.from_numpy(case.bt).cuda()
    sl = torch.from_numpy(case.lens.astype(np.int32)).cuda()
    out, lse = ops.decode_step(case.q.cuda(), cache, bt, sl, case.scale, f32_out=f32_out)
    torch.cuda.synchronize()
    return out.float().cpu().numpy(), lse.cpu().numpy()


def check(case):
    cache = bf16_cache(case)
    out32, lse32 = decode(case, cache, True)
    out16, _ = decode(case, cache, False)
    rne = torch.from_numpy(out32.astype(np.float32)).to(torch.bfloat16).float().numpy()
    assert np.array_equal(rne, out16), "bf16 output is not RNE(fp32 output)"
    refs, gots, lref, lgot, bounds = [], [], [], [], []
    off = np.concatenate([[0], np.cumsum(case.lens)])
    for b in range(case.B):
        L = int(case.lens[b])
        c, r = case.c_kv[off[b]:off[b + 1]].float().numpy(), case.k_pe[off[b]:off[b + 1]].float().numpy()
        if case.q_len == 1:
            if L == 0:
                assert np.all(out32[b] == 0) and np.all(np.isneginf(lse32[b]))
                continue
            o8, l8 = O.attn_o8(case.q[b].float().numpy(), c, r, case.scale)
            refs.append(o8), gots.append(out32[b]), lref.append(l8), lgot.append(lse32[b])
            bounds.append(np.broadcast_to(2.0 ** -9 * np.abs(c).max(axis=0), o8.shape))
        else:
            o8, l8 = O.attn_o8_mtp(case.q[b].float().numpy(), c, r, case.scale)
            vis = np.isfinite(l8)
            assert np.all(out32[b][~vis] == 0) and np.all(np.isneginf(lse32[b][~vis]))
            refs.append(o8[vis]), gots.append(out32[b][vis]), lref.append(l8[vis]), lgot.append(lse32[b][vis])
            bounds.append(np.broadcast_to(2.0 ** -9 * np.abs(c).max(axis=0), o8[vis].shape))
    got, ref = np.concatenate(gots), np.concatenate(refs)
    mx, mn = parity_stats(got, ref)
    rms = float(np.sqrt(np.mean(ref ** 2)))
    excess = float((np.abs(got - ref) - np.concatenate(bounds) - 1e-4 * rms).max())
    lerr = float(np.max(np.abs(np.concatenate(lgot) - np.concatenate(lref))))
    msg = f"bf16 decode vs O8: max/rms={mx:.2e} mean/rms={mn:.2e} lse={lerr:.2e} bound excess={excess:.2e}"
    print(msg)
    assert mx <= GATE_MAX and mn <= GATE_MEAN and excess <= 0, msg
    assert lerr <= LSE_ABS, msg


def test_append_bf16_is_a_copy():
    case = Case([1, 63, 64, 65, 300], 16, seed=501)
    cache = bf16_cache(case)
    slots = case.tok_page.astype(np.int64) * PAGE + case.tok_pos % PAGE
    got_c = cache.kv_c.view(-1, 512)[torch.from_numpy(slots).cuda()].cpu()
    got_r = cache.kv_rope.view(-1, 64)[torch.from_numpy(slots).cuda()].cpu()
    assert torch.equal(got_c.view(torch.int16), case.c_kv.view(torch.int16))
    assert torch.equal(got_r.view(torch.int16), case.k_pe.view(torch.int16))


def test_bf16_tiny():
    check(Case([256], 16, seed=502))


@pytest.mark.parametrize("L", [1, 2, 63, 64, 65, 129, 4096 + 17])
def test_bf16_seq_len_sweep(L):
    check(Case([L], 16, seed=503 + L))


@pytest.mark.parametrize("H", [16, 32, 64, 128, 96])
def test_bf16_head_counts(H):
    check(Case([700, 65, 1], H, seed=504 + H))


@pytest.mark.parametrize("dist", ["mla", "iid"])
def test_bf16_many_requests(dist):
    rng = np.random.default_rng(505)
    check(Case(rng.integers(0, 2000, 23), 64, seed=506, dist=dist))


def test_bf16_splits_single_long_request():
    check(Case([148 * 64 * 2 + 5], 64, seed=507))


@pytest.mark.parametrize("q_len,H", [(2, 16), (2, 64)])
def test_bf16_mtp(q_len, H):
    check(Case([1, 2, 64, 65, 700], H, seed=508 + H, q_len=q_len))
