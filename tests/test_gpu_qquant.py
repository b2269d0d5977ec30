"""a2 parity: the Fused-Q-Quant results the plan launch writes into the decode workspace (E4M3 codes,
sigma_q, q_r' = q_r / sigma_q in BF16) against oracle.snapmla.q_quant, bit for bit, for
every query row -- including MTP rows, padded head counts and the three decode kernels' row ranges.
The workspace layout mirrors csrc/snapmla_internal.h (ws_layout)."""
import numpy as np
import pytest
import torch

from gpu_cases import Case
from oracle import snapmla as O
from paper_2602_10718_b200 import ops

pytestmark = pytest.mark.gpu


def _align(x, a):
    return (x + a - 1) // a * a


def _q_regions(batch, rows, sms):
    """(offset of codes, offset of q_r', offset of sigma_q) in the workspace (snapmla_internal.h)."""
    n_ht = (rows + 63) // 64
    groups = sms // n_ht
    slots = batch + groups
    cum = 16 * 4
    first = _align(cum + (batch + 1) * 4, 16)
    lse = _align(first + (groups + 1) * 4, 256)
    o = _align(lse + slots * n_ht * 64 * 4, 256)
    qc = _align(o + slots * n_ht * 64 * 512 * 4, 256)
    qr = _align(qc + batch * rows * 512, 256)
    sq = _align(qr + batch * rows * 64 * 2, 256)
    return qc, qr, sq


@pytest.mark.parametrize("lens,H,q_len", [([300, 65, 1], 16, 1), ([4096, 0, 777], 128, 1), ([129, 2000], 64, 1),
                                         ([1, 5000], 8, 2), ([70, 64], 100, 1), ([33], 1, 1)])
def test_plan_q_quant_bit_exact(lens, H, q_len):
    case = Case(lens, H, seed=700 + H + q_len, q_len=q_len)
    cache = case.gpu_cache()
    rows = H * q_len
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    ws = torch.zeros(ops.mla_decode_workspace_bytes(case.B, rows), dtype=torch.uint8, device="cuda")
    case.gpu_decode(cache, workspace=ws)
    qc_off, qr_off, sq_off = _q_regions(case.B, rows, sms)
    n = case.B * rows
    w = ws.cpu().numpy()
    codes = w[qc_off:qc_off + n * 512].reshape(n, 512)
    rope = w[qr_off:qr_off + n * 128].view(np.uint16).reshape(n, 64)
    sigma = w[sq_off:sq_off + n * 4].view(np.float32)
    qf = case.q.float().numpy().reshape(n, 576)   # row = b * rows + t * H + h, the kernels' order
    c_ref, s_ref, r_ref = O.q_quant(qf)
    assert np.array_equal(sigma.view(np.uint32), s_ref.astype(np.float32).view(np.uint32)), "sigma_q"
    assert np.array_equal(codes, c_ref), f"codes: {int((codes != c_ref).sum())} of {codes.size} differ"
    assert np.array_equal(rope, r_ref), f"q_r': {int((rope != r_ref).sum())} of {rope.size} differ"
