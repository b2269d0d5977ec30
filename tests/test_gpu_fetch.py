"""NEXT-3 parity: Fused-Fetch-Dequant on the GPU is bit-exact vs the oracle
(reading R26), over token ranges that cross pages, start mid-page, are empty,
or cover whole requests."""
import numpy as np
import pytest
import torch

from gpu_cases import Case
from oracle import snapmla as O
from paper_2602_10718_b200 import ops

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [0, 1])
def test_fetch_dequant_bit_exact(seed):
    rng = np.random.default_rng(500 + seed)
    lens = [1, 63, 64, 65, 300, 2000, 0, 4096 + 5]
    case = Case(lens, 16, seed=600 + seed)
    cache = case.gpu_cache()
    starts, counts = [], []
    for L in lens:
        s = int(rng.integers(0, L)) if L > 0 else 0
        n = int(rng.integers(0, L - s + 1)) if L > 0 else 0
        starts.append(s)
        counts.append(n)
    counts[-1] = lens[-1] - starts[-1]            # one range runs to the end of its request
    offs = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int32)
    total = int(np.sum(counts))
    dev = "cuda"
    c_out, r_out = ops.mla_kv_fetch_dequant(
        cache.kv_fp8, cache.kv_rope, cache.kv_scale, torch.from_numpy(case.bt).to(dev),
        torch.tensor(starts, dtype=torch.int32, device=dev), torch.from_numpy(offs).to(dev), total)
    torch.cuda.synchronize()
    c_got = c_out.view(torch.int16).cpu().numpy().view(np.uint16)
    r_got = r_out.view(torch.int16).cpu().numpy().view(np.uint16)
    pools = case.oracle_pools()
    for b, (s, n) in enumerate(zip(starts, counts)):
        if n == 0:
            continue
        cb, rb = O.fetch_dequant(pools, case.bt[b], s, n)
        np.testing.assert_array_equal(c_got[offs[b]:offs[b] + n], cb)
        np.testing.assert_array_equal(r_got[offs[b]:offs[b] + n], rb)


def test_fetch_after_append_is_dequantized_append():
    """SPEC invariant: fetch(append(x)) = dequantize(quantize(x)), on the GPU path."""
    case = Case([129], 16, seed=610)
    cache = case.gpu_cache()
    dev = "cuda"
    c_out, r_out = ops.mla_kv_fetch_dequant(cache.kv_fp8, cache.kv_rope, cache.kv_scale,
                                            torch.from_numpy(case.bt).to(dev),
                                            torch.zeros(1, dtype=torch.int32, device=dev),
                                            torch.zeros(1, dtype=torch.int32, device=dev), 129)
    codes, sig, rope = O.append_quant(case.c_kv.float().numpy(), case.k_pe.float().numpy())
    c_ref = O.bf16_rne_bits(O.decode_e4m3(codes).astype(np.float32) * sig[:, None])
    r_ref = O.bf16_rne_bits(O.bf16_bits_to_f64(rope).astype(np.float32) * sig[:, None])
    np.testing.assert_array_equal(c_out.view(torch.int16).cpu().numpy().view(np.uint16), c_ref)
    np.testing.assert_array_equal(r_out.view(torch.int16).cpu().numpy().view(np.uint16), r_ref)
