"""Both kernels for rows <= 32 (q_len x heads), forced through include/snapmla_debug.h
mla_debug_set_small: the single-CTA kernel with the heads padded to M = 64 and the
swapped-operand kernel (heads on the MMA N dimension, §7.11; the default for rows <= 16), each through the same
cases: N = 16 and N = 32 tiles, padded head counts, ragged tails,
empty requests, single-block and many-block units, causal MTP.  Same O7 gate as
test_gpu_decode.py; the swapped kernel must also agree bit for bit with itself across runs and
stay within the gate of the padded kernel's result."""
import numpy as np
import pytest

from gpu_cases import Case, parity_stats
from paper_2602_10718_b200 import ops
from test_gpu_decode import _check
from test_gpu_mtp import _check_mtp

pytestmark = pytest.mark.gpu


@pytest.fixture(params=[0, 1], ids=["single", "swapped"])
def small_kernel(request):
    """0: single-CTA kernel (§7.3), 1: swapped-operand kernel (§7.11); the default (-1) restored after."""
    L = ops.lib()
    L.mla_debug_set_small(request.param)
    yield request.param
    L.mla_debug_set_small(-1)


# block counts: one block, ragged tails, empty requests, units split across CTAs, long units
@pytest.mark.parametrize("lens", [[1], [2, 63], [64, 65, 127, 128, 129], [0, 300, 0, 7], [148 * 64 + 3, 5],
                                  [40000, 9000, 1]])
@pytest.mark.parametrize("H", [1, 8, 16, 17, 24, 32])
def test_small_heads(small_kernel, H, lens):
    _check(Case(lens, H, seed=500 + H + len(lens)))


def test_small_many_requests(small_kernel):
    rng = np.random.default_rng(51)
    _check(Case(rng.integers(0, 3000, 37), 16, seed=52))


@pytest.mark.parametrize("q_len,H", [(2, 16), (2, 8), (4, 8), (3, 5)])
def test_small_mtp(small_kernel, q_len, H):
    _check_mtp(Case([1, 2, 64, 65, 129, 4096 + 1], H, seed=540 + 7 * q_len + H, q_len=q_len))


@pytest.mark.parametrize("H", [16, 32])
def test_swapped_deterministic_and_close_to_padded(H):
    """Bitwise reproducible, and within the north_star gate of the padded kernel (both implement O7)."""
    L = ops.lib()
    case = Case([5000, 65, 1, 9000], H, seed=560 + H)
    cache = case.gpu_cache()
    try:
        L.mla_debug_set_small(1)
        a1, _ = case.gpu_decode(cache, f32_out=True)
        a2, _ = case.gpu_decode(cache, f32_out=True)
        L.mla_debug_set_small(0)
        b, _ = case.gpu_decode(cache, f32_out=True)
    finally:
        L.mla_debug_set_small(-1)
    assert np.array_equal(a1.view(np.uint32), a2.view(np.uint32))
    mx, mn = parity_stats(a1.reshape(-1, 512), b.reshape(-1, 512))
    assert mx <= 2e-2 and mn <= 2e-3, (mx, mn)
