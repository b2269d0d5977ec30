"""Both kernels for 64 < rows <= 128, forced through include/snapmla_debug.h
mla_debug_set_pair: the single-CTA kernel and the block-pair 2-SM kernel
(§7.9, the default from 16K blocks of work), each through the same cases.  Same O7
gate as test_gpu_decode.py; the pair kernel must also agree bit for bit with itself
across runs.  The switch is process-global, so every test restores the default."""
import numpy as np
import pytest

from gpu_cases import Case
from paper_2602_10718_b200 import ops
from test_gpu_decode import _check
from test_gpu_mtp import _check_mtp

pytestmark = pytest.mark.gpu


@pytest.fixture(params=[0, 1], ids=["single", "bp"])
def pair_kernel(request):
    """0: single-CTA kernel (§7.3), 1: block-pair 2-SM kernel (§7.9); -1 (automatic) restored after."""
    L = ops.lib()
    L.mla_debug_set_pair(request.param)
    yield request.param
    L.mla_debug_set_pair(-1)


# unit shapes: single blocks (per = 1), odd units (pair + lone block: [148*64+3, 5]),
# many-block units, ragged tails, empty requests
@pytest.mark.parametrize("lens", [[1], [2, 63], [64, 65, 127, 128, 129], [4096 + 17], [0, 300, 0, 7],
                                  [148 * 64 + 3, 5], [40000, 9000, 1]])
@pytest.mark.parametrize("H", [128, 96, 65])
def test_pair_two_head_tiles(pair_kernel, H, lens):
    heads = np.unique(np.array([0, 1, 31, 32, 63, 64, 95, H - 1]) % H)
    _check(Case(lens, H, seed=300 + H + len(lens)), heads_per_req=heads)


def test_pair_many_requests_all_heads(pair_kernel):
    rng = np.random.default_rng(31)
    _check(Case(rng.integers(0, 3000, 37), 128, seed=32))


def test_pair_deterministic(pair_kernel):
    case = Case([5000, 65, 1], 128, seed=33)
    cache = case.gpu_cache()
    o1, _ = case.gpu_decode(cache, f32_out=True)
    o2, _ = case.gpu_decode(cache, f32_out=True)
    assert np.array_equal(o1.view(np.uint32), o2.view(np.uint32))


@pytest.mark.parametrize("q_len,H", [(2, 64), (2, 48)])
def test_pair_mtp(pair_kernel, q_len, H):
    _check_mtp(Case([1, 2, 64, 65, 129, 4096 + 1], H, seed=340 + H, q_len=q_len))
