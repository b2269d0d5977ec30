"""CPU-side checks of the C ABI: the library builds for sm_100a, loads without
a GPU, exports every symbol include/snapmla.h declares, and its host-side
argument validation returns the documented status codes before touching CUDA.
"""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "snapmla.h")


@pytest.fixture(scope="module")
def L():
    from paper_2602_10718_b200 import build, ops
    build.build()
    return ops.lib()


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mla_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_three_calls():
    d = _declared()
    for name in ("mla_kv_append_quant", "mla_decode_fp8", "mla_combine", "mla_decode_workspace_bytes"):
        assert name in d


def test_every_declared_symbol_is_exported(L):
    from paper_2602_10718_b200 import ops
    out = subprocess.run(["nm", "-D", "--defined-only", ops.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (mla_[a-z0-9_]+)", out))
    for name in _declared():
        assert name in exported, name
        assert hasattr(L, name)
    assert sorted(ops.exported_symbols()) == _declared()


def test_debug_header_symbols_exported(L):
    """include/snapmla_debug.h (trace, kernel override, read-stream measurement) is exported too."""
    from paper_2602_10718_b200 import ops
    src = re.sub(r"/\*.*?\*/", "", open(os.path.join(ROOT, "include", "snapmla_debug.h")).read(), flags=re.S)
    names = sorted(set(re.findall(r"\b(mla_[a-z0-9_]+)\s*\(", src)))
    assert names == ["mla_debug_cvt_e4m3", "mla_debug_set_pair", "mla_debug_set_small", "mla_debug_set_trace",
                     "mla_measure_read_stream"]
    out = subprocess.run(["nm", "-D", "--defined-only", ops.LIB_PATH], capture_output=True, text=True).stdout
    for name in names:
        assert re.search(r"\bT " + name + r"\b", out), name


def test_read_stream_argument_checks(L):
    f = L.mla_measure_read_stream
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    assert f(None, 1024, 4096, 16, None) == 1                 # NULL buffer
    assert f(4096, 1000, 4096, 16, None) == 2                 # bytes not a multiple of 16
    assert f(4104, 1024, 4096, 16, None) == 4                 # misaligned buffer


def test_sass_is_sm100a_tcgen05_tma(L):
    from paper_2602_10718_b200 import ops
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", ops.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "sm_100a" in sass
    for mnem in ("UTCQMMA", "UTCHMMA", "UTMALDG", "LDTM", "UTCBAR"):
        assert mnem in sass, mnem


def test_status_strings_and_version(L):
    assert L.mla_abi_version() == 1
    names = [L.mla_status_str(i).decode() for i in range(7)]
    assert names == ["MLA_OK", "MLA_ERR_NULL", "MLA_ERR_SHAPE", "MLA_ERR_UNSUPPORTED", "MLA_ERR_ALIGN",
                     "MLA_ERR_WORKSPACE", "MLA_ERR_CUDA"]


def test_host_validation_without_gpu(L):
    P = ctypes.c_void_p
    fake = P(4096)
    # unsupported dims -> 3 before any CUDA call
    assert L.mla_kv_append_quant(fake, fake, fake, fake, 4, 256, 64, 64, 1, 8, fake, fake, fake, None) == 3
    assert L.mla_kv_append_quant(fake, fake, fake, fake, 4, 512, 64, 32, 1, 8, fake, fake, fake, None) == 3
    # NULL pointer -> 1
    assert L.mla_kv_append_quant(None, fake, fake, fake, 4, 512, 64, 64, 1, 8, fake, fake, fake, None) == 1
    # negative batch -> 2 ; empty batch -> OK without touching anything
    assert L.mla_kv_append_quant(fake, fake, fake, fake, -1, 512, 64, 64, 1, 8, fake, fake, fake, None) == 2
    assert L.mla_kv_append_quant(None, None, None, None, 0, 512, 64, 64, 1, 8, None, None, None, None) == 0
    # misaligned -> 4
    assert L.mla_kv_append_quant(P(4097), fake, fake, fake, 4, 512, 64, 64, 1, 8, fake, fake, fake, None) == 4
    # decode: >128 heads unsupported, missing workspace
    assert L.mla_decode_fp8(fake, fake, fake, fake, fake, fake, 2, 256, 512, 64, 64, 4, 8, 0.1, fake, 1 << 20,
                            None) == 3
    assert L.mla_decode_fp8(fake, fake, fake, fake, fake, fake, 2, 16, 512, 64, 64, 4, 8, 0.1, None, 0,
                            None) == 5
    assert L.mla_combine(fake, 2, 16, 256, fake, None, None) == 3
    # NEXT-2 BF16 baseline: same host checks
    assert L.mla_kv_append_bf16(fake, fake, fake, fake, 4, 256, 64, 64, 1, 8, fake, fake, None) == 3
    assert L.mla_kv_append_bf16(fake, None, fake, fake, 4, 512, 64, 64, 1, 8, fake, fake, None) == 1
    assert L.mla_kv_append_bf16(fake, fake, fake, fake, 4, 512, 64, 64, 1, 8, P(4104), fake, None) == 4
    assert L.mla_decode_bf16(fake, fake, fake, fake, fake, 2, 16, 1, 512, 64, 32, 4, 8, 0.1, fake, 1 << 20,
                             None) == 3
    assert L.mla_decode_bf16(fake, fake, fake, fake, fake, 2, 16, 1, 512, 64, 64, 4, 8, 0.1, None, 0, None) == 5
    assert L.mla_decode_bf16(fake, None, fake, fake, fake, 2, 16, 1, 512, 64, 64, 4, 8, 0.1, fake, 1 << 30,
                             None) == 1
    # NEXT-4(c) fused gather: > 8 peers unsupported, rank outside the world, NULL peer
    peers = (P * 9)(*([4096] * 9))
    assert L.mla_combine_gather(fake, 2, 16, 512, peers, 9, 0, None, None) == 3
    assert L.mla_combine_gather(fake, 2, 16, 512, peers, 2, 2, None, None) == 2
    assert L.mla_combine_gather(fake, 2, 16, 512, (P * 2)(4096, None), 2, 0, None, None) == 1


def test_workspace_size_formula(L):
    # explicit SM count: no device query needed
    n1 = L.mla_decode_workspace_bytes(64, 128, 148)
    n2 = L.mla_decode_workspace_bytes(64, 64, 148)
    # slots = batch + groups; partials = slots * n_ht * 64 rows * 512 fp32
    assert n1 >= (64 + 74) * 2 * 64 * 512 * 4
    assert n2 >= (64 + 148) * 1 * 64 * 512 * 4
    # plus the plan's Fused-Q-Quant output per query row: 512 E4M3 codes + 64 BF16 q_r' + fp32 sigma_q
    assert n1 >= (64 + 74) * 2 * 64 * 512 * 4 + 64 * 128 * (512 + 128 + 4)
    assert n2 >= (64 + 148) * 1 * 64 * 512 * 4 + 64 * 64 * (512 + 128 + 4)
    grow = L.mla_decode_workspace_bytes(65, 16, 148) - L.mla_decode_workspace_bytes(64, 16, 148)
    assert grow >= 64 * 512 * 4 + 16 * (512 + 128 + 4) - 3 * 256   # one more slot of partials + 16 rows (alignment slack)
    assert L.mla_decode_workspace_bytes(-1, 16, 148) == 0
