"""Thin Python binding of libsnapmla.so (ctypes).  Argument marshalling only:
every step of the hot path runs in the library's CUDA kernels.  torch supplies
device memory and the current stream; nothing else of torch is used.

Same names as the C ABI (include/snapmla.h):
  mla_kv_append_quant, mla_decode_workspace_bytes, mla_decode_fp8,
  mla_decode_fp8_ex, mla_combine, mla_combine_f32, mla_kv_fetch_dequant,
  mla_kv_append_bf16, mla_decode_bf16 (NEXT-2: the unquantized BF16 baseline in the same skeleton)
There is no CPU fallback: a missing library or a non-CUDA tensor raises.
"""
import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SNAPMLA_LIB", os.path.join(_HERE, "libsnapmla.so"))   # override: experiments only
_lib = None

D_C, D_R, PAGE = 512, 64, 64

_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_SZ = ctypes.c_size_t
_F = ctypes.c_float


def lib():
    """Load libsnapmla.so (built by __graft_entry__.build()); raise loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                           "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    L.mla_status_str.restype = ctypes.c_char_p
    L.mla_status_str.argtypes = [_I]
    L.mla_abi_version.restype = _I
    L.mla_abi_version.argtypes = []
    L.mla_kv_append_quant.restype = _I
    L.mla_kv_append_quant.argtypes = [_P, _P, _P, _P, _I, _I, _I, _I, _I, _I64, _P, _P, _P, _P]
    L.mla_decode_workspace_bytes.restype = _SZ
    L.mla_decode_workspace_bytes.argtypes = [_I, _I, _I]
    L.mla_decode_fp8.restype = _I
    L.mla_decode_fp8.argtypes = [_P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I64, _F, _P, _SZ, _P]
    L.mla_decode_fp8_ex.restype = _I
    L.mla_decode_fp8_ex.argtypes = [_P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _I64, _F, _P, _SZ, _P]
    L.mla_decode_fp8_mx.restype = _I
    L.mla_decode_fp8_mx.argtypes = [_P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _I64, _F, _P, _SZ, _P]
    L.mla_kv_fetch_dequant.restype = _I
    L.mla_kv_fetch_dequant.argtypes = [_P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I64, _I64, _P, _P, _P]
    L.mla_combine.restype = _I
    L.mla_combine.argtypes = [_P, _I, _I, _I, _P, _P, _P]
    L.mla_combine_f32.restype = _I
    L.mla_combine_f32.argtypes = [_P, _I, _I, _I, _P, _P, _P]
    L.mla_combine_gather.restype = _I
    L.mla_combine_gather.argtypes = [_P, _I, _I, _I, ctypes.POINTER(ctypes.c_void_p), _I, _I, _P, _P]
    L.mla_kv_append_bf16.restype = _I
    L.mla_kv_append_bf16.argtypes = [_P, _P, _P, _P, _I, _I, _I, _I, _I, _I64, _P, _P, _P]
    L.mla_decode_bf16.restype = _I
    L.mla_decode_bf16.argtypes = [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _I64, _F, _P, _SZ, _P]
    _lib = L
    return L


def exported_symbols():
    return ["mla_status_str", "mla_abi_version", "mla_kv_append_quant", "mla_decode_workspace_bytes",
            "mla_decode_fp8", "mla_decode_fp8_ex", "mla_decode_fp8_mx", "mla_combine", "mla_combine_f32", "mla_kv_fetch_dequant",
            "mla_kv_append_bf16", "mla_decode_bf16", "mla_combine_gather"]


def _check(status, what):
    if status != 0:
        raise RuntimeError(f"{what} failed: {lib().mla_status_str(status).decode()}")


def _dev(t, dtype, name):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name}: expected a CUDA tensor (no CPU fallback)")
    if t.dtype != dtype:
        raise TypeError(f"{name}: expected {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def mla_kv_append_quant(c_kv, k_pe, block_table, seq_lens, kv_fp8, kv_rope, kv_scale, stream=None):
    """Quantize-on-append of one token per request into the paged pools (in place)."""
    batch = c_kv.shape[0]
    _check(lib().mla_kv_append_quant(
        _dev(c_kv, torch.bfloat16, "c_kv"), _dev(k_pe, torch.bfloat16, "k_pe"),
        _dev(block_table, torch.int32, "block_table"), _dev(seq_lens, torch.int32, "seq_lens"),
        batch, c_kv.shape[1], k_pe.shape[1], kv_fp8.shape[1], block_table.shape[1], kv_fp8.shape[0],
        _dev(kv_fp8, torch.uint8, "kv_fp8"), _dev(kv_rope, torch.bfloat16, "kv_rope"),
        _dev(kv_scale, torch.float32, "kv_scale"), _stream(stream)), "mla_kv_append_quant")


def mla_decode_workspace_bytes(batch, num_heads, num_sms=0):
    return int(lib().mla_decode_workspace_bytes(batch, num_heads, num_sms))


def mla_decode_fp8(q, kv_fp8, kv_rope, kv_scale, block_table, seq_lens, softmax_scale, workspace, stream=None):
    """Enqueue the FP8 decode; partials land in `workspace` (uint8 CUDA tensor)."""
    batch, num_heads = q.shape[0], q.shape[1]
    _check(lib().mla_decode_fp8(
        _dev(q, torch.bfloat16, "q"), _dev(kv_fp8, torch.uint8, "kv_fp8"),
        _dev(kv_rope, torch.bfloat16, "kv_rope"), _dev(kv_scale, torch.float32, "kv_scale"),
        _dev(block_table, torch.int32, "block_table"), _dev(seq_lens, torch.int32, "seq_lens"),
        batch, num_heads, D_C, D_R, kv_fp8.shape[1], block_table.shape[1], kv_fp8.shape[0],
        float(softmax_scale), _dev(workspace, torch.uint8, "workspace"), workspace.numel(),
        _stream(stream)), "mla_decode_fp8")


def mla_decode_fp8_ex(q, kv_fp8, kv_rope, kv_scale, block_table, seq_lens, softmax_scale, workspace,
                      stream=None):
    """MTP decode: q bf16 [batch, q_len, num_heads, 576]; partials for q_len * num_heads rows."""
    batch, q_len, num_heads = q.shape[0], q.shape[1], q.shape[2]
    _check(lib().mla_decode_fp8_ex(
        _dev(q, torch.bfloat16, "q"), _dev(kv_fp8, torch.uint8, "kv_fp8"),
        _dev(kv_rope, torch.bfloat16, "kv_rope"), _dev(kv_scale, torch.float32, "kv_scale"),
        _dev(block_table, torch.int32, "block_table"), _dev(seq_lens, torch.int32, "seq_lens"),
        batch, num_heads, q_len, D_C, D_R, kv_fp8.shape[1], block_table.shape[1], kv_fp8.shape[0],
        float(softmax_scale), _dev(workspace, torch.uint8, "workspace"), workspace.numel(),
        _stream(stream)), "mla_decode_fp8_ex")


def mla_decode_fp8_mx(q, kv_fp8, kv_rope, kv_scale, block_table, seq_lens, softmax_scale, workspace,
                      stream=None):
    """NEXT-4(b) MX-scaled P variant (not the paper's method): q bf16 [batch, num_heads, 576] or
    [batch, q_len, num_heads, 576], q_len x num_heads <= 128; partials in `workspace` as mla_decode_fp8_ex."""
    batch = q.shape[0]
    q_len, num_heads = (q.shape[1], q.shape[2]) if q.dim() == 4 else (1, q.shape[1])
    _check(lib().mla_decode_fp8_mx(
        _dev(q, torch.bfloat16, "q"), _dev(kv_fp8, torch.uint8, "kv_fp8"),
        _dev(kv_rope, torch.bfloat16, "kv_rope"), _dev(kv_scale, torch.float32, "kv_scale"),
        _dev(block_table, torch.int32, "block_table"), _dev(seq_lens, torch.int32, "seq_lens"),
        batch, num_heads, q_len, D_C, D_R, kv_fp8.shape[1], block_table.shape[1], kv_fp8.shape[0],
        float(softmax_scale), _dev(workspace, torch.uint8, "workspace"), workspace.numel(),
        _stream(stream)), "mla_decode_fp8_mx")


def mla_combine(workspace, batch, num_heads, out, lse=None, stream=None):
    """Merge split partials -> out bf16 [batch, num_heads, 512], lse fp32 [batch, num_heads]."""
    _check(lib().mla_combine(
        _dev(workspace, torch.uint8, "workspace"), batch, num_heads, D_C, _dev(out, torch.bfloat16, "out"),
        None if lse is None else _dev(lse, torch.float32, "lse"), _stream(stream)), "mla_combine")


def mla_combine_gather(workspace, batch, num_heads, out_peers, rank, lse=None, stream=None):
    """NEXT-4(c): combine + fused TP all-gather.  `out_peers`: one entry per rank -- a CUDA
    bf16 tensor [batch, world * num_heads, 512] (local buffers on one GPU) or an int device
    pointer of a peer-mapped buffer of that shape (e.g. symmetric-memory buffer_ptrs)."""
    world = len(out_peers)
    ptrs = (ctypes.c_void_p * world)()
    for i, o in enumerate(out_peers):
        if isinstance(o, torch.Tensor):
            if o.shape != (batch, world * num_heads, D_C):
                raise ValueError(f"out_peers[{i}]: expected [{batch}, {world * num_heads}, {D_C}], got {tuple(o.shape)}")
            ptrs[i] = _dev(o, torch.bfloat16, f"out_peers[{i}]").value
        else:
            ptrs[i] = int(o)
    _check(lib().mla_combine_gather(
        _dev(workspace, torch.uint8, "workspace"), batch, num_heads, D_C, ptrs, world, rank,
        None if lse is None else _dev(lse, torch.float32, "lse"), _stream(stream)), "mla_combine_gather")


def mla_combine_f32(workspace, batch, num_heads, out, lse=None, stream=None):
    _check(lib().mla_combine_f32(
        _dev(workspace, torch.uint8, "workspace"), batch, num_heads, D_C, _dev(out, torch.float32, "out"),
        None if lse is None else _dev(lse, torch.float32, "lse"), _stream(stream)), "mla_combine_f32")


def mla_kv_fetch_dequant(kv_fp8, kv_rope, kv_scale, block_table, tok_start, out_offset, total_rows,
                         c_kv_out=None, k_pe_out=None, stream=None):
    """Fused-Fetch-Dequant: rows of the paged FP8 cache -> BF16 (c_kv [total, 512], k_pe [total, 64])."""
    dev = kv_fp8.device
    if c_kv_out is None:
        c_kv_out = torch.empty(total_rows, D_C, dtype=torch.bfloat16, device=dev)
    if k_pe_out is None:
        k_pe_out = torch.empty(total_rows, D_R, dtype=torch.bfloat16, device=dev)
    _check(lib().mla_kv_fetch_dequant(
        _dev(kv_fp8, torch.uint8, "kv_fp8"), _dev(kv_rope, torch.bfloat16, "kv_rope"),
        _dev(kv_scale, torch.float32, "kv_scale"), _dev(block_table, torch.int32, "block_table"),
        _dev(tok_start, torch.int32, "tok_start"), _dev(out_offset, torch.int32, "out_offset"),
        tok_start.shape[0], D_C, D_R, kv_fp8.shape[1], block_table.shape[1], kv_fp8.shape[0], int(total_rows),
        _dev(c_kv_out, torch.bfloat16, "c_kv_out"), _dev(k_pe_out, torch.bfloat16, "k_pe_out"),
        _stream(stream)), "mla_kv_fetch_dequant")
    return c_kv_out, k_pe_out


def mla_kv_append_bf16(c_kv, k_pe, block_table, seq_lens, kv_c, kv_rope, stream=None):
    """NEXT-2 baseline: copy one token per request into the unquantized BF16 paged pools."""
    batch = c_kv.shape[0]
    _check(lib().mla_kv_append_bf16(
        _dev(c_kv, torch.bfloat16, "c_kv"), _dev(k_pe, torch.bfloat16, "k_pe"),
        _dev(block_table, torch.int32, "block_table"), _dev(seq_lens, torch.int32, "seq_lens"),
        batch, c_kv.shape[1], k_pe.shape[1], kv_c.shape[1], block_table.shape[1], kv_c.shape[0],
        _dev(kv_c, torch.bfloat16, "kv_c"), _dev(kv_rope, torch.bfloat16, "kv_rope"), _stream(stream)),
        "mla_kv_append_bf16")


def mla_decode_bf16(q, kv_c, kv_rope, block_table, seq_lens, softmax_scale, workspace, stream=None):
    """NEXT-2 baseline decode: q bf16 [batch, num_heads, 576] or [batch, q_len, num_heads, 576]."""
    batch = q.shape[0]
    q_len, num_heads = (q.shape[1], q.shape[2]) if q.dim() == 4 else (1, q.shape[1])
    _check(lib().mla_decode_bf16(
        _dev(q, torch.bfloat16, "q"), _dev(kv_c, torch.bfloat16, "kv_c"), _dev(kv_rope, torch.bfloat16, "kv_rope"),
        _dev(block_table, torch.int32, "block_table"), _dev(seq_lens, torch.int32, "seq_lens"),
        batch, num_heads, q_len, D_C, D_R, kv_c.shape[1], block_table.shape[1], kv_c.shape[0],
        float(softmax_scale), _dev(workspace, torch.uint8, "workspace"), workspace.numel(),
        _stream(stream)), "mla_decode_bf16")


class PagedMLACacheBF16:
    """NEXT-2 baseline: unquantized paged cache, kv_c bf16 [P,64,512], kv_rope bf16 [P,64,64] (1152 B / token)."""

    def __init__(self, num_pages, device="cuda"):
        self.num_pages = int(num_pages)
        self.kv_c = torch.zeros(num_pages, PAGE, D_C, dtype=torch.bfloat16, device=device)
        self.kv_rope = torch.zeros(num_pages, PAGE, D_R, dtype=torch.bfloat16, device=device)

    def append(self, c_kv, k_pe, block_table, seq_lens, stream=None):
        mla_kv_append_bf16(c_kv, k_pe, block_table, seq_lens, self.kv_c, self.kv_rope, stream)


class PagedMLACache:
    """Device-resident paged FP8 latent cache (three planes sharing one slot index):
    kv_fp8 u8 [P,64,512] E4M3 codes, kv_rope bf16 [P,64,64] = k_pe/sigma, kv_scale f32 [P,64].
    Zero-initialised (stale bytes must never be FP8 NaN codes)."""

    def __init__(self, num_pages, device="cuda"):
        self.num_pages = int(num_pages)
        self.kv_fp8 = torch.zeros(num_pages, PAGE, D_C, dtype=torch.uint8, device=device)
        self.kv_rope = torch.zeros(num_pages, PAGE, D_R, dtype=torch.bfloat16, device=device)
        self.kv_scale = torch.zeros(num_pages, PAGE, dtype=torch.float32, device=device)

    def append(self, c_kv, k_pe, block_table, seq_lens, stream=None):
        mla_kv_append_quant(c_kv, k_pe, block_table, seq_lens, self.kv_fp8, self.kv_rope, self.kv_scale, stream)


def decode_step(q, cache, block_table, seq_lens, softmax_scale, workspace=None, out=None, lse=None,
                stream=None, f32_out=False, mx=False):
    """mla_decode_fp8 (q [B, H, 576]) or mla_decode_fp8_ex (q [B, q_len, H, 576], MTP) + mla_combine;
    mla_decode_bf16 when `cache` is a PagedMLACacheBF16 (NEXT-2 baseline); mla_decode_fp8_mx with
    mx=True (NEXT-4(b) variant).
    Returns (out, lse) shaped like q's leading dims."""
    lead = tuple(q.shape[:-1])
    batch, rows = q.shape[0], 1
    for d in lead[1:]:
        rows *= d
    if workspace is None:
        workspace = torch.empty(mla_decode_workspace_bytes(batch, rows), dtype=torch.uint8, device=q.device)
    if out is None:
        out = torch.empty(lead + (D_C,), dtype=torch.float32 if f32_out else torch.bfloat16, device=q.device)
    if lse is None:
        lse = torch.empty(lead, dtype=torch.float32, device=q.device)
    if mx:
        mla_decode_fp8_mx(q, cache.kv_fp8, cache.kv_rope, cache.kv_scale, block_table, seq_lens, softmax_scale,
                          workspace, stream)
    elif isinstance(cache, PagedMLACacheBF16):
        mla_decode_bf16(q, cache.kv_c, cache.kv_rope, block_table, seq_lens, softmax_scale, workspace, stream)
    elif q.dim() == 4:
        mla_decode_fp8_ex(q, cache.kv_fp8, cache.kv_rope, cache.kv_scale, block_table, seq_lens, softmax_scale,
                          workspace, stream)
    else:
        mla_decode_fp8(q, cache.kv_fp8, cache.kv_rope, cache.kv_scale, block_table, seq_lens, softmax_scale,
                       workspace, stream)
    (mla_combine_f32 if f32_out else mla_combine)(workspace, batch, rows, out, lse, stream)
    return out, lse
