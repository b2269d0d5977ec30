"""SnapMLA hot path, plain CPU oracle (TEST INFRASTRUCTURE ONLY).

Follows PAPER.md (arXiv 2602.10718) step by step; ``P:n`` = PAPER.md line n.
Readings of silent / garbled passages (R1..R22) are listed in DESIGN.md §3.

Shapes (BASELINE.json north_star): kv_lora_rank d_c = 512, rope d_r = 64,
page = 64 tokens, P block B_c = 64 tokens, E4M3 max 448.

Conventions
  * BF16 tensors are passed as float32 arrays whose values lie on the BF16 grid
    (or as uint16 bit patterns where the name ends in ``_bits``).
  * Scales are float32 (north_star: "one fp32 scale per token").
  * All attention arithmetic is float64.

Pin status: every function here is pinned in tests/test_oracle_*.py against
closed forms, special cases, an independent library (torch SDPA in fp64,
torch.float8_e4m3fn / bfloat16 casts) or brute force; none is "parity unpinned".
"""
import numpy as np

from .codec import (E4M3_MAX, bf16_bits_to_f64, bf16_rne_bits, decode_e4m3,
                    encode_e4m3)

D_C = 512          # kv_lora_rank (BASELINE.json north_star)
D_R = 64           # rope dim
PAGE = 64          # tokens per page
B_C = 64           # P-quant / key block size, "BlockN = 64", "B_c = 64"
SIGMA_MIN = np.float32(2.0 ** -24)   # reading R2: zero / tiny amax clamp

_F448 = np.float32(E4M3_MAX)


def _check_bf16_grid(x, name):
    x = np.asarray(x, dtype=np.float32)
    if not np.array_equal(bf16_bits_to_f64(bf16_rne_bits(x)).astype(np.float32), x):
        raise ValueError(f"{name}: values must lie on the BF16 grid")
    return x


# --------------------------------------------------------------------------
# a1 / a2: RoPE-aware per-token quantization (Eq.6 P:208-210,
# Eq.9, Alg.1 requirements P:672-675)
# --------------------------------------------------------------------------
def per_token_quant(content, rope):
    """Quantize rows of ``content`` (FP8 E4M3, one fp32 scale per row) and
    pre-scale ``rope`` into the content quantization domain (Eq.6).

      sigma   = max(fp32(amax(|content_row|) / 448), 2^-24)   readings R1, R2
      codes   = E4M3_RNE_SAT(fp32(content / sigma))            Eq.9, R3, R4
      rope'   = BF16_RNE(fp32(rope / sigma))                   Eq.6, R5

    Only the content part enters the amax: "applies FP8 quantization
    exclusively to the content components, while retaining the RoPE components
    in BF16".  Returns (codes u8 [N,512], sigma f32 [N], rope' u16 [N,64]).
    """
    c = _check_bf16_grid(content, "content")
    r = _check_bf16_grid(rope, "rope")
    amax = np.max(np.abs(c), axis=-1)                       # exact in fp32
    sigma = (amax / _F448).astype(np.float32)               # IEEE fp32 division
    sigma = np.maximum(sigma, SIGMA_MIN).astype(np.float32)
    codes = encode_e4m3((c / sigma[..., None]).astype(np.float32))
    rope_bits = bf16_rne_bits((r / sigma[..., None]).astype(np.float32))
    return codes, sigma, rope_bits


def append_quant(c_kv, k_pe):
    """Fused-K-Append arithmetic: per new token, c_kv [N,512] and
    k_pe [N,64] (BF16 values) -> (kv codes, sigma_K, k_pe / sigma_K in BF16)."""
    return per_token_quant(c_kv, k_pe)


def q_quant(q):
    """Fused-Q-Quant arithmetic: q [R,576] = [absorbed q_nope
    (512) | q_pe (64)] per (token, head) row -> (codes, sigma_q, q_r / sigma_q).
    sigma_q is per row (reading R7: P:692 uses the outer product sigma_q sigma_K^T)."""
    q = np.asarray(q, dtype=np.float32)
    return per_token_quant(q[..., :D_C], q[..., D_C:])


def slot_of(block_table_row, pos):
    """Paged slot of token position ``pos`` (PagedAttention-style):
    page id = block_table[pos // 64], slot = page * 64 + pos % 64."""
    return int(block_table_row[pos // PAGE]) * PAGE + pos % PAGE


def append_to_pools(pools, c_kv, k_pe, block_table, seq_lens):
    """Write one new token per request at position seq_lens[b]-1 (post-append
    length) into the paged pools, in place.

    pools = dict(kv_fp8 u8 [P,64,512], kv_rope u16 [P,64,64], kv_scale f32 [P,64]).
    """
    codes, sigma, rope_bits = append_quant(c_kv, k_pe)
    kf = pools["kv_fp8"].reshape(-1, D_C)
    kr = pools["kv_rope"].reshape(-1, D_R)
    ks = pools["kv_scale"].reshape(-1)
    for b in range(len(seq_lens)):
        s = slot_of(block_table[b], int(seq_lens[b]) - 1)
        kf[s] = codes[b]
        kr[s] = rope_bits[b]
        ks[s] = sigma[b]


def gather_request(pools, block_table_row, L):
    """Read tokens 0..L-1 of one request from the paged pools, in order."""
    slots = np.array([slot_of(block_table_row, j) for j in range(L)], dtype=np.int64)
    kc = pools["kv_fp8"].reshape(-1, D_C)[slots]
    kr = pools["kv_rope"].reshape(-1, D_R)[slots]
    sk = pools["kv_scale"].reshape(-1)[slots]
    return kc, sk, kr


# --------------------------------------------------------------------------
# Dequantized operands and logits (Eq.5, Eq.6)
# --------------------------------------------------------------------------
def _deq_rows(codes, sigma, rope_bits):
    """[dec(codes), bf16val(rope')] * sigma  (576-wide, fp64).  Because rope'
    was pre-divided by sigma (Eq.6), multiplying the whole row by sigma puts
    content and RoPE back in one domain."""
    x = np.concatenate([decode_e4m3(codes), bf16_bits_to_f64(rope_bits)], axis=-1)
    return x * np.asarray(sigma, dtype=np.float64)[..., None]


def logits(qc, sq, qr_bits, kc, sk, kr_bits, softmax_scale):
    """s[r,j] = softmax_scale * <q_deq[r], k_deq[j]>  (absorbed-mode score, Eq.5,
    with Alg.1 step 3's descale by sigma_q sigma_K^T).  Reading R8: the
    caller's softmax_scale multiplies the dequantized logit (Alg.1 omits it)."""
    q_deq = _deq_rows(qc, sq, qr_bits)
    k_deq = _deq_rows(kc, sk, kr_bits)
    return float(softmax_scale) * (q_deq @ k_deq.T)


# --------------------------------------------------------------------------
# O7: closed form of the SnapMLA decode (the parity gate)
# --------------------------------------------------------------------------
def p_quant_mx(w, group):
    """NEXT-4(b) variant (NOT the paper's method): MX-style power-of-two P scales, one per
    (row, `group` tokens) as a UE8M0 shared exponent (OCP MX format, the operand format of
    B200's kind::mxf8f6f4.block_scale).  The paper quantizes with sigma_p = M/448 per 64-token
    block; here sigma_g = 2^ceil(log2(M_g / 448)), so M_g / sigma_g lies in (224, 448]
    and one bit of headroom is lost at worst.  Returns A = sigma_g * dec(E4M3(w / sigma_g))
    (0 for a group whose max is 0)."""
    w = np.asarray(w, dtype=np.float64)
    A = np.zeros_like(w)
    for start in range(0, w.shape[1], group):
        sl = slice(start, min(start + group, w.shape[1]))
        wb = w[:, sl]
        M = wb.max(axis=1)
        e = np.ceil(np.log2(np.where(M > 0, M, 1.0) / E4M3_MAX))
        sig = np.ldexp(1.0, e.astype(np.int64))
        pd = decode_e4m3(encode_e4m3((wb / sig[:, None]).astype(np.float32)))
        pd[M == 0] = 0.0
        A[:, sl] = sig[:, None] * pd
    return A


def decode_o7(qc, sq, qr_bits, kc, sk, kr_bits, softmax_scale,
              block=B_C, p_quant=True, block_range=None, p_mx_group=None):
    """Closed form of Algorithm 1 for one request.

      w[r,j]   = exp(s[r,j] - m[r]) * sigma_K[j]          scale fusion, Alg.1 step 6
      M[r,b]   = max_{j in block b} w[r,j]                  Alg.1 step 6
      P'[r,j]  = E4M3(fp32(w[r,j] * 448 / M[r,b]))          step 7, sigma_p = M/448
      num[r,:] = sum_b (M[r,b]/448) sum_{j in b} dec(P'[r,j]) dec(kc[j,:])
                                                           V = latent codes, implicit
                                                           dequantization
      den[r]   = sum_j exp(s[r,j] - m[r])                  unquantized l (step 5), R12
      o = num / den ;  lse = m + ln(den)

    Alg.1 keeps O and l in units of the running sigma_p and rescales them by
    gamma = e^{m-m_new} sigma_p/sigma_p^cur; sigma_p*O and sigma_p*l are
    then exactly num and den above, and P' depends only on w / max_block(w), so
    the running max cancels (R13/R14).  Blocks are aligned to
    token 0 (R10); a block with M = 0 contributes nothing (R11).

    ``block_range=(b0, b1)`` restricts to key blocks [b0, b1) (one split-KV
    partial, combined by ``combine``).  ``p_quant=False`` replaces the P
    rounding by the identity (then O7 == O6 up to fp64 rounding).
    ``p_mx_group=g`` replaces the paper's P quantization by the NEXT-4(b) MX
    variant (``p_quant_mx``, power-of-two scale per g tokens) -- not the method.

    Returns (o [H,512] fp64, lse [H] fp64, natural log).
    """
    L = kc.shape[0]
    nb = (L + block - 1) // block
    b0, b1 = (0, nb) if block_range is None else block_range
    j0, j1 = b0 * block, min(b1 * block, L)
    s = logits(qc, sq, qr_bits, kc[j0:j1], sk[j0:j1], kr_bits[j0:j1], softmax_scale)
    m = s.max(axis=1)
    e = np.exp(s - m[:, None])
    w = e * np.asarray(sk[j0:j1], dtype=np.float64)[None, :]
    A = np.zeros_like(w)              # A[r,j] = (M[r,b]/448) dec(P'[r,j])
    if p_mx_group is not None:
        A = p_quant_mx(w, p_mx_group)
    for start in (range(0, j1 - j0, block) if p_mx_group is None else ()):
        sl = slice(start, min(start + block, j1 - j0))
        wb = w[:, sl]
        M = wb.max(axis=1)
        if p_quant:
            Ms = np.where(M > 0, M, 1.0)
            p_codes = encode_e4m3((wb * E4M3_MAX / Ms[:, None]).astype(np.float32))
            pd = decode_e4m3(p_codes)
            pd[M == 0] = 0.0
            A[:, sl] = (M / E4M3_MAX)[:, None] * pd
        else:
            A[:, sl] = wb
    num = A @ decode_e4m3(kc[j0:j1])
    den = e.sum(axis=1)
    return num / den[:, None], m + np.log(den)


def decode_mx(qc, sq, qr_bits, kc, sk, kr_bits, softmax_scale, block=B_C, p_quant=True):
    """NEXT-4(b) MX variant as the B200 kernel mla_decode_fp8_mx defines it (NOT the paper's
    method; DESIGN.md §7.10 and reading R28).  Per row r and 64-token block b (aligned to token 0):

      L2[r,j]  = s[r,j] * log2(e)                               (s: the O7 logits)
      R[r,b]   = ceil(max_{j in b} L2[r,j])                     integer reference of the block
      p[r,j]   = 2^(L2[r,j] - R[r,b]) ;  w = p * sigma_K[j]     (scale fusion as in P:237-239)
      e[r,b]   = ceil(log2(fp32(max_{j in b} w / 448)))         power-of-two P scale (UE8M0)
      P'[r,j]  = E4M3(fp32(w[r,j] / 2^e[r,b]))
      num[r,:] = sum_b 2^(e + R) sum_{j in b} dec(P'[r,j]) dec(kc[j,:])
      den[r]   = sum_b 2^R sum_{j in b} p[r,j] = sum_j 2^L2[r,j] = sum_j exp(s[r,j])
      o = num / den ;  lse = ln(den)

    The codes do not depend on the integer references (scaling w by 2^k scales 2^e by 2^k),
    so the kernel's clamped references give the same P'.  ``p_quant=False`` replaces the
    E4M3 rounding by the identity: then o == O6 exactly (the 2^(e+R) factors cancel).
    Returns (o [H,512] fp64, lse [H] fp64)."""
    L = kc.shape[0]
    s = logits(qc, sq, qr_bits, kc, sk, kr_bits, softmax_scale)
    L2 = s / np.log(2.0)
    skd = np.asarray(sk, dtype=np.float64)
    kd = decode_e4m3(kc)
    num = np.zeros((s.shape[0], kd.shape[1]))
    den = np.zeros(s.shape[0])
    for start in range(0, L, block):
        sl = slice(start, min(start + block, L))
        R = np.ceil(L2[:, sl].max(axis=1))
        p = np.exp2(L2[:, sl] - R[:, None])
        w = p * skd[None, sl]
        M = w.max(axis=1)
        Mf = (M / E4M3_MAX).astype(np.float32).astype(np.float64)
        e = np.ceil(np.log2(np.where(Mf > 0, Mf, 1.0)))
        if p_quant:
            A = decode_e4m3(encode_e4m3((w / np.exp2(e)[:, None]).astype(np.float32)))
            A[M == 0] = 0.0
        else:
            A = w / np.exp2(e)[:, None]
        num += np.exp2(e + R)[:, None] * (A @ kd[sl])
        den += np.exp2(R) * p.sum(axis=1)
    return num / den[:, None], np.log(den)


# --------------------------------------------------------------------------
# Algorithm 1, transcribed literally (dual warp group, o^L / o^R halves)
# --------------------------------------------------------------------------
def _alg1_block(s_blk, sK_blk, m, sigma_p, wg_l):
    """Alg.1 WG steps 4-9 for one key block (P:693-698 / P:718-723).
    Returns (p', sigma_p_cur, l_cur, gamma, m_new)."""
    m_cur = s_blk.max(axis=1)
    m_new = np.maximum(m, m_cur)                                   # step 4
    p = np.exp(s_blk - m_new[:, None])                             # step 5
    l_cur = p.sum(axis=1)
    p = p * sK_blk[None, :]                                        # step 6
    mc = p.max(axis=1)
    zero = mc == 0                                                 # R11
    sp_cur = np.where(zero, sigma_p, mc / E4M3_MAX)                # step 7
    pq = decode_e4m3(encode_e4m3((p / sp_cur[:, None]).astype(np.float32)))
    pq[zero] = 0.0
    l_cur = l_cur / sp_cur                                         # step 8
    with np.errstate(invalid="ignore"):
        gamma = np.where(np.isneginf(m), 0.0, np.exp(m - m_new)) * sigma_p / sp_cur  # step 9
    return pq, sp_cur, l_cur, gamma, m_new


def decode_alg1(qc, sq, qr_bits, kc, sk, kr_bits, softmax_scale, block=B_C):
    """Literal transcription of Algorithm 1 for one request with
    the Appendix-C strictly monotonic order.

    Two warp groups: WG0 owns o^L (first d_c/2 output columns) and processes
    even key blocks first; WG1 owns o^R and the odd blocks.  Each WG holds its
    own l register, summed by BlockReduceSum at the end (reading R14).  With an
    odd block count the last iteration has no K_1: WG1 folds o^R and its l with
    gamma_0 only and adds p_0 V_0^R (reading R15).
    """
    L = kc.shape[0]
    Tc = (L + block - 1) // block
    s_all = logits(qc, sq, qr_bits, kc, sk, kr_bits, softmax_scale)
    V = decode_e4m3(kc)                      # V = K_c
    sk = np.asarray(sk, dtype=np.float64)
    H = s_all.shape[0]
    half = D_C // 2
    m = np.full(H, -np.inf)
    sigma_p = np.ones(H)
    oL = np.zeros((H, half))
    oR = np.zeros((H, half))
    l0 = np.zeros(H)
    l1 = np.zeros(H)

    def blk(j):
        sl = slice(j * block, min((j + 1) * block, L))
        return s_all[:, sl], sk[sl], V[sl]

    for j in range(0, Tc, 2):
        # ---- WG0 (steps 1-15) on K_0 = K_j
        s0, sk0, V0 = blk(j)
        p0, sp0, lc0, g0, m0 = _alg1_block(s0, sk0, m, sigma_p, "L")
        oL = g0[:, None] * oL                                       # step 10
        l0 = g0 * l0 + lc0
        m, sigma_p = m0, sp0                                        # step 11
        oL = oL + p0 @ V0[:, :half]                                 # step 15
        if j + 1 < Tc:
            # ---- WG1 (steps 1-18) on K_1 = K_{j+1}; waits for gamma_0
            s1, sk1, V1 = blk(j + 1)
            p1, sp1, lc1, g1, m1 = _alg1_block(s1, sk1, m, sigma_p, "R")
            oR = g0[:, None] * oR                                   # step 11
            l1 = g1 * g0 * l1 + lc1
            m, sigma_p = m1, sp1                                    # step 12
            oR = oR + p0 @ V0[:, half:]                             # step 15
            oR = g1[:, None] * oR                                   # step 17
            oR = oR + p1 @ V1[:, half:]                             # step 18
            # ---- WG0 steps 16-18
            oL = g1[:, None] * oL
            l0 = g1 * l0
            oL = oL + p1 @ V1[:, :half]
        else:
            oR = g0[:, None] * oR                                   # R15 tail
            l1 = g0 * l1
            oR = oR + p0 @ V0[:, half:]
    l = l0 + l1                                                     # BlockReduceSum
    o = np.concatenate([oL, oR], axis=1) / l[:, None]
    lse = m + np.log(sigma_p * l)
    return o, lse


# --------------------------------------------------------------------------
# Reported references O6 / O8 (not gates)
# --------------------------------------------------------------------------
def attn_o6(qc, sq, qr_bits, kc, sk, kr_bits, softmax_scale):
    """Exact fp64 softmax attention over the dequantized cache:
    V_deq = dec(kc) * sigma_K (north_star: "fp64 attention over the
    dequantized cache").  Returns (o, lse)."""
    s = logits(qc, sq, qr_bits, kc, sk, kr_bits, softmax_scale)
    m = s.max(axis=1)
    e = np.exp(s - m[:, None])
    den = e.sum(axis=1)
    V = decode_e4m3(kc) * np.asarray(sk, dtype=np.float64)[:, None]
    return (e @ V) / den[:, None], m + np.log(den)


def attn_o8(q, c_kv, k_pe, softmax_scale):
    """fp64 absorbed-MLA attention over the UNQUANTIZED BF16 inputs (Eq.5):
    s = scale * (q_c . c_kv + q_r . k_pe), o = softmax(s) c_kv.  This is the
    "error against unquantized BF16 MLA" reference."""
    q = np.asarray(q, dtype=np.float64)
    c = np.asarray(c_kv, dtype=np.float64)
    r = np.asarray(k_pe, dtype=np.float64)
    s = float(softmax_scale) * (q[:, :D_C] @ c.T + q[:, D_C:] @ r.T)
    m = s.max(axis=1)
    e = np.exp(s - m[:, None])
    den = e.sum(axis=1)
    return (e @ c) / den[:, None], m + np.log(den)


# --------------------------------------------------------------------------
# a10: split-KV combine (Alg.1 returns o and the logsumexp L)
# --------------------------------------------------------------------------
def combine(o_parts, lse_parts):
    """o_parts [S,H,512], lse_parts [S,H] -> (o [H,512], lse [H]).
    L = log sum_s e^{L_s};  o = sum_s e^{L_s - L} o_s."""
    o_parts = np.asarray(o_parts, dtype=np.float64)
    lse_parts = np.asarray(lse_parts, dtype=np.float64)
    mx = lse_parts.max(axis=0)
    wts = np.exp(lse_parts - mx[None])
    tot = wts.sum(axis=0)
    lse = mx + np.log(tot)
    o = np.einsum("sh,shd->hd", wts / tot[None], o_parts)
    return o, lse


# --------------------------------------------------------------------------
# Whole request from the paged cache (a2 + gather + O7)
# --------------------------------------------------------------------------
def decode_request(q_rows, pools, block_table_row, L, softmax_scale, mx=False, **kw):
    """q-quant (a2), gather (a4), O7 (a5-a9) for one request; ``mx=True``: the NEXT-4(b)
    MX variant (decode_mx) instead.  q_rows [H,576] BF16 values.  Returns (o, lse)."""
    qc, sq, qr = q_quant(q_rows)
    kc, sk, kr = gather_request(pools, block_table_row, L)
    if mx:
        return decode_mx(qc, sq, qr, kc, sk, kr, softmax_scale, **kw)
    return decode_o7(qc, sq, qr, kc, sk, kr, softmax_scale, **kw)


# --------------------------------------------------------------------------
# NEXT-1: multi-token prediction (MTP).  The paper evaluates query
# lengths MTP in {1, 2} but does not spell out the mask; reading R25: the q_len new
# tokens are all in the cache and query token t (0-based) at position L - q_len + t
# attends causally to keys 0 .. L - q_len + t.
# --------------------------------------------------------------------------
def mtp_visible(L, q_len):
    """Visible key count of each query token: L - (q_len - 1 - t), t = 0..q_len-1 (>= 0)."""
    return [max(0, int(L) - (q_len - 1 - t)) for t in range(q_len)]


def decode_request_mtp(q_tok_rows, pools, block_table_row, L, softmax_scale, **kw):
    """q_tok_rows [q_len, H, 576]: O7 per query token over its visible keys.
    Returns o [q_len, H, 512], lse [q_len, H]; a token with no visible key -> 0, -inf."""
    q_tok_rows = np.asarray(q_tok_rows)
    T, H = q_tok_rows.shape[0], q_tok_rows.shape[1]
    o = np.zeros((T, H, D_C))
    lse = np.full((T, H), -np.inf)
    for t, Lt in enumerate(mtp_visible(L, T)):
        if Lt > 0:
            o[t], lse[t] = decode_request(q_tok_rows[t], pools, block_table_row, Lt, softmax_scale, **kw)
    return o, lse


def attn_o8_mtp(q_tok_rows, c_kv, k_pe, softmax_scale):
    """O8 (unquantized BF16 MLA, fp64) for q_len query tokens with the causal MTP mask."""
    q_tok_rows = np.asarray(q_tok_rows, dtype=np.float64)
    T, H = q_tok_rows.shape[0], q_tok_rows.shape[1]
    o = np.zeros((T, H, D_C))
    lse = np.full((T, H), -np.inf)
    for t, Lt in enumerate(mtp_visible(len(c_kv), T)):
        if Lt > 0:
            o[t], lse[t] = attn_o8(q_tok_rows[t], c_kv[:Lt], k_pe[:Lt], softmax_scale)
    return o, lse


# --------------------------------------------------------------------------
# NEXT-3: Fused-Fetch-Dequant (§3.3).  SPEC: C[i] = fp8_decode(code_i)
# * scale_i; K_r[i] = rope_i * scale_i (undoing the domain alignment); rows in
# token order.  Reading R26 (the paper names no output precision; the cache
# inputs were BF16): one fp32 product (IEEE RNE), then RNE to BF16.
# --------------------------------------------------------------------------
def fetch_dequant(pools, block_table_row, start, count):
    """Tokens start .. start+count-1 of one request -> (c_kv bf16 bits [count,512],
    k_pe bf16 bits [count,64])."""
    slots = np.array([slot_of(block_table_row, start + i) for i in range(count)], dtype=np.int64)
    codes = pools["kv_fp8"].reshape(-1, D_C)[slots]
    rope = pools["kv_rope"].reshape(-1, D_R)[slots]
    sig = pools["kv_scale"].reshape(-1)[slots].astype(np.float32)
    c = decode_e4m3(codes).astype(np.float32) * sig[:, None]                       # fp32 RNE product
    r = bf16_bits_to_f64(rope).astype(np.float32) * sig[:, None]
    return bf16_rne_bits(c), bf16_rne_bits(r)


# --------------------------------------------------------------------------
# NEXT-4(a): Table 2 KV-cache quantization configurations (granularities
# of Appendix A), for the numerical-accuracy ablation.  Each returns the
# DEQUANTIZED cache (content [L,512], rope [L,64]) in fp64; E4M3 RNE/satfinite codec
# throughout; dynamic scales sigma = max(amax / 448, 2^-24) (R1, R2).
# --------------------------------------------------------------------------
def _deq(x, sigma):
    return decode_e4m3(encode_e4m3(np.asarray(x, np.float64) / sigma)) * sigma


def kv_quant_config(content, rope, config, block=64):
    """config: "snapmla" (per-token content, RoPE BF16 pre-scaled, Eq.6), "A" (per-token
    over the whole 576-d row, RoPE quantized too), "B" (per-tensor static scale 1.0,
    RoPE unquantized), "C" (per-tensor dynamic, RoPE unquantized), "D" (per-block
    block x block tiles of the content, RoPE unquantized)."""
    c = np.asarray(content, np.float64)
    r = np.asarray(rope, np.float64)
    if config == "snapmla":
        codes, sig, rbits = per_token_quant(c.astype(np.float32), r.astype(np.float32))
        s = sig.astype(np.float64)[:, None]
        return decode_e4m3(codes) * s, bf16_bits_to_f64(rbits) * s
    if config == "A":
        row = np.concatenate([c, r], axis=1)
        sig = np.maximum(np.abs(row).max(axis=1, keepdims=True) / E4M3_MAX, 2.0 ** -24)
        q = _deq(row, sig)
        return q[:, :D_C], q[:, D_C:]
    if config == "B":
        return _deq(c, 1.0), r
    if config == "C":
        return _deq(c, max(np.abs(c).max() / E4M3_MAX, 2.0 ** -24)), r
    if config == "D":
        out = np.empty_like(c)
        for i in range(0, c.shape[0], block):
            for j in range(0, c.shape[1], block):
                blk = c[i:i + block, j:j + block]
                out[i:i + block, j:j + block] = _deq(blk, max(np.abs(blk).max() / E4M3_MAX, 2.0 ** -24))
        return out, r
    raise ValueError(config)


def attn_dequantized(q, c_deq, r_deq, softmax_scale):
    """exact fp64 softmax attention (Eq.5) of unquantized queries over a dequantized cache,
    V = the dequantized content (the KV-only part of the ablation)."""
    q = np.asarray(q, np.float64)
    s = float(softmax_scale) * (q[:, :D_C] @ c_deq.T + q[:, D_C:] @ r_deq.T)
    m = s.max(axis=1)
    e = np.exp(s - m[:, None])
    den = e.sum(axis=1)
    return (e @ c_deq) / den[:, None], m + np.log(den)


# --------------------------------------------------------------------------
# §4.3 error metrics: RMSE, cosine difference, relative L2
# --------------------------------------------------------------------------
def error_metrics(x, ref):
    x = np.asarray(x, dtype=np.float64).ravel()
    ref = np.asarray(ref, dtype=np.float64).ravel()
    d = x - ref
    rms_ref = np.sqrt(np.mean(ref ** 2))
    cos = float(x @ ref / (np.linalg.norm(x) * np.linalg.norm(ref)))
    return {
        "rmse": float(np.sqrt(np.mean(d ** 2))),
        "cos_diff": 1.0 - cos,
        "rel_l2": float(np.linalg.norm(d) / np.linalg.norm(ref)),
        "max_abs_rel_rms": float(np.max(np.abs(d)) / rms_ref),
        "mean_abs_rel_rms": float(np.mean(np.abs(d)) / rms_ref),
    }


def effective_peak(bf16_peak, n_fp8_tiles=16, n_bf16_tiles=1):
    """Eq.7: BF16-unit cost of 16 FP8 tiles + 1 BF16 tile is
    16/2 + 1 = 9 instead of 17, so peak_eff = peak_bf16 * 17 / 9."""
    return bf16_peak * (n_fp8_tiles + n_bf16_tiles) / (n_fp8_tiles / 2 + n_bf16_tiles)
