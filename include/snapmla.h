/*
 * snapmla.h -- C ABI of the B200 (sm_100a) SnapMLA FP8 MLA decode hot path.
 *
 * Method: SnapMLA, arXiv 2602.10718 ("P:n" = PAPER.md line n).  The library
 * implements three calls, one per step of BASELINE.json's north_star:
 *   mla_kv_append_quant  RoPE-aware per-token FP8 quantize-on-append (Fused-K-Append,
 *                        §3.3; §3.1; Eq.6)
 *   mla_decode_fp8       absorbed-MLA FP8 decode with the reconstructed PV pipeline
 *                        (Eq.5, §3.2, Algorithm 1 P:666-744,
 *                        Appendix C order enforcement P:759-764); Q quantization
 *                        (Fused-Q-Quant) runs in its prologue
 *   mla_decode_fp8_ex    the same with q_len query tokens per request (MTP)
 *   mla_kv_fetch_dequant Fused-Fetch-Dequant (§3.3): paged FP8 cache -> BF16
 *   mla_combine          split-KV merge of the per-split (o, logsumexp) partials
 *                        (Algorithm 1 returns o and L)
 *
 * Conventions (all calls)
 *   - Every tensor pointer is a DEVICE pointer owned by the caller.  The library
 *     never allocates, frees or synchronizes; each call only enqueues work on
 *     `stream` (a cudaStream_t; NULL = legacy default stream).
 *   - Tensors are dense, row-major.  Base pointers must be 16-byte aligned; the
 *     three KV pools must be 128-byte aligned (TMA).
 *   - Fixed problem dims (north_star): kv_lora_rank = 512, rope_dim = 64,
 *     page_size = 64.  Anything else returns MLA_ERR_UNSUPPORTED.
 *   - Host-side argument errors return before anything is enqueued; launch
 *     failures return MLA_ERR_CUDA.  No exception crosses the ABI.
 *   - Device-side preconditions (undefined behaviour if violated): valid page
 *     ids in block_table; 0 <= seq_lens[b] <= max_pages_per_seq * 64; KV pools
 *     zero-initialised at allocation (stale bytes must never be FP8 NaN codes);
 *     finite inputs; appends for a request are stream-ordered before the decode
 *     that reads them.
 *   - Deterministic: identical inputs on the same GPU give bitwise identical
 *     outputs (no atomics in reductions).
 *   - Thread safety: every call may be made concurrently from several host
 *     threads, on any streams and devices (the current device of the calling
 *     thread is used).  The only process-wide state is (a) per-device launch
 *     records (SM count, dynamic-SMEM attributes, cluster occupancy) set once,
 *     (b) a 32-entry cache of encoded TMA tensor maps keyed by (device, pool
 *     base, pool rows, kind) -- a pool freed and re-allocated at the same
 *     address with the same extent reuses a map that is still valid -- both
 *     under one mutex, and (c) the debug switches of snapmla_debug.h (atomics).
 *   - Kernel choice (mla_decode_fp8 / _ex, 64 < q_len x heads <= 128): the
 *     block-pair 2-SM kernel when batch x max_pages_per_seq >= 16384 (the
 *     block table's extent bounds the work; seq_lens stay on the device), else
 *     the single-CTA kernel.  Both compute the same closed form (O7).
 */
#ifndef SNAPMLA_H_
#define SNAPMLA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* mla_stream_t; /* == cudaStream_t */

typedef enum {
  MLA_OK = 0,
  MLA_ERR_NULL = 1,        /* a required pointer is NULL                     */
  MLA_ERR_SHAPE = 2,       /* negative / inconsistent sizes                  */
  MLA_ERR_UNSUPPORTED = 3, /* dims outside the supported set                 */
  MLA_ERR_ALIGN = 4,       /* pointer alignment violated                     */
  MLA_ERR_WORKSPACE = 5,   /* workspace missing or too small                 */
  MLA_ERR_CUDA = 6         /* CUDA runtime / driver error (launch, encode)   */
} mla_status;

/* Human-readable name of a status code (static storage). */
const char* mla_status_str(mla_status s);

/* ABI version of this header (bumped on any signature change). */
int mla_abi_version(void);

/*
 * mla_kv_append_quant -- quantize-on-append of one new token per request.
 *
 * Per request b, with the new token at position p = seq_lens[b] - 1
 * (seq_lens is the length AFTER the append):
 *   sigma      = max(fp32(max_i |c_kv[b,i]| / 448), 2^-24)       (content dims only)
 *   code[i]    = E4M3_RNE_SATFINITE(fp32(c_kv[b,i] / sigma))     (IEEE division)
 *   rope'[k]   = BF16_RNE(fp32(k_pe[b,k] / sigma))              (Eq.6 pre-scaled alignment)
 *   slot       = block_table[b, p / 64] * 64 + p % 64
 *   kv_fp8[slot,:] = code;  kv_rope[slot,:] = rope';  kv_scale[slot] = sigma
 * Bit-exact with the oracle (tests/test_gpu_append.py).  Requests with
 * seq_lens[b] <= 0 are skipped.
 *
 *   c_kv        bf16  [batch, kv_lora_rank]        latent of the new token
 *   k_pe        bf16  [batch, rope_dim]            post-RoPE key of the new token
 *   block_table int32 [batch, max_pages_per_seq]   page ids into the pools
 *   seq_lens    int32 [batch]                      lengths after the append
 *   kv_fp8      uint8 [num_pages, page_size, kv_lora_rank]   E4M3 codes (written)
 *   kv_rope     bf16  [num_pages, page_size, rope_dim]       k_pe / sigma (written)
 *   kv_scale    fp32  [num_pages, page_size]                 sigma (written)
 */
mla_status mla_kv_append_quant(const void* c_kv, const void* k_pe, const int32_t* block_table,
                               const int32_t* seq_lens, int batch, int kv_lora_rank, int rope_dim,
                               int page_size, int max_pages_per_seq, int64_t num_pages, uint8_t* kv_fp8,
                               void* kv_rope, float* kv_scale, mla_stream_t stream);

/*
 * Workspace bytes that mla_decode_fp8 / mla_combine need for `batch` requests
 * and `num_heads` query heads.  num_sms <= 0 means "the current device".
 * The workspace holds the split plan, the Fused-Q-Quant results (E4M3 codes, q_r', sigma_q
 * per query row) and the fp32 per-split partials.
 */
size_t mla_decode_workspace_bytes(int batch, int num_heads, int num_sms);

/*
 * mla_decode_fp8 -- absorbed-MLA FP8 decode over the paged cache, one query
 * token per request (MTP = 1).
 *
 * Per request b and head h (q row = [q_nope absorbed (512) | q_pe (64)]):
 *   sigma_q = max(fp32(amax(q[b,h,:512]) / 448), 2^-24); q codes = E4M3(q/sigma_q);
 *   q_r'    = BF16(q_pe / sigma_q)                                      (Fused-Q-Quant)
 *   s_j     = softmax_scale * sigma_q * sigma_K[j] * (q_codes . K_codes[j] + q_r' . k_r'[j])
 *   per 64-token key block (aligned to token 0): online softmax, scale fusion
 *   w_j = p_j * sigma_K[j], block-wise P quantization P' = E4M3(w * 448 / max_block w),
 *   O <- gamma O + P' V_codes with V = the latent codes, blocks in increasing order.
 * Result (through mla_combine): o = softmax-weighted latent (512), natural-log LSE.
 * Writes only the workspace (split plan + quantized q + fp32 partials); call mla_combine next.
 * Two launches on `stream`: the plan (which also runs Fused-Q-Quant, one warp per q row) and
 * the decode kernel, a programmatic dependent of it.
 *
 *   q             bf16  [batch, num_heads, 576]
 *   kv_*          the pools written by mla_kv_append_quant (read only)
 *   block_table   int32 [batch, max_pages_per_seq];  seq_lens int32 [batch]
 *   num_heads     1..128 (64-row head tiles, H < 64 zero-padded; H <= 16: heads on the MMA N
 *                 dimension instead)
 *   softmax_scale multiplies the dequantized logit (e.g. 1/sqrt(192) * mscale^2)
 *   workspace     device buffer of >= mla_decode_workspace_bytes(batch, num_heads, 0)
 */
mla_status mla_decode_fp8(const void* q, const uint8_t* kv_fp8, const void* kv_rope, const float* kv_scale,
                          const int32_t* block_table, const int32_t* seq_lens, int batch, int num_heads,
                          int kv_lora_rank, int rope_dim, int page_size, int max_pages_per_seq,
                          int64_t num_pages, float softmax_scale, void* workspace, size_t workspace_bytes,
                          mla_stream_t stream);

/*
 * mla_decode_fp8_ex -- the same decode with q_len >= 1 query tokens per request
 * (multi-token prediction, MTP; the paper evaluates MTP in {1, 2}).
 *
 *   q          bf16 [batch, q_len, num_heads, 576]; row (t, h) = t * num_heads + h
 *   query token t (0-based) sits at position seq_lens[b] - q_len + t and attends to
 *   keys 0 .. seq_lens[b] - q_len + t (causal; all q_len new tokens are already in
 *   the cache; reading R25).  A token that sees no key yields o = 0,
 *   lse = -inf.
 *   q_len * num_heads <= 256 rows per request (64-row tiles).
 * Workspace / mla_combine / mla_combine_f32 take num_heads = q_len * num_heads
 * (rows); out is then [batch, q_len, num_heads, 512].  mla_decode_fp8 is this call
 * with q_len = 1 (and num_heads <= 128).
 */
mla_status mla_decode_fp8_ex(const void* q, const uint8_t* kv_fp8, const void* kv_rope, const float* kv_scale,
                             const int32_t* block_table, const int32_t* seq_lens, int batch, int num_heads,
                             int q_len, int kv_lora_rank, int rope_dim, int page_size, int max_pages_per_seq,
                             int64_t num_pages, float softmax_scale, void* workspace, size_t workspace_bytes,
                             mla_stream_t stream);

/*
 * mla_decode_fp8_mx -- NEXT-4(b): the MX-scaled P variant (NOT the paper's method; reading R28,
 * DESIGN.md §7.10).  Same arguments, workspace and follow-up (mla_combine / _f32, num_heads =
 * q_len x heads rows) as mla_decode_fp8_ex, with q_len x num_heads <= 128.  P' of each 64-token
 * block is quantized with a power-of-two scale 2^ceil(log2(max w / 448)) instead of max w / 448
 * (P:696), the exponentials against an integer reference per block, so the tensor core applies
 * every block's scale (kind::mxf8f6f4.block_scale) and the output accumulates in tensor memory
 * without per-block rescaling.  Matches oracle.snapmla.decode_mx.  Valid while |logit| x log2(e)
 * < ~90 (scale exponents are clamped beyond).
 */
mla_status mla_decode_fp8_mx(const void* q, const uint8_t* kv_fp8, const void* kv_rope, const float* kv_scale,
                             const int32_t* block_table, const int32_t* seq_lens, int batch, int num_heads,
                             int q_len, int kv_lora_rank, int rope_dim, int page_size, int max_pages_per_seq,
                             int64_t num_pages, float softmax_scale, void* workspace, size_t workspace_bytes,
                             mla_stream_t stream);

/*
 * mla_combine -- merge split-KV partials left in `workspace` by the preceding
 * mla_decode_fp8 (same batch / num_heads, stream-ordered):
 *   L = log sum_s e^{L_s};   o = sum_s e^{L_s - L} o_s
 *   out  bf16 [batch, num_heads, kv_lora_rank]  (RNE from fp32)
 *   lse  fp32 [batch, num_heads], natural log; may be NULL
 * A request with seq_lens[b] == 0 yields out = 0 and lse = -inf.
 * The workspace must come from a decode with the same batch and num_heads (rows: q_len x
 * heads for MTP) on a device with the same SM count: the decode's plan header records
 * them and the combine kernel traps (the stream's context reports an error) on a mismatch
 * instead of reading partials at the wrong offsets.
 */
mla_status mla_combine(const void* workspace, int batch, int num_heads, int kv_lora_rank, void* out, float* lse,
                       mla_stream_t stream);

/*
 * mla_kv_fetch_dequant -- Fused-Fetch-Dequant (§3.3; NEXT-3): read the
 * cached tokens [tok_start[b], tok_start[b] + count_b) of every request from the
 * paged pools and dequantize them on load:
 *   c_kv_out[i, d] = BF16(fp32(dec(code) * sigma_K))        d < 512
 *   k_pe_out[i, e] = BF16(fp32(k_r'[e] * sigma_K))          e < 64 (undoes Eq.6)
 * (one fp32 RNE product, then RNE to BF16; reading R26).
 *   out_offset   int32 [batch] exclusive prefix of the per-request counts: request
 *                b's tokens are output rows out_offset[b] .. out_offset[b] + count_b - 1,
 *                rows in token order; total_rows = sum of counts.  Ranges must lie
 *                inside each request's cache (not checked on the device).
 *   c_kv_out     bf16 [total_rows, 512];  k_pe_out bf16 [total_rows, 64]
 */
mla_status mla_kv_fetch_dequant(const uint8_t* kv_fp8, const void* kv_rope, const float* kv_scale,
                                const int32_t* block_table, const int32_t* tok_start, const int32_t* out_offset,
                                int batch, int kv_lora_rank, int rope_dim, int page_size, int max_pages_per_seq,
                                int64_t num_pages, int64_t total_rows, void* c_kv_out, void* k_pe_out,
                                mla_stream_t stream);

/*
 * NEXT-2 baseline: the UNQUANTIZED BF16 MLA decode in the same
 * kernel skeleton, for the paper's FP8-vs-BF16 comparison.
 * It is not the method: no quantization anywhere; P (the softmax weights) is
 * rounded to BF16 for the PV tensor-core product, as BF16 FlashMLA-style kernels do.
 *
 * mla_kv_append_bf16 -- copy the new token's latent into the BF16 paged pools
 *   kv_c    bf16 [num_pages, page_size, 512]   (slot as in mla_kv_append_quant)
 *   kv_rope bf16 [num_pages, page_size, 64]    (raw k_pe: no scale, no Eq.6 alignment)
 *
 * mla_decode_bf16 -- s_j = softmax_scale * (q . [c_kv_j | k_pe_j]) in fp32 (BF16 x BF16
 * tensor-core products), online softmax per 64-token block, O <- gamma O + BF16(p) c_kv,
 * split-KV partials in `workspace` exactly like mla_decode_fp8_ex (same q layout,
 * q_len, row limits, workspace size and mla_combine / mla_combine_f32 follow-up).
 * Pools must be 128-byte aligned; errors as for mla_decode_fp8_ex.
 */
mla_status mla_kv_append_bf16(const void* c_kv, const void* k_pe, const int32_t* block_table,
                              const int32_t* seq_lens, int batch, int kv_lora_rank, int rope_dim, int page_size,
                              int max_pages_per_seq, int64_t num_pages, void* kv_c, void* kv_rope,
                              mla_stream_t stream);
mla_status mla_decode_bf16(const void* q, const void* kv_c, const void* kv_rope, const int32_t* block_table,
                           const int32_t* seq_lens, int batch, int num_heads, int q_len, int kv_lora_rank,
                           int rope_dim, int page_size, int max_pages_per_seq, int64_t num_pages,
                           float softmax_scale, void* workspace, size_t workspace_bytes, mla_stream_t stream);

/*
 * mla_combine_gather -- NEXT-4(c): mla_combine with the tensor-parallel all-gather fused
 * into its epilogue.  With heads partitioned over `world` ranks (rank r decoded heads
 * [r * num_heads, (r + 1) * num_heads) into `workspace`), every rank's combined BF16 rows
 * are stored straight into ALL ranks' gathered outputs:
 *   out_peers[i]  bf16 [batch, world * num_heads, 512] on rank i (host array of `world`
 *                 device pointers, peer-mapped, e.g. CUDA IPC / symmetric memory over
 *                 NVLink; world <= 8); rank r writes rows r * num_heads + h.
 *   lse           fp32 [batch, num_heads] of this rank's heads (local), may be NULL.
 * The stores are plain P2P writes: the caller orders them before any consumer on another
 * rank with a stream-ordered barrier (e.g. a one-element NCCL all-reduce) after this call.
 * Write-after-read: rank r's NEXT gather may overwrite rank j's output while rank j still
 * reads the previous step's rows, so successive steps must alternate between two output
 * buffers (step parity; bench.py --fused-gather does) or put a stream-ordered barrier
 * BEFORE this call as well.
 */
mla_status mla_combine_gather(const void* workspace, int batch, int num_heads, int kv_lora_rank,
                              void* const* out_peers, int world, int rank, float* lse, mla_stream_t stream);

/* Same as mla_combine but writes fp32 output [batch, num_heads, kv_lora_rank]
 * (diagnostic: exposes the kernel result before the final BF16 rounding). */
mla_status mla_combine_f32(const void* workspace, int batch, int num_heads, int kv_lora_rank, float* out,
                           float* lse, mla_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* SNAPMLA_H_ */
