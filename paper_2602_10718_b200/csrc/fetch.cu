// NEXT-3: Fused-Fetch-Dequant (§3.3): read cached tokens from the paged
// FP8 pools and dequantize on the fly, for paths that reuse the cache at high
// precision (chunk prefill, prefix caching).
//
//   c_kv[i, d] = BF16(fp32(dec(code[i, d]) * sigma_K[i]))
//   k_pe[i, e] = BF16(fp32(rope'[i, e] * sigma_K[i]))          (undoes Eq.6's alignment)
//
// (reading R26: one fp32 product, RNE, then RNE to BF16 — the arithmetic a
// register-level dequantization performs; the oracle does the same two roundings.)
//
// One warp per 4 consecutive output rows (request found by a binary search over the
// caller's exclusive prefix `out_offset`, then advanced row by row); all loads are
// issued before any store.  Lane l dequantizes content dims [16l, 16l+16) from one
// 16-byte load into two 16-byte BF16 stores, lanes 0-7 the RoPE (16-byte load /
// store each).  Memory-bound: 644 B in, 1152 B out per token.
#include "snapmla_internal.h"

namespace snapmla {

__device__ __forceinline__ float e4m3_to_f32(uint32_t c) {
  // exact: every E4M3 value is an fp32 value (bias 7, 3 mantissa bits, subnormals at 2^-9)
  const uint32_t s = (c & 0x80u) << 24, e = (c >> 3) & 15u, m = c & 7u;
  const float mag = e == 0 ? __uint_as_float(0) + (float)m * 0x1p-9f : __uint_as_float(((e + 120u) << 23) | (m << 20));
  return __uint_as_float(__float_as_uint(mag) | s);
}

constexpr int kRowsPerWarp = 4;   // consecutive output rows per warp: 4 x 644 B of loads in flight

__global__ void __launch_bounds__(256) fetch_dequant_kernel(
    const uint8_t* __restrict__ kv_fp8, const __nv_bfloat16* __restrict__ kv_rope, const float* __restrict__ kv_scale,
    const int32_t* __restrict__ block_table, const int32_t* __restrict__ tok_start, const int32_t* __restrict__ out_offset,
    int batch, int max_pages, int64_t total_rows, __nv_bfloat16* __restrict__ c_out, __nv_bfloat16* __restrict__ r_out) {
  const int lane = threadIdx.x & 31;
  const int64_t row0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * kRowsPerWarp;
  if (row0 >= total_rows) return;
  // request of the first row: the last b with out_offset[b] <= row0 (offsets non-decreasing)
  int lo = 0, hi = batch - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if ((int64_t)__ldg(out_offset + mid) <= row0) lo = mid;
    else hi = mid - 1;
  }
  int b = lo;
  int64_t slot[kRowsPerWarp];
  bool ok[kRowsPerWarp];
#pragma unroll
  for (int k = 0; k < kRowsPerWarp; ++k) {
    const int64_t row = row0 + k;
    ok[k] = row < total_rows;
    while (ok[k] && b + 1 < batch && (int64_t)__ldg(out_offset + b + 1) <= row) ++b;
    const int pos = __ldg(tok_start + b) + (int)(row - __ldg(out_offset + b));
    slot[k] = ok[k] ? (int64_t)__ldg(block_table + (int64_t)b * max_pages + pos / kPage) * kPage + pos % kPage : 0;
  }
  // all loads first (memory-level parallelism), then dequantize and store
  uint4 codes[kRowsPerWarp], rr[kRowsPerWarp];
  float sigma[kRowsPerWarp];
#pragma unroll
  for (int k = 0; k < kRowsPerWarp; ++k) {
    if (!ok[k]) continue;
    codes[k] = __ldg(reinterpret_cast<const uint4*>(kv_fp8 + slot[k] * kDc) + lane);
    if (lane < 8) rr[k] = __ldg(reinterpret_cast<const uint4*>(kv_rope + slot[k] * kDr) + lane);
    sigma[k] = __ldg(kv_scale + slot[k]);
  }
#pragma unroll
  for (int k = 0; k < kRowsPerWarp; ++k) {
    if (!ok[k]) continue;
    const int64_t row = row0 + k;
    const uint32_t* cw = reinterpret_cast<const uint32_t*>(&codes[k]);
    uint32_t o[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t w = cw[i >> 1] >> (16 * (i & 1));
      const __nv_bfloat162 v =
          __halves2bfloat162(__float2bfloat16_rn(__fmul_rn(e4m3_to_f32(w & 0xffu), sigma[k])),
                             __float2bfloat16_rn(__fmul_rn(e4m3_to_f32((w >> 8) & 0xffu), sigma[k])));
      o[i] = *reinterpret_cast<const uint32_t*>(&v);
    }
    uint4* dst = reinterpret_cast<uint4*>(c_out + row * kDc) + 2 * lane;
    dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
    dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
    if (lane < 8) {
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&rr[k]);
      uint32_t ro[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __bfloat1622float2(h[q]);
        const __nv_bfloat162 v = __halves2bfloat162(__float2bfloat16_rn(__fmul_rn(f.x, sigma[k])),
                                                    __float2bfloat16_rn(__fmul_rn(f.y, sigma[k])));
        ro[q] = *reinterpret_cast<const uint32_t*>(&v);
      }
      reinterpret_cast<uint4*>(r_out + row * kDr)[lane] = make_uint4(ro[0], ro[1], ro[2], ro[3]);
    }
  }
}

}  // namespace snapmla

using namespace snapmla;

extern "C" mla_status mla_kv_fetch_dequant(const uint8_t* kv_fp8, const void* kv_rope, const float* kv_scale,
                                           const int32_t* block_table, const int32_t* tok_start,
                                           const int32_t* out_offset, int batch, int kv_lora_rank, int rope_dim,
                                           int page_size, int max_pages_per_seq, int64_t num_pages,
                                           int64_t total_rows, void* c_kv_out, void* k_pe_out, mla_stream_t stream) {
  if (batch < 0 || max_pages_per_seq < 0 || num_pages < 0 || total_rows < 0) return MLA_ERR_SHAPE;
  if (kv_lora_rank != kDc || rope_dim != kDr || page_size != kPage) return MLA_ERR_UNSUPPORTED;
  if (batch == 0 || total_rows == 0) return MLA_OK;
  if (!kv_fp8 || !kv_rope || !kv_scale || !block_table || !tok_start || !out_offset || !c_kv_out || !k_pe_out)
    return MLA_ERR_NULL;
  if (max_pages_per_seq < 1) return MLA_ERR_SHAPE;
  if (!aligned(kv_fp8, 16) || !aligned(kv_rope, 16) || !aligned(kv_scale, 4) || !aligned(c_kv_out, 16) ||
      !aligned(k_pe_out, 16))
    return MLA_ERR_ALIGN;
  const int warps = 8;
  const int64_t grid = (total_rows + warps * kRowsPerWarp - 1) / (warps * kRowsPerWarp);
  if (grid > 0x7fffffff) return MLA_ERR_UNSUPPORTED;
  fetch_dequant_kernel<<<(unsigned)grid, warps * 32, 0, (cudaStream_t)stream>>>(
      kv_fp8, (const __nv_bfloat16*)kv_rope, kv_scale, block_table, tok_start, out_offset, batch, max_pages_per_seq,
      total_rows, (__nv_bfloat16*)c_kv_out, (__nv_bfloat16*)k_pe_out);
  return cudaGetLastError() == cudaSuccess ? MLA_OK : MLA_ERR_CUDA;
}
