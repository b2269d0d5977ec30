// a1: RoPE-aware per-token FP8 quantize-on-append (Fused-K-Append).
//
// One warp per new token.  Lane l owns content dims [16l, 16l+16): two 16-byte
// loads, a shuffle-xor amax over the 512 content dims (RoPE excluded),
// sigma = max(amax / 448, 2^-24) with IEEE division (reading R1/R2/R4),
// E4M3 codes via cvt.rn.satfinite.e4m3x2.f32 of the IEEE quotient (R3), and one
// coalesced 16-byte store per lane into the paged slot (512 B per token).
// Lanes 0-7 also store the pre-scaled BF16 RoPE (Eq.6: k_pe / sigma, R5) and
// lane 0 the fp32 scale.  No FTZ (compiled without fast-math): subnormal BF16
// inputs divide exactly like the oracle.
#include "snapmla_internal.h"

namespace snapmla {

__global__ void __launch_bounds__(256) append_quant_kernel(const __nv_bfloat16* __restrict__ c_kv,
                                                           const __nv_bfloat16* __restrict__ k_pe,
                                                           const int32_t* __restrict__ block_table,
                                                           const int32_t* __restrict__ seq_lens, int batch,
                                                           int max_pages, uint8_t* __restrict__ kv_fp8,
                                                           __nv_bfloat16* __restrict__ kv_rope,
                                                           float* __restrict__ kv_scale) {
  pdl_launch_dependents();   // the decode's plan may start now (it reads no append output)
  const int lane = threadIdx.x & 31;
  const int tok = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (tok >= batch) return;
  const int L = seq_lens[tok];
  if (L <= 0) return;
  const int pos = L - 1;
  const int64_t slot = (int64_t)block_table[(int64_t)tok * max_pages + pos / kPage] * kPage + pos % kPage;

  // ---- content: 16 bf16 per lane
  const uint4* src = reinterpret_cast<const uint4*>(c_kv + (int64_t)tok * kDc) + lane * 2;
  uint4 raw[2] = {__ldg(src), __ldg(src + 1)};
  float x[16];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw[i]);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float2 f = __bfloat1622float2(h[k]);
      x[i * 8 + 2 * k] = f.x;
      x[i * 8 + 2 * k + 1] = f.y;
    }
  }
  float amax = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) amax = fmaxf(amax, fabsf(x[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  const float sigma = fmaxf(__fdiv_rn(amax, 448.0f), kSigmaMin);

  uint32_t packed[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint16_t lo = cvt_e4m3x2(__fdiv_rn(x[4 * i + 0], sigma), __fdiv_rn(x[4 * i + 1], sigma));
    const uint16_t hi = cvt_e4m3x2(__fdiv_rn(x[4 * i + 2], sigma), __fdiv_rn(x[4 * i + 3], sigma));
    packed[i] = (uint32_t)lo | ((uint32_t)hi << 16);
  }
  *reinterpret_cast<uint4*>(kv_fp8 + slot * kDc + lane * 16) = make_uint4(packed[0], packed[1], packed[2], packed[3]);

  // ---- RoPE: lanes 0-7, 8 bf16 each
  if (lane < 8) {
    const uint4 rr = __ldg(reinterpret_cast<const uint4*>(k_pe + (int64_t)tok * kDr) + lane);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&rr);
    uint4 outv;
    uint32_t* o = reinterpret_cast<uint32_t*>(&outv);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float2 f = __bfloat1622float2(h[k]);
      __nv_bfloat162 q = __halves2bfloat162(__float2bfloat16_rn(__fdiv_rn(f.x, sigma)),
                                            __float2bfloat16_rn(__fdiv_rn(f.y, sigma)));
      o[k] = *reinterpret_cast<uint32_t*>(&q);
    }
    *reinterpret_cast<uint4*>(kv_rope + slot * kDr + lane * 8) = outv;
  }
  if (lane == 0) kv_scale[slot] = sigma;
}

}  // namespace snapmla

using namespace snapmla;

extern "C" mla_status mla_kv_append_quant(const void* c_kv, const void* k_pe, const int32_t* block_table,
                                          const int32_t* seq_lens, int batch, int kv_lora_rank, int rope_dim,
                                          int page_size, int max_pages_per_seq, int64_t num_pages,
                                          uint8_t* kv_fp8, void* kv_rope, float* kv_scale,
                                          mla_stream_t stream) {
  if (batch < 0 || max_pages_per_seq < 0 || num_pages < 0) return MLA_ERR_SHAPE;
  if (kv_lora_rank != kDc || rope_dim != kDr || page_size != kPage) return MLA_ERR_UNSUPPORTED;
  if (batch == 0) return MLA_OK;
  if (!c_kv || !k_pe || !block_table || !seq_lens || !kv_fp8 || !kv_rope || !kv_scale) return MLA_ERR_NULL;
  if (max_pages_per_seq < 1) return MLA_ERR_SHAPE;
  if (!aligned(c_kv, 16) || !aligned(k_pe, 16) || !aligned(kv_fp8, 16) || !aligned(kv_rope, 16) ||
      !aligned(kv_scale, 4))
    return MLA_ERR_ALIGN;
  const int warps = 8;
  const int grid = (batch + warps - 1) / warps;
  append_quant_kernel<<<grid, warps * 32, 0, (cudaStream_t)stream>>>(
      (const __nv_bfloat16*)c_kv, (const __nv_bfloat16*)k_pe, block_table, seq_lens, batch, max_pages_per_seq,
      kv_fp8, (__nv_bfloat16*)kv_rope, kv_scale);
  return cudaGetLastError() == cudaSuccess ? MLA_OK : MLA_ERR_CUDA;
}

// NEXT-2 baseline: the unquantized BF16 cache of the same paged layout (content
// [P, 64, 512] and RoPE [P, 64, 64] planes, no scales).  One warp per new token,
// a straight 16-byte-vector copy into its paged slot.
namespace snapmla {
__global__ void __launch_bounds__(256) append_bf16_kernel(const uint4* __restrict__ c_kv, const uint4* __restrict__ k_pe,
                                                          const int32_t* __restrict__ block_table,
                                                          const int32_t* __restrict__ seq_lens, int batch,
                                                          int max_pages, uint4* __restrict__ kv_c,
                                                          uint4* __restrict__ kv_rope) {
  pdl_launch_dependents();   // the decode's plan may start now (it reads no append output)
  const int lane = threadIdx.x & 31;
  const int tok = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (tok >= batch) return;
  const int L = seq_lens[tok];
  if (L <= 0) return;
  const int pos = L - 1;
  const int64_t slot = (int64_t)block_table[(int64_t)tok * max_pages + pos / kPage] * kPage + pos % kPage;
  // 512 bf16 = 64 x 16 B: two vectors per lane; RoPE 64 bf16 = 8 vectors (lanes 0-7)
  const uint4 a = __ldg(c_kv + (int64_t)tok * 64 + lane), b = __ldg(c_kv + (int64_t)tok * 64 + 32 + lane);
  kv_c[slot * 64 + lane] = a;
  kv_c[slot * 64 + 32 + lane] = b;
  if (lane < 8) kv_rope[slot * 8 + lane] = __ldg(k_pe + (int64_t)tok * 8 + lane);
}
}  // namespace snapmla

extern "C" mla_status mla_kv_append_bf16(const void* c_kv, const void* k_pe, const int32_t* block_table,
                                         const int32_t* seq_lens, int batch, int kv_lora_rank, int rope_dim,
                                         int page_size, int max_pages_per_seq, int64_t num_pages, void* kv_c,
                                         void* kv_rope, mla_stream_t stream) {
  if (batch < 0 || max_pages_per_seq < 0 || num_pages < 0) return MLA_ERR_SHAPE;
  if (kv_lora_rank != kDc || rope_dim != kDr || page_size != kPage) return MLA_ERR_UNSUPPORTED;
  if (batch == 0) return MLA_OK;
  if (!c_kv || !k_pe || !block_table || !seq_lens || !kv_c || !kv_rope) return MLA_ERR_NULL;
  if (max_pages_per_seq < 1) return MLA_ERR_SHAPE;
  if (!aligned(c_kv, 16) || !aligned(k_pe, 16) || !aligned(kv_c, 16) || !aligned(kv_rope, 16)) return MLA_ERR_ALIGN;
  const int warps = 8;
  append_bf16_kernel<<<(batch + warps - 1) / warps, warps * 32, 0, (cudaStream_t)stream>>>(
      (const uint4*)c_kv, (const uint4*)k_pe, block_table, seq_lens, batch, max_pages_per_seq, (uint4*)kv_c,
      (uint4*)kv_rope);
  return cudaGetLastError() == cudaSuccess ? MLA_OK : MLA_ERR_CUDA;
}
