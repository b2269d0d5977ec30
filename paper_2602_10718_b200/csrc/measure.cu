// Measurement kernel for the roofline denominator (not on the hot path): a read-only
// HBM stream, so bench.py can report the decode's DRAM traffic -- which is all reads
// (644 B per cached token in, ~0 out) -- against what this B200 sustains for reads,
// next to MEASURED_PEAKS.json's copy bandwidth (read + write).  SURVEY.md §8(d) asks
// for "a read-only stream ... on the box".
//
// Grid-stride loop of 16-byte loads, 4 in flight per thread, 4 CTAs of 512 threads
// per SM; every loaded word is folded into an XOR so the loads cannot be elided; one
// 8-byte result per CTA.
#include "snapmla_internal.h"

namespace snapmla {

__global__ void __launch_bounds__(512) read_stream_kernel(const uint4* __restrict__ src, size_t n16,
                                                          unsigned long long* __restrict__ sink) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t acc = 0;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = __ldcs(src + i + k * stride);
#pragma unroll
    for (int k = 0; k < 4; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
  }
  for (; i < n16; i += stride) {
    const uint4 v = __ldcs(src + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  acc = __reduce_xor_sync(0xffffffffu, acc);
  if ((threadIdx.x & 31) == 0) atomicXor(sink + blockIdx.x, (unsigned long long)acc);
}

// Exhaustive check of the product's E4M3 encoder (cvt4_e4m3 -> cvt.rn.satfinite.e4m3x2.f32, used
// by the append, the Q quantization and the P quantization): out[i] = E4M3 code of the fp32 whose
// bit pattern is first + i.  Four consecutive patterns per thread, exactly as the kernels pack them.
__global__ void __launch_bounds__(256) cvt_sweep_kernel(uint32_t first, uint32_t count, uint32_t* __restrict__ out) {
  const uint32_t n4 = count / 4;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x) {
    const uint32_t b = first + 4 * i;
    out[i] = cvt4_e4m3(__uint_as_float(b), __uint_as_float(b + 1), __uint_as_float(b + 2), __uint_as_float(b + 3));
  }
}

}  // namespace snapmla

using namespace snapmla;

// Debug / test only (include/snapmla_debug.h).
extern "C" mla_status mla_debug_cvt_e4m3(uint32_t first_bits, uint32_t count, uint8_t* out, mla_stream_t stream) {
  if (!out) return MLA_ERR_NULL;
  if (count % 4 != 0) return MLA_ERR_SHAPE;
  if (!aligned(out, 4)) return MLA_ERR_ALIGN;
  if (count == 0) return MLA_OK;
  const int sms = device_num_sms();
  if (sms <= 0) return MLA_ERR_CUDA;
  cvt_sweep_kernel<<<sms * 8, 256, 0, (cudaStream_t)stream>>>(first_bits, count, reinterpret_cast<uint32_t*>(out));
  return cudaGetLastError() == cudaSuccess ? MLA_OK : MLA_ERR_CUDA;
}

// Debug / measurement only (include/snapmla_debug.h).
extern "C" mla_status mla_measure_read_stream(const void* buf, size_t bytes, unsigned long long* sink,
                                              int sink_len, mla_stream_t stream) {
  if (!buf || !sink) return MLA_ERR_NULL;
  if (bytes % 16 != 0 || sink_len <= 0) return MLA_ERR_SHAPE;
  if (!aligned(buf, 16)) return MLA_ERR_ALIGN;
  const int sms = device_num_sms();
  if (sms <= 0) return MLA_ERR_CUDA;
  const int grid = sms * 4 < sink_len ? sms * 4 : sink_len;
  read_stream_kernel<<<grid, 512, 0, (cudaStream_t)stream>>>(static_cast<const uint4*>(buf), bytes / 16, sink);
  return cudaGetLastError() == cudaSuccess ? MLA_OK : MLA_ERR_CUDA;
}
