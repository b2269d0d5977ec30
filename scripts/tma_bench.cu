// Micro-benchmark: paged KV streaming through TMA, no compute.  One CTA per SM
// walks its share of randomly permuted pages; a consumer thread releases each
// stage as soon as it lands.  Measures HBM GB/s vs pipeline depth and box shape.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda.h>
#include "../paper_2602_10718_b200/csrc/ptx.cuh"
using namespace snapmla;

__global__ void __launch_bounds__(128, 1) stream(const __grid_constant__ CUtensorMap tm_kv,
                                                 const __grid_constant__ CUtensorMap tm_rope, const int* pages,
                                                 int pages_per_cta, int stages, int blocks_per_stage, int rope) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[8], empty[8];
  const uint32_t sbase = smem_u32(smem);
  const uint32_t stage_bytes = blocks_per_stage * (32768 + (rope ? 8192 : 0));
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  const int* pg = pages + (size_t)blockIdx.x * pages_per_cta;
  const int ngroups = pages_per_cta / blocks_per_stage;
  if (threadIdx.x == 0) {
    const uint64_t pol = l2_policy_evict_first();
    for (int g = 0; g < ngroups; ++g) {
      const int st = g % stages;
      mbar_wait(&empty[st], ((g / stages) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[st], stage_bytes);
      for (int b = 0; b < blocks_per_stage; ++b) {
        const int row = pg[g * blocks_per_stage + b] * 64;
        const uint32_t dst = sbase + st * stage_bytes + b * (32768 + (rope ? 8192 : 0));
        for (int c = 0; c < 4; ++c) tma_load_2d(dst + c * 8192, &tm_kv, &full[st], c * 128, row, pol);
        if (rope) tma_load_2d(dst + 32768, &tm_rope, &full[st], 0, row, pol);
      }
    }
  } else if (threadIdx.x == 32) {
    for (int g = 0; g < ngroups; ++g) {
      const int st = g % stages;
      mbar_wait(&full[st], (g / stages) & 1);
      mbar_arrive(&empty[st]);
    }
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const long num_pages = 150000;   // 150000 x 40 KB = 6.1 GB
  uint8_t *kv, *rope;
  cudaMalloc(&kv, (size_t)num_pages * 32768);
  cudaMalloc(&rope, (size_t)num_pages * 8192);
  cudaMemset(kv, 0, (size_t)num_pages * 32768);
  cudaMemset(rope, 0, (size_t)num_pages * 8192);
  void* fnp;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fnp;
  CUtensorMap tkv, trope;
  cuuint64_t d1[2] = {512, (cuuint64_t)num_pages * 64}, s1[1] = {512};
  cuuint32_t b1[2] = {128, 64}, e[2] = {1, 1};
  enc(&tkv, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, kv, d1, s1, b1, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint64_t d2[2] = {64, (cuuint64_t)num_pages * 64}, s2[1] = {128};
  cuuint32_t b2[2] = {64, 64};
  enc(&trope, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, rope, d2, s2, b2, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int ctas = 148, per = 1000;   // 148 x 1000 pages
  std::vector<int> perm(num_pages);
  for (long i = 0; i < num_pages; ++i) perm[i] = (int)i;
  std::shuffle(perm.begin(), perm.end(), std::mt19937(1));
  int* dp;
  cudaMalloc(&dp, sizeof(int) * ctas * per);
  cudaMemcpy(dp, perm.data(), sizeof(int) * ctas * per, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  struct Cfg { int stages, bps, rope; };
  for (Cfg c : {Cfg{1, 1, 1}, Cfg{2, 1, 1}, Cfg{3, 1, 1}, Cfg{4, 1, 1}, Cfg{5, 1, 1}, Cfg{2, 2, 1}, Cfg{4, 1, 0},
                Cfg{6, 1, 0}, Cfg{3, 2, 0}}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      stream<<<ctas, 128, 220 * 1024>>>(tkv, trope, dp, per, c.stages, c.bps, c.rope);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double bytes = (double)ctas * per * (32768 + (c.rope ? 8192 : 0));
      if (rep == 1)
        printf("stages=%d blocks/stage=%d rope=%d in-flight/SM=%3d KB: %.0f GB/s (%s)\n", c.stages, c.bps, c.rope,
               c.stages * c.bps * (32 + 8 * c.rope), bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
