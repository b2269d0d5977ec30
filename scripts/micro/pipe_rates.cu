// Per-SMSP throughput of the softmax's instruction types on B200 (one CTA of 4 warps per SM,
// i.e. one warp per SMSP, 8 independent chains per thread): cycles per warp instruction.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(float* out, int iters, long long* cyc) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
  uint32_t u[8] = {};
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (OP == 1) { uint16_t r; asm volatile("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(a[i]), "f"(a[(i + 1) & 7])); u[i] += r; }
      if (OP == 2) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(a[(i + 3) & 7]), "f"(a[(i + 5) & 7]));
      if (OP == 3) { float2 x = make_float2(a[i], a[(i+1)&7]); asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(*(unsigned long long*)&x) : "l"(*(unsigned long long*)&x)); a[i] = x.x; }
      if (OP == 4) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a[i]));
      if (OP == 5) asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
    }
  }
  const long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i] + u[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 8);
  const char* names[] = {"MUFU.EX2", "F2FP e4m3x2", "FMNMX3", "FFMA2", "FFMA", "MUFU.RCP"};
  for (int op = 0; op < 6; ++op) {
    for (int warps : {1, 4, 8}) {
      const int iters = 4096;
      void (*fn)(float*, int, long long*) = op == 0 ? k<0> : op == 1 ? k<1> : op == 2 ? k<2> : op == 3 ? k<3> : op == 4 ? k<4> : k<5>;
      fn<<<148, 32 * warps>>>(out, iters, cyc);
      fn<<<148, 32 * warps>>>(out, iters, cyc);
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double per_smsp_instr = (double)iters * 8 * warps / (warps < 4 ? warps : 4);  // warp instrs per SMSP
      printf("%-12s warps/CTA %d: %.2f cycles per warp-instruction per SMSP\n", names[op], warps, c / per_smsp_instr);
    }
  }
  return 0;
}
