// TMEM load latency / throughput in the accumulator pattern (tcgen05.ld 32x32b -> FFMA2 on the
// loaded registers), per SMSP, vs chunk width and warps per SMSP.  One CTA per SM, 512 TMEM columns.
// Prints cycles per 64-column round trip per warp and the SM's TMEM read rate.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tmem_ld_lat.cu
#include <cstdio>
#include "../../paper_2602_10718_b200/csrc/ptx.cuh"
using namespace snapmla;

template <int W>   // W = 16 or 32 columns per load; MODE 0: load -> use; 1: two loads in flight, one wait
__global__ void __launch_bounds__(512, 1) k(float* out, int iters, long long* cyc, int nwarps, int mode) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(smem_u32(&tbase), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase + ((uint32_t)(32 * (warp & 3)) << 16);
  float o[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) o[i] = 0.f;
  const float g = 0.999f;
  long long t0 = clock64();
  if (warp < nwarps) {
    for (int it = 0; it < iters; ++it) {
      const uint32_t a = tmem + 64 * ((it + warp) & 7) % 448;
      if (mode == 0) {
#pragma unroll
        for (int c = 0; c < 64; c += W) {
          uint32_t r[W];
          if (W == 32) tmem_ld_32x32b_x32(a + c, *reinterpret_cast<uint32_t(*)[32]>(r));
          else tmem_ld_32x32b_x16(a + c, *reinterpret_cast<uint32_t(*)[16]>(r));
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < W; e += 2) {
            float2 v = __ffma2_rn(make_float2(o[c + e], o[c + e + 1]), make_float2(g, g),
                                  make_float2(__uint_as_float(r[e]), __uint_as_float(r[e + 1])));
            o[c + e] = v.x;
            o[c + e + 1] = v.y;
          }
        }
      } else if (mode == 2) {   // 16x256b.x4: lanes 0-15 and 16-31, 32 columns -> 32 registers per round
#pragma unroll
        for (int c = 0; c < 64; c += 32) {
          uint32_t r[32];
          asm volatile(
              "tcgen05.ld.sync.aligned.16x256b.x4.b32 "
              "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
              : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
              : "r"(a + c));
          asm volatile(
              "tcgen05.ld.sync.aligned.16x256b.x4.b32 "
              "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
              : "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
              : "r"(a + c + (16u << 16)));
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            float2 v = __ffma2_rn(make_float2(o[c + e], o[c + e + 1]), make_float2(g, g),
                                  make_float2(__uint_as_float(r[e]), __uint_as_float(r[e + 1])));
            o[c + e] = v.x;
            o[c + e + 1] = v.y;
          }
        }
      } else {
        uint32_t r[64];
        tmem_ld_32x32b_x32(a, *reinterpret_cast<uint32_t(*)[32]>(r));
        tmem_ld_32x32b_x32(a + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 64; e += 2) {
          float2 v = __ffma2_rn(make_float2(o[e], o[e + 1]), make_float2(g, g),
                                make_float2(__uint_as_float(r[e]), __uint_as_float(r[e + 1])));
          o[e] = v.x;
          o[e + 1] = v.y;
        }
      }
    }
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 64; ++i) s += o[i];
  out[blockIdx.x * 512 + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 512 * 4);
  cudaMalloc(&cyc, 8);
  const int iters = 2000;
  for (int mode = 0; mode < 3; ++mode)
    for (int W : {16, 32}) {
      if (mode >= 1 && W == 16) continue;
      for (int nw : {4, 8, 12, 16}) {
        auto fn = W == 16 ? k<16> : k<32>;
        fn<<<148, 512>>>(out, iters, cyc, nw, mode);
        fn<<<148, 512>>>(out, iters, cyc, nw, mode);
        cudaError_t e = cudaDeviceSynchronize();
        if (e) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        long long c;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        const double per = (double)c / iters;   // cycles per 64-column round per warp
        const double bytes = (double)nw * 64 * 32 * 4 * iters;
        printf("mode %d W=%2d warps/SM=%2d (per SMSP %d): %7.1f cycles per 64 cols per warp, SM TMEM read %6.1f B/cycle %s\n",
               mode, W, nw, nw / 4, per, bytes / c, e ? cudaGetErrorString(e) : "");
      }
    }
  return 0;
}
