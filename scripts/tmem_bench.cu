// Micro-benchmark: TMEM load / store / load-scale-store throughput vs number of
// warps (the O-rescale pattern of the decode correction step).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
#include <cstdio>
#include "../paper_2602_10718_b200/csrc/ptx.cuh"
using namespace snapmla;

DEVI void ld32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
DEVI void st32x32b_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
      "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]),
      "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

// full-lane 32x32b variant: 128 lanes x 256 cols per sweep = 128 KB
template <int MODE>
__global__ void tbench32(unsigned long long* out, int reps) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&tbase, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const int nw = blockDim.x >> 5;
  const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
  const int sharers = nw / 4, my = warp >> 2;
  const int cols = 256 / sharers;
  uint32_t v[32];
  for (int i = 0; i < 32; ++i) v[i] = i;
  const float g = 1.0001f;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    for (int c = my * cols; c < (my + 1) * cols; c += 32) {
      const uint32_t ta = tbase + lane_base + c;
      if (MODE == 0) { ld32x32b_x32(ta, v); tmem_wait_ld(); }
      else if (MODE == 1) st32x32b_x32(ta, v);
      else {
        ld32x32b_x32(ta, v); tmem_wait_ld();
        for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * g);
        st32x32b_x32(ta, v);
      }
    }
    tmem_wait_st();
  }
  __syncthreads();
  if (threadIdx.x == 0) out[0] = clock64() - t0;
  if (threadIdx.x == 0 && v[3] == 12345) out[1] = 1;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tbase, 512); }
}

template <int MODE>   // 0: ld only, 1: st only, 2: ld * g -> st
__global__ void tbench(unsigned long long* out, int reps) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&tbase, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const int nw = blockDim.x >> 5;
  const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
  // warps sharing a subpartition split the 512 columns
  const int sharers = nw / 4, my = warp >> 2;
  const int cols = 256 / sharers;   // SPLIT=256 covers [c, c+32) and [c+256, c+288)
  uint32_t v[32];
  for (int i = 0; i < 32; ++i) v[i] = i;
  const float g = 1.0001f;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    for (int c = my * cols; c < (my + 1) * cols; c += 32) {
      const uint32_t ta = tbase + lane_base + c;
      if (MODE == 0) {
        tmem_ld_16x32bx2_x32<256>(ta, v);
        tmem_wait_ld();
      } else if (MODE == 1) {
        tmem_st_16x32bx2_x32<256>(ta, v);
      } else {
        tmem_ld_16x32bx2_x32<256>(ta, v);
        tmem_wait_ld();
        for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * g);
        tmem_st_16x32bx2_x32<256>(ta, v);
      }
    }
    tmem_wait_st();
  }
  __syncthreads();
  if (threadIdx.x == 0) out[0] = clock64() - t0;
  if (threadIdx.x == 0 && v[3] == 12345) out[1] = 1;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tbase, 512); }
}

template <int MODE, bool FULL = false>
void run(const char* name, int nwarps) {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  const int reps = 200;
  if (FULL) tbench32<MODE><<<1, nwarps * 32>>>(d, reps);
  else tbench<MODE><<<1, nwarps * 32>>>(d, reps);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  // bytes touched per rep: 128 lanes... 16x32bx2 touches 16 lanes x 2 x 32 cols per warp-instr
  // whole sweep covers 64 lanes (half sub-partitions) x 512 cols x 4 B = 128 KB per rep
  const double bytes = 64.0 * 512 * 4 * (MODE == 2 ? 2 : 1);
  printf("%-28s warps=%2d: %7.1f cycles per 128 KB sweep (%.0f B/cycle)  %s\n", name, nwarps, (double)h / reps,
         bytes * reps / h, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  for (int w : {4, 8}) {
    run<0, true>("FULL 32x32b ld", w);
    run<1, true>("FULL 32x32b st", w);
    run<2, true>("FULL 32x32b rescale", w);
  }
  for (int w : {4, 8, 16}) {
    run<0>("tmem ld (16x32bx2.x32)", w);
    run<1>("tmem st", w);
    run<2>("tmem ld*g->st (rescale)", w);
  }
  return 0;
}
