// Micro-benchmark: tcgen05.mma throughput for the decode's MMA shapes (one CTA,
// single issuing thread, operands in SMEM, accumulator in TMEM).  Prints cycles
// per MMA instruction.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
#include <cstdio>
#include <cuda.h>
#include "../paper_2602_10718_b200/csrc/ptx.cuh"
using namespace snapmla;

DEVI bool elect_one() {
  uint32_t pred;
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\tselp.u32 %0, 1, 0, e;\n\t}" : "=r"(pred));
  return pred != 0;
}
DEVI uint32_t lane_id() { return threadIdx.x & 31; }

template <int M, int N, int KIND, int BMN, int ALAYOUT, int NACC = 1, int NISSUE = 1>
__global__ void bench(unsigned long long* out, int reps, int ninstr_arg) {
  const bool nowait = ninstr_arg < 0;
  const int ninstr = nowait ? -ninstr_arg : ninstr_arg;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bars[4];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&tbase, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (NISSUE == 0 && warp == 1) {
    // whole warp converged; one lane elected inside the asm
    uint64_t& bar = bars[0];
    const uint32_t sb = smem_u32(smem);
    constexpr uint32_t idesc = make_idesc(KIND == 0 ? 0 : 1, KIND == 0 ? 0 : 1, 0, BMN, M, N);
    unsigned long long t0 = 0;
    for (int r = 0; r < reps + 1; ++r) {
      if (r == 1) t0 = clock64();
#pragma unroll 4
      for (int i = 0; i < ninstr; ++i) {
        uint64_t a = make_smem_desc(sb + (i & 3) * 32, 16, 1024, LAYOUT_SW128);
        uint64_t b = make_smem_desc(sb + 65536 + (i & 3) * 32, 16, 1024, LAYOUT_SW128);
        asm volatile(
            "{\n\t.reg .pred p, e;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(tbase),
            "l"(a), "l"(b), "r"(idesc), "r"((uint32_t)(i > 0))
            : "memory");
      }
      if (elect_one()) mma_commit(&bar);
      __syncwarp();
      if (!nowait) mbar_wait(&bar, r & 1);
    }
    if (nowait) { uint64_t* b2 = &bars[3]; if (elect_one()) mma_commit(b2); __syncwarp(); mbar_wait(b2, 0); }
    if (lane_id() == 0) out[0] = clock64() - t0;
  }
  if (NISSUE > 0 && (threadIdx.x & 31) == 0 && warp >= 1 && warp <= NISSUE) {
    uint64_t& bar = bars[warp - 1];
    const uint32_t accoff = (warp - 1) * 128;
    const uint32_t sb = smem_u32(smem);
    constexpr uint32_t idesc = make_idesc(KIND == 0 ? 0 : 1, KIND == 0 ? 0 : 1, 0, BMN, M, N);
    unsigned long long t0 = 0;
    for (int r = 0; r < reps + 1; ++r) {
      if (r == 1) t0 = clock64();
      for (int i = 0; i < ninstr; ++i) {
        uint64_t a = ALAYOUT == 2 ? make_smem_desc(sb + (i & 3) * 32, 16, 1024, LAYOUT_SW128)
                                  : make_smem_desc(sb + (i & 1) * 2048, 1024, 128, LAYOUT_NONE);
        uint64_t b = BMN ? make_smem_desc(sb + 65536 + (i & 1) * 4096, 8192, 1024, LAYOUT_SW128)
                         : make_smem_desc(sb + 65536 + (i & 3) * 32, 16, 1024, LAYOUT_SW128);
        const uint32_t d = tbase + accoff + (uint32_t)((i % NACC) * (N >= 256 ? 256 : 128));
        if (KIND == 0) mma_f8(d, a, b, idesc, i >= NACC);
        else mma_bf16(d, a, b, idesc, i >= NACC);
      }
      const unsigned long long tc0 = clock64();
      mma_commit(&bar);
      const unsigned long long tc1 = clock64();
      if (r == reps && warp == 1) out[8] = tc1 - tc0;
      if (!nowait) mbar_wait(&bar, r & 1);
    }
    if (nowait) { uint64_t* b2 = &bars[3]; mma_commit(b2); mbar_wait(b2, 0); }
    out[warp - 1] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tbase, 512); }
}

template <int M, int N, int KIND, int BMN, int ALAYOUT, int NACC = 1, int NISSUE = 1>
void run(const char* name, int ninstr, int nctas) {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 256);
  auto k = bench<M, N, KIND, BMN, ALAYOUT, NACC, NISSUE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int reps = 200;
  k<<<nctas, 128, 200 * 1024>>>(d, reps, ninstr);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double per = (double)h / reps / (ninstr < 0 ? -ninstr : ninstr) / (NISSUE > 0 ? NISSUE : 1);
  const double macs = (double)M * N * (KIND == 0 ? 32 : 16);
  unsigned long long hc = 0;
  cudaMemcpy(&hc, d + 8, 8, cudaMemcpyDeviceToHost);
  printf("%-40s ctas=%3d: %7.1f cyc/instr  %7.0f MAC/cyc/SM  commit-stall %llu (%s)\n", name, nctas, per,
         macs / per, hc, cudaGetErrorString(e));
  cudaFree(d);
}

int main2();
int main() {
  run<64, 64, 0, 0, 2, 1, 0>("CONVERGED fp8 M64 N64, 128/commit", 128, 1);
  run<64, 64, 0, 0, 2, 1, 0>("CONVERGED fp8 M64 N64, 20/commit wait", 20, 1);
  run<64, 64, 0, 0, 2, 1, 0>("CONVERGED fp8 M64 N64, 20/commit nowait", -20, 1);
  run<64, 256, 0, 1, 0, 1, 0>("CONVERGED fp8 M64 N256, 64/commit", 64, 1);
  run<64, 64, 0, 0, 2, 1, 1>("fp8 M64 N64, commit/16, no wait", -16, 1);
  run<64, 64, 0, 0, 2, 1, 1>("fp8 M64 N64, commit/4, no wait", -4, 1);
  run<64, 256, 0, 1, 0, 1, 1>("fp8 M64 N256 PV, commit/2 no wait", -2, 1);
  run<128, 128, 0, 0, 2, 1, 1>("fp8 M128 N128, commit/4 no wait", -4, 1);
  run<64, 64, 0, 0, 2, 1, 1>("fp8 M64 N64, 1 issuer, 128/commit", 128, 1);
  run<64, 64, 0, 0, 2, 1, 1>("fp8 M64 N64, 1 issuer, 512/commit", 512, 1);
  run<128, 128, 0, 0, 2, 1, 1>("fp8 M128 N128, 1 issuer, 128/commit", 128, 1);
  run<64, 256, 0, 1, 0, 1, 1>("fp8 M64 N256 PV, 1 issuer 64/commit", 64, 1);
  run<128, 256, 0, 0, 2, 1, 1>("fp8 M128 N256, 1 issuer 64/commit", 64, 1);
  run<64, 64, 1, 0, 2, 1, 1>("bf16 M64 N64, 1 issuer, 128/commit", 128, 1);
  run<64, 128, 0, 0, 2, 1, 1>("fp8 M64 N128, 1 issuer, 128/commit", 128, 1);
  run<64, 64, 0, 0, 2, 1, 2>("fp8 M64 N64, 2 issuing warps", 16, 1);
  run<64, 64, 0, 0, 2, 1, 4>("fp8 M64 N64, 4 issuing warps", 16, 1);
  run<128, 128, 0, 0, 2, 1, 2>("fp8 M128 N128, 2 issuing warps", 16, 1);
  run<64, 256, 0, 1, 0, 1, 2>("fp8 M64 N256 PV, 2 issuing warps", 8, 1);
  run<64, 64, 0, 0, 2, 2>("fp8 M64 N64 2 accumulators", 16, 1);
  run<64, 64, 0, 0, 2, 4>("fp8 M64 N64 4 accumulators", 16, 1);
  run<128, 64, 0, 0, 2, 2>("fp8 M128 N64 2 accumulators", 16, 1);
  run<128, 64, 0, 0, 2, 4>("fp8 M128 N64 4 accumulators", 16, 1);
  run<128, 128, 0, 0, 2, 2>("fp8 M128 N128 2 accumulators", 16, 1);
  run<128, 128, 0, 0, 2, 4>("fp8 M128 N128 4 accumulators", 16, 1);
  run<64, 256, 0, 1, 0, 2>("fp8 M64 N256 PV 2 accumulators", 8, 1);
  run<128, 256, 0, 0, 2, 2>("fp8 M128 N256 2 accumulators", 8, 1);
  run<64, 128, 0, 0, 2, 1>("fp8 M64 N128", 16, 1);
  run<64, 128, 0, 0, 2, 2>("fp8 M64 N128 2 accumulators", 16, 1);
  run<64, 64, 1, 0, 2, 2>("bf16 M64 N64 2 accumulators", 16, 1);
  if (0) main2();
  for (int nc : {1}) {
    run<64, 64, 0, 0, 2>("fp8 M64 N64 K-major (QK)", 16, nc);
    run<64, 64, 1, 0, 2>("bf16 M64 N64 K-major (QK rope)", 16, nc);
    run<64, 256, 0, 1, 0>("fp8 M64 N256 B MN-major, A none (PV)", 8, nc);
    run<64, 256, 0, 1, 2>("fp8 M64 N256 B MN-major, A SW128", 8, nc);
    run<64, 256, 0, 0, 2>("fp8 M64 N256 B K-major", 8, nc);
    run<128, 64, 0, 0, 2>("fp8 M128 N64 K-major", 16, nc);
    run<128, 128, 0, 0, 2>("fp8 M128 N128 K-major", 16, nc);
    run<128, 256, 0, 0, 2>("fp8 M128 N256 K-major", 8, nc);
    run<128, 256, 0, 1, 2>("fp8 M128 N256 B MN-major", 8, nc);
    run<128, 256, 1, 0, 2>("bf16 M128 N256 K-major", 8, nc);
  }
  return 0;
}

// ---------------------------------------------------------------- cta_group::2
namespace snapmla {
DEVI void mma_f8_2sm(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
DEVI void mma_commit_2sm(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(smem_u32(bar)), "h"((uint16_t)3) : "memory");
}
DEVI uint32_t cluster_rank() { uint32_t r; asm volatile("mov.u32 %0, %cluster_ctarank;" : "=r"(r)); return r; }
DEVI void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
}  // namespace snapmla

template <int M, int N>
__global__ void __cluster_dims__(2, 1, 1) bench2(unsigned long long* out, int reps, int ninstr) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_rank();
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  fence_proxy_async_smem();
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (threadIdx.x == 32 && rank == 0) {
    const uint32_t sb = smem_u32(smem);
    constexpr uint32_t idesc = make_idesc(0, 0, 0, 0, M, N);
    unsigned long long t0 = 0;
    for (int r = 0; r < reps + 1; ++r) {
      if (r == 1) t0 = clock64();
      for (int i = 0; i < ninstr; ++i) {
        uint64_t a = make_smem_desc(sb + (i & 3) * 32, 16, 1024, LAYOUT_SW128);
        uint64_t b = make_smem_desc(sb + 65536 + (i & 3) * 32, 16, 1024, LAYOUT_SW128);
        mma_f8_2sm(tbase, a, b, idesc, i > 0);
      }
      mma_commit_2sm(&bar);
      mbar_wait(&bar, r & 1);
    }
    out[blockIdx.x] = clock64() - t0;
  }
  if (threadIdx.x == 32 && rank == 1) {
    for (int r = 0; r < reps + 1; ++r) mbar_wait(&bar, r & 1);
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512) : "memory");
  }
}

template <int M, int N>
void run2(const char* name, int ninstr, int nctas) {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 256);
  cudaMemset(d, 0, 8 * 256);
  auto k = bench2<M, N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int reps = 200;
  k<<<nctas, 128, 200 * 1024>>>(d, reps, ninstr);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double per = (double)h / reps / ninstr;
  const double macs = (double)M * N * 32 / 2;   // per SM
  printf("%-40s ctas=%3d: %7.1f cyc/instr  %7.0f MAC/cyc/SM  (%s)\n", name, nctas, per, macs / per,
         cudaGetErrorString(e));
  cudaFree(d);
}

int main2() {
  for (int nc : {2, 148}) {
    run2<128, 64>("2SM fp8 M128 N64", 16, nc);
    run2<128, 128>("2SM fp8 M128 N128", 16, nc);
    run2<128, 256>("2SM fp8 M128 N256", 8, nc);
    run2<256, 64>("2SM fp8 M256 N64", 16, nc);
    run2<256, 128>("2SM fp8 M256 N128", 16, nc);
    run2<256, 256>("2SM fp8 M256 N256", 8, nc);
  }
  return 0;
}
