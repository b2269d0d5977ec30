// Layout check: tcgen05.mma kind::f8f6f4, M = 64, N = 64, K = 128 (4 x K = 32) with the
// A operand (a) in SMEM (K-major SWIZZLE_128B) and (b) in TMEM, same codes; the two
// fp32 accumulators must agree bit for bit.  Hypothesis for A in TMEM (M = 64 data-path
// layout, the one the M = 64 accumulator uses): row m at lane (m % 16) + 32 (m / 16)
// (+16 for the upper half-subpartition), column c holds K bytes 4c..4c+3 (low byte first).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
#include <cstdio>
#include <cstdlib>
#include "../paper_2602_10718_b200/csrc/ptx.cuh"
using namespace snapmla;

template <int SPLIT>
DEVI void st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x32bx2.x16.b32 [%0], %1, "
      "{%2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17};" ::"r"(taddr),
      "n"(SPLIT), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
DEVI void mma_f8_ta(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ uint8_t code_a(int m, int k) { return (uint8_t)(0x30 + ((m * 7 + k * 3) % 24)) | (((m + k) % 5 == 0) ? 0x80 : 0); }
__device__ uint8_t code_b(int n, int k) { return (uint8_t)(0x2c + ((n * 5 + k * 11) % 28)) | (((n * k) % 7 == 3) ? 0x80 : 0); }

__global__ void check(float* out, int bank_b) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // A (64 x 128 B) at 0, B (64 x 128 B) at 8192, both K-major SW128
  for (int i = tid; i < 64 * 128; i += blockDim.x) {
    const int r = i / 128, kb = i % 128;
    const int off = r * 128 + ((((kb >> 4) ^ (r & 7))) << 4) + (kb & 15);
    smem[off] = code_a(r, kb);
    smem[8192 + off] = code_b(r, kb);
  }
  if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&tbase, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  // A into TMEM: warp w -> rows 16w..16w+15; thread t<16 cols [256, 272), t>=16 cols [272, 288)
  const uint32_t abase = tm + (bank_b ? (16u << 16) : 0u) + 256u;
  {
    const int t = lane & 15, h = lane >> 4;
    const int m = 16 * warp + t;
    uint32_t v[16];
    for (int c = 0; c < 16; ++c) {
      const int col = 16 * h + c;   // 32-bit column inside the row: K bytes 4col..4col+3
      v[c] = (uint32_t)code_a(m, 4 * col) | ((uint32_t)code_a(m, 4 * col + 1) << 8) |
             ((uint32_t)code_a(m, 4 * col + 2) << 16) | ((uint32_t)code_a(m, 4 * col + 3) << 24);
    }
    st16<16>(abase + ((uint32_t)(32 * warp) << 16), v);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  constexpr uint32_t idesc = make_idesc(0, 0, 0, 0, 64, 64);
  const uint32_t sb = smem_u32(smem);
  if (warp == 0 && lane == 0) {
    for (int kk = 0; kk < 4; ++kk) {
      mma_f8(tm + 0, make_smem_desc(sb + kk * 32, 16, 1024, LAYOUT_SW128),
             make_smem_desc(sb + 8192 + kk * 32, 16, 1024, LAYOUT_SW128), idesc, kk > 0);
      mma_f8_ta(tm + 64, abase + 8 * kk, make_smem_desc(sb + 8192 + kk * 32, 16, 1024, LAYOUT_SW128), idesc, kk > 0);
    }
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  // read both accumulators (lanes 0-15 of each subpartition, M = 64 layout)
  {
    const int t = lane & 15, h = lane >> 4;
    const int m = 16 * warp + t;
    uint32_t d1[32], d2[32];
    tmem_ld_16x32bx2_x32<32>(tm + ((uint32_t)(32 * warp) << 16), d1);
    tmem_ld_16x32bx2_x32<32>(tm + 64 + ((uint32_t)(32 * warp) << 16), d2);
    tmem_wait_ld();
    for (int c = 0; c < 32; ++c) {
      out[m * 64 + 32 * h + c] = __uint_as_float(d1[c]);
      out[4096 + m * 64 + 32 * h + c] = __uint_as_float(d2[c]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tm, 512); }
}

static float dec(uint8_t c) {
  const int s = c >> 7, e = (c >> 3) & 15, mt = c & 7;
  float v = e == 0 ? ldexpf((float)mt, -9) : ldexpf(1.f + mt / 8.f, e - 7);
  return s ? -v : v;
}

int main() {
  float* d;
  cudaMalloc(&d, 8192 * 4);
  cudaFuncSetAttribute(check, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  for (int bank = 0; bank < 2; ++bank) {
    cudaMemset(d, 0, 8192 * 4);
    check<<<1, 128, 32768>>>(d, bank);
    cudaError_t e = cudaDeviceSynchronize();
    float h[8192];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    int same = 0, ref_ok = 0;
    for (int i = 0; i < 4096; ++i) {
      same += h[i] == h[4096 + i];
    }
    // host reference for D1 (SMEM path) as a sanity check of the test itself
    for (int m = 0; m < 64; ++m)
      for (int n = 0; n < 64; ++n) {
        double acc = 0;
        for (int k = 0; k < 128; ++k) {
          auto ca = [&](int mm, int kk) { return (uint8_t)(0x30 + ((mm * 7 + kk * 3) % 24)) | (((mm + kk) % 5 == 0) ? 0x80 : 0); };
          auto cb = [&](int nn, int kk) { return (uint8_t)(0x2c + ((nn * 5 + kk * 11) % 28)) | (((nn * kk) % 7 == 3) ? 0x80 : 0); };
          acc += (double)dec(ca(m, k)) * dec(cb(n, k));
        }
        ref_ok += fabs(acc - h[m * 64 + n]) <= 1e-3 * (1 + fabs(acc));
      }
    printf("A in TMEM bank %d: %s; smem path vs host ref %d/4096; tmem path == smem path %d/4096  (d1[0]=%g d2[0]=%g)\n",
           bank, cudaGetErrorString(e), ref_ok, same, h[0], h[4096]);
  }
  return 0;
}
