// Probe of the two MMA forms the MX-scaled decode kernel (NEXT-4(b)) relies on,
// checked against a CPU product on the same operands:
//  (1) tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale, M = 128, N = 256, K = 2 x 32:
//      A = P' (E4M3, SMEM, K-major core matrices), B = V (E4M3, SMEM, MN-major SW128, two 64-token x
//      128-dim boxes), SFA = one UE8M0 per row copied SMEM -> TMEM with tcgen05.cp 32x128b.warpx4
//      (row m at lane m % 32 of column m / 32, all four bytes equal), SFB = 127 (2^0) everywhere;
//      the second K step accumulates.  D[r][n] = 2^(e_r - 127) sum_k A[r][k] B[k][n].
//  (2) tcgen05.mma.cta_group::1.kind::f8f6f4, M = 128, N = 64, K = 32, A from TMEM (lane r = row r,
//      columns = 4 codes each), B = K tile (SMEM, K-major SW128).
//  nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2602_10718_b200/csrc -o scripts/mx_probe scripts/mx_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "ptx.cuh"

using namespace snapmla;

static float dec_e4m3(uint8_t c) {
  const int s = c >> 7, e = (c >> 3) & 15, m = c & 7;
  float v = e == 0 ? m * std::ldexp(1.f, -9) : (1.f + m / 8.f) * std::ldexp(1.f, e - 7);
  return s ? -v : v;
}

__device__ __forceinline__ void tmem_cp_32x128b_warpx4(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}

__host__ __device__ constexpr uint32_t idesc_bs(uint32_t M, uint32_t N, uint32_t a_mn, uint32_t b_mn) {
  // block-scaled: a/b format E4M3 (0), scale_format E8M0 (bit 23), sf ids 0
  return (a_mn << 15) | (b_mn << 16) | ((N >> 3) << 17) | (1u << 23) | ((M >> 4) << 24);
}

__global__ void probe_kernel(const uint8_t* gA, const uint8_t* gB, const uint8_t* gSF, const uint8_t* gQ,
                             const uint8_t* gK, float* out1, float* out2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* sm = smem_raw + (sbase - smem_u32(smem_raw));
  // layout: A 8 KB @0 | B 16 KB @8192 | SF 512 B @24576 | K tile 8 KB @32768 | bars @40960
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 8192; i += blockDim.x) {   // A: byte(row, k) = (k/16)*2048 + row*16 + k%16
    const int row = i / 64, k = i % 64;
    sm[(k / 16) * 2048 + row * 16 + k % 16] = gA[i];
  }
  for (int i = tid; i < 64 * 256; i += blockDim.x) {   // B: token t, dim d -> box d/128, SW128
    const int t = i / 256, d = i % 256, box = d / 128, db = d % 128;
    const int chunk = (db / 16) ^ (t % 8);
    sm[8192 + box * 8192 + t * 128 + chunk * 16 + db % 16] = gB[i];
  }
  for (int i = tid; i < 512; i += blockDim.x) sm[24576 + i] = gSF[i];
  for (int i = tid; i < 64 * 32; i += blockDim.x) {   // K tile for (2): token n, dim k (32) -> SW128 row of 128 B
    const int n = i / 32, k = i % 32;
    const int chunk = (k / 16) ^ (n % 8);
    sm[32768 + n * 128 + chunk * 16 + k % 16] = gK[i];
  }
  const uint32_t bar = sbase + 40960, tslot = sbase + 40968;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = lds_u32(tslot);
  // SFB = 127 in columns 264..271 of every lane; Q codes for (2) in columns 384..391 (lane = row)
  {
    uint32_t v[32];
    for (int i = 0; i < 32; ++i) v[i] = 0x7F7F7F7Fu;
    const uint32_t lane_off = (uint32_t)(32 * (warp & 3)) << 16;
    if (warp < 4) tmem_st_32x32b_x32(tmem + lane_off + 264, v);   // cols 264..295
    const int row = 32 * (warp & 3) + (tid & 31);
    for (int c = 0; c < 8; ++c) {
      const uint8_t* q = gQ + row * 32 + 4 * c;
      v[c] = q[0] | (q[1] << 8) | (q[2] << 16) | ((uint32_t)q[3] << 24);
    }
    for (int c = 8; c < 32; ++c) v[c] = 0;
    if (warp < 4) tmem_st_32x32b_x32(tmem + lane_off + 384, v);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    if (elect_one()) {
      const uint64_t dSF = make_smem_desc(sbase + 24576, 16, 128, LAYOUT_NONE);
      tmem_cp_32x128b_warpx4(tmem + 256, dSF);   // SFA: columns 256..259
      const uint64_t dA = make_smem_desc(sbase, 2048, 128, LAYOUT_NONE);
      const uint64_t dB = make_smem_desc(sbase + 8192, 8192, 1024, LAYOUT_SW128);
      const uint32_t id = idesc_bs(128, 256, 0, 1);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %6, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], %1, %2, %3, [%4], [%5], p;\n\t}" ::"r"(tmem),
          "l"(dA), "l"(dB), "r"(id), "r"(tmem + 256), "r"(tmem + 264), "r"(0)
          : "memory");
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %6, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], %1, %2, %3, [%4], [%5], p;\n\t}" ::"r"(tmem),
          "l"(dA + 256), "l"(dB + 256), "r"(id), "r"(tmem + 256), "r"(tmem + 264), "r"(1)
          : "memory");
      // (2): D2 (cols 400..463) = Q (TMEM) x K^T
      const uint64_t dK = make_smem_desc(sbase + 32768, 16, 1024, LAYOUT_SW128);
      const uint32_t id2 = make_idesc(0, 0, 0, 0, 128, 64);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + 400),
          "r"(tmem + 384), "l"(dK), "r"(id2), "r"(0)
          : "memory");
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
    }
    __syncwarp();
  }
  mbar_wait(bar, 0);
  tc_fence_after();
  if (warp < 4) {
    const int row = 32 * warp + (tid & 31);
    const uint32_t lane_off = (uint32_t)(32 * warp) << 16;
    for (int c = 0; c < 256; c += 32) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tmem + lane_off + c, v);
      tmem_wait_ld();
      for (int i = 0; i < 32; ++i) out1[row * 256 + c + i] = __uint_as_float(v[i]);
    }
    for (int c = 0; c < 64; c += 32) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tmem + lane_off + 400 + c, v);
      tmem_wait_ld();
      for (int i = 0; i < 32; ++i) out2[row * 64 + c + i] = __uint_as_float(v[i]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

static uint8_t rnd_code(unsigned& s) {
  s = s * 1664525u + 1013904223u;
  uint8_t c = (s >> 24) & 0xFF;
  if ((c & 0x7F) == 0x7F) c ^= 1;   // no NaN
  return c;
}

int main() {
  unsigned seed = 1;
  std::vector<uint8_t> A(128 * 64), B(64 * 256), SF(512), Q(128 * 32), K(64 * 32);
  for (auto& x : A) x = rnd_code(seed);
  for (auto& x : B) x = rnd_code(seed);
  for (auto& x : Q) x = rnd_code(seed);
  for (auto& x : K) x = rnd_code(seed);
  std::vector<int> e(128);
  for (int m = 0; m < 128; ++m) {
    e[m] = 127 + (getenv("MXSPREAD") ? ((m * 37) % 81) - 40 : (m % 9) - 4);
    for (int s = 0; s < 4; ++s) SF[(m % 32) * 16 + (m / 32) * 4 + s] = (uint8_t)e[m];
  }
  uint8_t *dA, *dB, *dSF, *dQ, *dK;
  float *o1, *o2;
  cudaMalloc(&dA, A.size()); cudaMalloc(&dB, B.size()); cudaMalloc(&dSF, 512); cudaMalloc(&dQ, Q.size());
  cudaMalloc(&dK, K.size()); cudaMalloc(&o1, 128 * 256 * 4); cudaMalloc(&o2, 128 * 64 * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dSF, SF.data(), 512, cudaMemcpyHostToDevice);
  cudaMemcpy(dQ, Q.data(), Q.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dK, K.data(), K.size(), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  probe_kernel<<<1, 256, 48 * 1024>>>(dA, dB, dSF, dQ, dK, o1, o2);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(err)); return 1; }
  std::vector<float> h1(128 * 256), h2(128 * 64);
  cudaMemcpy(h1.data(), o1, h1.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(h2.data(), o2, h2.size() * 4, cudaMemcpyDeviceToHost);
  double e1 = 0, e2 = 0, r1 = 0, r2 = 0;
  int bad1 = 0;
  for (int r = 0; r < 128; ++r)
    for (int n = 0; n < 256; ++n) {
      double acc = 0;
      for (int k = 0; k < 64; ++k) acc += (double)dec_e4m3(A[r * 64 + k]) * dec_e4m3(B[k * 256 + n]);
      acc *= std::ldexp(1.0, e[r] - 127);
      const double d = std::fabs(acc - h1[r * 256 + n]);
      e1 = std::max(e1, d); r1 = std::max(r1, std::fabs(acc));
      if (d > 1e-5 * (1 + std::fabs(acc)) && bad1 < 8) { printf("mx mismatch r=%d e=%d n=%d ref=%g got=%g\n", r, e[r] - 127, n, acc, h1[r * 256 + n]); ++bad1; }
    }
  for (int r = 0; r < 128; ++r)
    for (int n = 0; n < 64; ++n) {
      double acc = 0;
      for (int k = 0; k < 32; ++k) acc += (double)dec_e4m3(Q[r * 32 + k]) * dec_e4m3(K[n * 32 + k]);
      e2 = std::max(e2, std::fabs(acc - h2[r * 64 + n])); r2 = std::max(r2, std::fabs(acc));
    }
  printf("block_scale PV probe: max|err| %.3g (max|ref| %.3g)  -> %s\n", e1, r1, e1 <= 1e-3 * r1 ? "OK" : "FAIL");
  printf("A-in-TMEM M=128 QK probe: max|err| %.3g (max|ref| %.3g)  -> %s\n", e2, r2, e2 <= 1e-4 * r2 ? "OK" : "FAIL");
  return 0;
}
