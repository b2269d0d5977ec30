// Probe: data-path layout of tcgen05.mma.cta_group::2 (CTA pair, M = 128 = 64 rows per CTA)
// kind::f8f6f4, as the H = 128 decode would use it.  Dumps both CTAs' TMEM and matches every
// (lane, col) against the expected D of every (cta, row, col) on the host.
//   mode 0: QK-like  A (64 x 128 B, K-major SW128) in SMEM, B = 32 rows per CTA (K-major SW128), N = 64
//   mode 1: QK-like  A from TMEM (written with the M = 64 layout: row m at lane (m%16) + 32 (m/16))
//   mode 2: PV-like  A = 64 x 64 B K-major no swizzle (core matrices), B = MN-major SW128, 64 K rows x
//           128 N bytes per CTA, N = 256
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/pair_probe.cu -o /tmp/pair_probe -lcuda
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2602_10718_b200/csrc/ptx.cuh"
using namespace snapmla;

__host__ __device__ uint32_t hash3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t h = a * 0x9E3779B1u ^ (b + 0x7F4A7C15u) * 0x85EBCA77u ^ (c + 0x165667B1u) * 0xC2B2AE3Du;
  h ^= h >> 15; h *= 0x2C1B3C6Du; h ^= h >> 12; h *= 0x297A2D39u; h ^= h >> 15;
  return h;
}
// E4M3 codes with exponents 2^-3..2^2 (|v| in [0.125, 7.5]) and random sign/mantissa
__host__ __device__ uint8_t code_a(int cta, int m, int k) {
  const uint32_t h = hash3(1 + cta, m, k);
  return (uint8_t)(((4 + (h % 6)) << 3) | ((h >> 8) & 7) | ((h >> 12) & 1 ? 0x80 : 0));
}
__host__ __device__ uint8_t code_b(int cta, int n, int k) {
  const uint32_t h = hash3(11 + cta, n, k);
  return (uint8_t)(((4 + (h % 6)) << 3) | ((h >> 8) & 7) | ((h >> 12) & 1 ? 0x80 : 0));
}
double dec_e4m3(uint8_t c) {
  const int s = c >> 7, e = (c >> 3) & 15, m = c & 7;
  double v = e == 0 ? ldexp(m / 8.0, -6) : ldexp(1.0 + m / 8.0, e - 7);
  return s ? -v : v;
}

DEVI void st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x32bx2.x16.b32 [%0], 16, "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) probe(float* dump, int mode) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar, bar1;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cta = (int)cluster_ctarank();
  // A at 0 (8 KB), B at 8192 (8 KB)
  if (mode != 2) {
    for (int i = tid; i < 64 * 128; i += blockDim.x) {
      const int r = i / 128, kb = i % 128;
      const int off = r * 128 + ((((kb >> 4) ^ (r & 7))) << 4) + (kb & 15);
      smem[off] = code_a(cta, r, kb);
      if (r < 32) smem[8192 + off] = code_b(cta, r, kb);   // B: 32 N rows (tokens) x 128 K bytes
    }
  } else {
    for (int i = tid; i < 64 * 64; i += blockDim.x) {   // A: 64 rows x 64 K bytes, core matrices
      const int r = i / 64, k = i % 64;
      smem[(k / 16) * 1024 + r * 16 + (k % 16)] = code_a(cta, r, k);
    }
    for (int i = tid; i < 64 * 128; i += blockDim.x) {  // B: K = 64 rows (tokens), N = 128 bytes (dims), SW128
      const int k = i / 128, nb = i % 128;
      const int off = k * 128 + ((((nb >> 4) ^ (k & 7))) << 4) + (nb & 15);
      smem[8192 + off] = code_b(cta, nb, k);
    }
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bar1, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (mode == 1) {   // A codes into TMEM cols 256.. with the M = 64 layout
    const int t = lane & 15, h = lane >> 4;
    const int m = 16 * warp + t;
    for (int half = 0; half < 1; ++half) {
      uint32_t v[16];
      for (int c = 0; c < 16; ++c) {
        const int col = 16 * h + c;
        v[c] = (uint32_t)code_a(cta, m, 4 * col) | ((uint32_t)code_a(cta, m, 4 * col + 1) << 8) |
               ((uint32_t)code_a(cta, m, 4 * col + 2) << 16) | ((uint32_t)code_a(cta, m, 4 * col + 3) << 24);
      }
      st16(tm + ((uint32_t)(32 * warp) << 16) + 256u, v);
    }
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
  }
  if (mode == 4 && warp == 0) {   // a cta_group::1 MMA in the same kernel (each CTA, own data)
    const uint32_t a_s = smem_u32(smem), b_s = a_s + 8192;
    const uint64_t ad = make_smem_desc(a_s, 16, 1024, LAYOUT_SW128), bd = make_smem_desc(b_s, 16, 1024, LAYOUT_SW128);
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, 0;\n\t}" ::"r"(tm + 384u),
        "l"(ad), "l"(bd), "r"(make_idesc(0, 0, 0, 0, 64, 32))
        : "memory");
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(&bar1))
        : "memory");
    mbar_wait(&bar1, 0);
  }
  const uint32_t dbase = mode == 3 ? tm + (64u << 16) : tm;
  if (cta == 0 && warp == 0) {
    const uint32_t a_s = smem_u32(smem), b_s = a_s + 8192;
    if (mode != 2) {
      const uint32_t idesc = make_idesc(0, 0, 0, 0, 128, 64);
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t bd = make_smem_desc(b_s + 32 * kk, 16, 1024, LAYOUT_SW128);
        if (mode != 1) {
          const uint64_t ad = make_smem_desc(a_s + 32 * kk, 16, 1024, LAYOUT_SW128);
          asm volatile(
              "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
              "@e tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(dbase),
              "l"(ad), "l"(bd), "r"(idesc), "r"(kk)
              : "memory");
        } else {
          asm volatile(
              "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
              "@e tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm),
              "r"(tm + 256u + 8u * kk), "l"(bd), "r"(idesc), "r"(kk)
              : "memory");
        }
      }
    } else {
      const uint32_t idesc = make_idesc(0, 0, 0, 1, 128, 256);
      for (int kk = 0; kk < 2; ++kk) {
        const uint64_t ad = make_smem_desc(a_s + 2048 * kk, 1024, 128, LAYOUT_NONE);
        const uint64_t bd = make_smem_desc(b_s + 4096 * kk, 8192, 1024, LAYOUT_SW128);
        asm volatile(
            "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
            "l"(ad), "l"(bd), "r"(idesc), "r"(kk)
            : "memory");
      }
    }
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
            smem_u32(&bar)),
        "h"((uint16_t)3)
        : "memory");
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  // dump 128 lanes x 256 cols of this CTA
  for (int c0 = 0; c0 < 512; c0 += 32) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(tm + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0, r);
    tmem_wait_ld();
    for (int j = 0; j < 32; ++j) dump[((size_t)cta * 128 + 32 * warp + lane) * 512 + c0 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512) : "memory");
  }
}

int main() {
  float* d;
  cudaMalloc(&d, 2 * 128 * 512 * 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  for (int mode = 0; mode < 5; ++mode) {
    cudaMemset(d, 0, 2 * 128 * 512 * 4);
    probe<<<2, 128, 32768>>>(d, mode);
    cudaError_t e = cudaDeviceSynchronize();
    printf("mode %d: %s\n", mode, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    std::vector<float> h(2 * 128 * 512);
    cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
    const int N = mode == 2 ? 256 : 64, K = mode == 2 ? 64 : 128, half = N / 2;
    // expected D[c][r][n] = sum_k A_c[r][k] * B[k][n]; B column n lives in CTA n / half, local n % half
    std::vector<double> ex(2 * 64 * N);
    for (int c = 0; c < 2; ++c)
      for (int r = 0; r < 64; ++r)
        for (int n = 0; n < N; ++n) {
          const int bc = n / half, nl = n % half;
          double s = 0;
          for (int k = 0; k < K; ++k) s += dec_e4m3(code_a(c, r, k)) * dec_e4m3(code_b(bc, nl, k));
          ex[(c * 64 + r) * N + n] = s;
        }
    // for every expected (c, r, n): where is it?  print a compact summary of row -> lane, n -> col
    int found = 0, ambiguous = 0, missing = 0, wrong_cta = 0;
    std::vector<int> lane_of(2 * 64, -1), col_ok(2 * 64, 1), colmap(2 * N, -1);
    for (int c = 0; c < 2; ++c)
      for (int r = 0; r < 64; ++r)
        for (int n = 0; n < N; ++n) {
          const double v = ex[(c * 64 + r) * N + n];
          int hits = 0, hl = -1, hc = -1, hcta = -1;
          for (int cc = 0; cc < 2; ++cc)
            for (int l = 0; l < 128; ++l)
              for (int col = 0; col < 256; ++col) {
                const double g = h[((size_t)cc * 128 + l) * 512 + col];
                if (fabs(g - v) <= 1e-6 * (1 + fabs(v))) { ++hits; hl = l; hc = col; hcta = cc; }
              }
          if (hits == 0) ++missing;
          else if (hits > 1) ++ambiguous;
          else {
            ++found;
            if (hcta != c) ++wrong_cta;
            if (n == 0) lane_of[c * 64 + r] = hl;
            if (r == 5) colmap[c * N + n] = hc;
            if (r == 5 && n == half) printf("  cta %d row 5 n=%d -> cta %d lane %d col %d\n", c, n, hcta, hl, hc);
            if (hc != n) col_ok[c * 64 + r] = 0;
          }
        }
    if (mode == 4) {   // the cta_group::1 M = 64 N = 32 K = 32 MMA at col 384 (M = 64 layout)
      int bad = 0;
      for (int c = 0; c < 2; ++c)
        for (int r = 0; r < 64; ++r)
          for (int n = 0; n < 32; ++n) {
            double v = 0;
            for (int k = 0; k < 32; ++k) v += dec_e4m3(code_a(c, r, k)) * dec_e4m3(code_b(c, n, k));
            const int ln = (r % 16) + 32 * (r / 16);
            const double g = h[((size_t)c * 128 + ln) * 512 + 384 + n];
            if (fabs(g - v) > 1e-6 * (1 + fabs(v))) ++bad;
          }
      printf("  mixed cta_group::1 MMA mismatches: %d of 4096\n", bad);
    }
    printf("  found %d ambiguous %d missing %d wrong_cta %d\n", found, ambiguous, missing, wrong_cta);
    for (int c = 0; c < 2; ++c) {
      printf("  cta %d row->lane:", c);
      for (int r = 0; r < 64; ++r) printf(" %d", lane_of[c * 64 + r]);
      int ok = 1;
      for (int r = 0; r < 64; ++r) ok &= col_ok[c * 64 + r];
      printf("\n  cta %d col == n for all rows: %d\n  cta %d row 5 n->col:", c, ok, c);
      for (int n = 0; n < N; ++n) printf(" %d", colmap[c * N + n]);
      printf("\n");
    }
  }
  return 0;
}
