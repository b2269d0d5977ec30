// a2-a9: absorbed-MLA FP8 decode with the reconstructed PV pipeline, sm_100a.
//
// Method (PAPER.md, arXiv 2602.10718): Eq.5 absorbed score, Eq.6
// pre-scaled RoPE alignment, scale fusion + block-wise dynamic P
// quantization + implicit dequantization, Algorithm 1
// with Appendix C's strictly monotonic accumulation order.
//
// B200 design: one persistent CTA per SM, one 64-row query-head
// tile per CTA (UMMA M = 64), split-KV over 64-token key blocks planned on the
// device, a 5-slot ring of KV blocks in SMEM.  Warp roles (16 warps; the SM
// schedulers prefer the highest eligible warp id, so latency-critical roles get
// the high ids):
//   warps 0-7    two accumulator warpgroups (O columns 0-255 / 256-511): the
//                scalar Alg.1 recurrence (m, sigma_p, l, gamma; steps 4, 8-10)
//                and O <- gamma O + T_n with O in REGISTERS (as Alg.1 keeps
//                o^L / o^R in registers), epilogue (fp32 split partials)
//   warp 8       TMA producer: per block 4 x 8 KB FP8 boxes + 8 KB BF16 RoPE box
//                (SWIZZLE_128B, row coordinate from the block table) + 256 B scales
//   warp 9       QK issuer (owns TMEM): 16 x kind::f8f6f4 (K=32) + 4 x kind::f16
//                (K=16) into ONE fp32 accumulator S (Eq.6 makes the domains agree)
//   warps 10, 11 PV_L / PV_R issuers: T = P'_n (SMEM, K-major) x V (the SAME
//                FP8 tile read MN-major: no transpose) into a 3-slot TMEM ring
//   warps 12-15  Q-quant prologue (Fused-Q-Quant), softmax, scale fusion, block
//                P quantization; thread = (head row, 32-token half)
// Why O lives in registers (measured, scripts/tmem_bench.cu): TMEM stores run at
// ~235 B/cycle/SM, so rescaling a 64 x 512 fp32 O in TMEM every block costs
// >= 550 cycles and serialises PV(n-1) -> rescale -> PV(n).
// Issue economy (measured, scripts/acc_bench.cu + ncu source counters): the
// accumulate step is issue-bound when it shares an SMSP with busy higher-priority
// warps, so the per-block instruction count is kept minimal: one elect per MMA
// block (single asm), u32 shared-window barrier addresses, packed f32x2 math,
// a branch-free first block (gamma = 0 on a zeroed O), E4M3 packing via F2FP
// merge, and the debug timeline compiled out of production builds.
// Each block's softmax is computed against its OWN max (the P' codes depend only
// on w / max_block(w)); the accumulator warps carry the running max.
// TMEM map: see t_slot_addr (lanes 0-15: S slots, the q_c codes, T slot 0; lanes 16-31:
// T slots 1 / 2).  PV half h = 2n + (0: L, 1: R) goes to T slot h % 3, so PV(n+1)
// overlaps the accumulation of block n.
// The same kernel templated on kBf is the BF16 baseline (NEXT-2, Variant<true>); the
// experimental CTA-pair kernels for 64 < rows <= 128 (mla_decode_pair_kernel,
// mla_decode_2sm_kernel) follow below it.
#include <atomic>
#include <mutex>

#include "decode_common.cuh"

namespace snapmla {

constexpr int kWarpAcc = 0;       // 0-3 accumulators, O cols 0-255; 4-7 cols 256-511
constexpr int kWarpTma = 8;       // 8     TMA producer
constexpr int kWarpQk = 9;        // 9     QK issuer, owns TMEM
constexpr int kWarpPv = 10;       // 10-11 PV_L / PV_R issuers
constexpr int kWarpSoftmax = 12;  // 12-15 softmax
// register budget (setmaxnreg; balanced per SMSP: 2 acc + 1 issue + 1 softmax warp each):
// 256 x 176 + 128 x 40 + 128 x 120 = 65,536 = 512 x 128 (launch)
constexpr uint32_t kRegsAcc = 176, kRegsIssue = 40, kRegsSoftmax = 120;
constexpr int kPSlots = 2;        // P' + stats ring depth (blocks)
constexpr int kSSlots = 2;        // S ring depth (TMEM)
constexpr uint32_t kKvTx = kBc * (kDc + 2 * kDr + 4);       // 41216 B per block
constexpr uint32_t kStage = 41984;                          // kKvTx rounded up to 1024 (FP8 KV slot)
constexpr uint32_t kOffQr = 0;                              // [64 rows x 128 B] SW128 (q_r / sigma_q, BF16)
constexpr uint32_t kOffP = 8192;                            // 2 P' slots (4 KB E4M3 / 8 KB BF16), K-major core matrices
constexpr uint32_t kOffScaleHi = 5 * 8192 + 144;            // sigma_K of tokens 32-63 (bank-shifted by 16 B)
// KV slots, barrier region and SMEM size per variant: Variant<kBf> below
static_assert(2 * 32 * kRegsAcc + 32 * kRegsIssue + 32 * kRegsSoftmax <= 4 * 32 * 128,
              "setmaxnreg budget per SMSP (launch: 4 warps x 128 registers)");

// instruction descriptors (M = 64)
constexpr uint32_t kIdescQk8 = make_idesc(0, 0, 0, 0, 64, 64);      // E4M3 x E4M3, both K-major
constexpr uint32_t kIdescQk16 = make_idesc(1, 1, 0, 0, 64, 64);     // BF16 x BF16
constexpr uint32_t kIdescPv = make_idesc(0, 0, 0, 1, 64, 256);      // P' K-major, V MN-major
constexpr uint32_t kIdescQkB = make_idesc(1, 1, 0, 0, 64, 64);      // BF16 variant: q content x K content
constexpr uint32_t kIdescPvB = make_idesc(1, 1, 0, 1, 64, 256);     // BF16 variant: P K-major, V MN-major
// FP8 single-CTA kernel, swapped PV (build knob SNAPMLA_SC_SWAPPV, default 0): T^T (dims x 64 heads) =
// V^T (MN-major) P'^T (K-major), M = 128 dims per tile -- half the M = 64 PV's tensor time.  Correct
// (the full -m gpu suite passes with it) and it lifts the power-capped clock of the LongCat line from
// ~1,220 to ~1,510 MHz, but it runs ~14% slower there: every accumulator thread then needs all 64
// rows' gammas per block (the recurrence moves to warp 11) and T^T has one TMEM slot per half
// (profiles/r2w_swapped_pv_ab_longcat.txt).
#ifndef SNAPMLA_SC_SWAPPV
#define SNAPMLA_SC_SWAPPV 0
#endif
constexpr uint32_t kIdescPvSw = make_idesc(0, 0, 1, 0, 128, 64);

struct Bars {
  uint64_t kv_full[5], kv_empty[5];             // TMA -> QK / PV_L + PV_R -> TMA (max over variants)
  uint64_t s_full[kSSlots], s_empty[kSSlots];   // QK -> softmax / softmax -> QK
  uint64_t p_full[kPSlots], p_empty[kPSlots];   // P' + stats: softmax -> PV, acc / PV_L + PV_R + acc -> softmax
  uint64_t t_full[3], t_free[3];                // T ring: PV -> WG / WG -> PV
  uint64_t q_full, q_free;                      // Q-quant prologue -> QK / QK of a unit done -> prologue
  uint64_t fin_full, fin_empty;                 // swapped PV: epilogue factors warp 11 -> accumulators
  uint64_t gam_full[4], gam_empty[4];           // swapped PV: gamma ring, warp 11 -> accumulators -> warp 11
  uint32_t tmem_base;
  float stat[kPSlots][3][64];         // per block and row: max(t) * c (log2 units), sigma_loc, l_loc
  alignas(16) float gam[4][64];       // swapped PV: gamma ring (see del)
  alignas(16) float del[4][64];       // swapped PV: O^T <- gamma O^T + delta T^T per row (head), ring of 4 blocks
  alignas(16) float skipw[4][4];                  // swapped PV: per block and softmax warp, 1 if some row is skipped (delta = 0)
  alignas(16) float fin[64];          // swapped PV: epilogue factor per row
};
static_assert(sizeof(Bars) <= 5120, "barrier region");
#define BAR(field) (bar0 + (uint32_t)offsetof(Bars, field))

// ------------------------------------------------------------------ plan (a3)
// One CTA.  cum[b] = sum_{b'<b} ceil(L_b'/64) (exclusive scan), total T.
// Groups of n_ht CTAs share a contiguous range of `per` key blocks; group g
// covers blocks [g*per, (g+1)*per) of the concatenated request sequence.
// first_req[g] = request holding block g*per.  Splits fall on 64-token block
// boundaries, so the result is split-invariant (oracle test
// test_block_aligned_split_plus_combine_equals_unsplit).
// Fused-Q-Quant (a2: "per-token scale calculation, mixed-precision conversion and Scale
// Domain Alignment ... into a single operation"), in the plan launch: CTAs 1.. of the plan grid, one
// warp per query row (b, h).  Lane l: content dims [16 l, 16 l + 16) -> 16 E4M3 codes (one 16-B
// store); lanes 0-7 also RoPE dims [8 l, 8 l + 8) -> q_r' = q_r / sigma_q in BF16 (Eq.6).
// sigma_q = max(amax / 448, 2^-24) (R2), IEEE division; codes = RNE(q / sigma_q) (Markstein).
__device__ __forceinline__ void q_quant_row(const __nv_bfloat16* __restrict__ q, int row, uint8_t* __restrict__ qc,
                                            __nv_bfloat16* __restrict__ qr, float* __restrict__ sq) {
  const int lane = threadIdx.x & 31;
  const uint4* qrow = reinterpret_cast<const uint4*>(q + (int64_t)row * kDqk);
  const uint4 v2[2] = {__ldg(qrow + 2 * lane), __ldg(qrow + 2 * lane + 1)};
  const uint4 vr = lane < 8 ? __ldg(qrow + 64 + lane) : make_uint4(0, 0, 0, 0);
  const __nv_bfloat162* a = reinterpret_cast<const __nv_bfloat162*>(v2);
  float amax = 0.f;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const float2 f = __bfloat1622float2(a[e]);
    amax = fmaxf(amax, fmaxf(fabsf(f.x), fabsf(f.y)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  const float s = fmaxf(__fdiv_rn(amax, 448.0f), kSigmaMin);
  const float rs = __frcp_rn(s);
  uint32_t wd[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 f0 = __bfloat1622float2(a[2 * e]), f1 = __bfloat1622float2(a[2 * e + 1]);
    const float2 d0 = div_by2(f0, s, rs), d1 = div_by2(f1, s, rs);
    wd[e] = cvt4_e4m3(d0.x, d0.y, d1.x, d1.y);
  }
  reinterpret_cast<uint4*>(qc + (int64_t)row * kDc)[lane] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
  if (lane < 8) {
    const __nv_bfloat162* r2 = reinterpret_cast<const __nv_bfloat162*>(&vr);
    uint32_t rw[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(r2[e]);
      __nv_bfloat162 o2 = __halves2bfloat162(__float2bfloat16_rn(div_by(f.x, s, rs)), __float2bfloat16_rn(div_by(f.y, s, rs)));
      rw[e] = *reinterpret_cast<uint32_t*>(&o2);
    }
    reinterpret_cast<uint4*>(qr + (int64_t)row * kDr)[lane] = make_uint4(rw[0], rw[1], rw[2], rw[3]);
  }
  if (lane == 0) sq[row] = s;
}

__global__ void __launch_bounds__(1024) plan_kernel(const int32_t* __restrict__ seq_lens, int batch, int num_heads,
                                                    int groups, int32_t* __restrict__ hdr,
                                                    int32_t* __restrict__ cum, int32_t* __restrict__ first_req,
                                                    int num_sms, const __nv_bfloat16* __restrict__ q,
                                                    uint8_t* __restrict__ qc, __nv_bfloat16* __restrict__ qr,
                                                    float* __restrict__ sq) {
  __shared__ int warp_sums[32];
  __shared__ int s_per;
  const int tid = threadIdx.x;
  pdl_launch_dependents();
  if (blockIdx.x > 0) {   // Fused-Q-Quant CTAs: 32 rows each (q is an input: no dependence on the append)
    const int row = (blockIdx.x - 1) * 32 + (tid >> 5);
    if (row < batch * num_heads) q_quant_row(q, row, qc, qr, sq);
    pdl_wait();
    return;
  }
  const int per_thr = (batch + 1023) / 1024;
  const int b0 = tid * per_thr;
  int local = 0;
  for (int i = 0; i < per_thr; ++i) {
    const int b = b0 + i;
    if (b < batch) {
      const int L = seq_lens[b];
      local += L > 0 ? (L + kBc - 1) / kBc : 0;
    }
  }
  // block exclusive scan of `local`
  const int lane = tid & 31, warp = tid >> 5;
  int incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = warp_sums[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += v;
    }
    warp_sums[lane] = w;   // inclusive
  }
  __syncthreads();
  int run = incl - local + (warp > 0 ? warp_sums[warp - 1] : 0);
  for (int i = 0; i < per_thr; ++i) {
    const int b = b0 + i;
    if (b < batch) {
      cum[b] = run;
      const int L = seq_lens[b];
      run += L > 0 ? (L + kBc - 1) / kBc : 0;
    }
  }
  if (tid == 1023) {
    const int total = warp_sums[31];
    cum[batch] = total;
    // at least kMinPer blocks per CTA group: a small problem spread one block per group writes (and
    // the combine reads) a 64-row fp32 partial per block -- more bytes than the block's KV itself
#ifndef SNAPMLA_MIN_PER
#define SNAPMLA_MIN_PER 8
#endif
    constexpr int kMinPer = SNAPMLA_MIN_PER;
    const int per = total > 0 ? max((total + groups - 1) / groups, kMinPer) : 1;
    s_per = per;
    hdr[H_TOTAL] = total;
    hdr[H_PER] = per;
    hdr[H_GROUPS] = groups;
    hdr[H_NHT] = (num_heads + kHeadTile - 1) / kHeadTile;
    hdr[H_BATCH] = batch;
    hdr[H_HEADS] = num_heads;
    hdr[H_SMS] = num_sms;   // the SM count the workspace layout was computed with (combine checks it)
  }
  __syncthreads();
  const int per = s_per;
  // first_req: group starts inside request b
  for (int i = 0; i < per_thr; ++i) {
    const int b = b0 + i;
    if (b >= batch) break;
    const int c0 = cum[b];
    const int L = seq_lens[b];
    const int c1 = c0 + (L > 0 ? (L + kBc - 1) / kBc : 0);
    for (int g = (c0 + per - 1) / per; g < groups && g * per < c1; ++g) first_req[g] = b;
  }
  // launched as a programmatic dependent of the append: complete only after it, so the
  // decode's griddepcontrol.wait (on this grid) also orders its cache reads after the append
  pdl_wait();
}

// ------------------------------------------------------------- decode kernel
// One QK block into S (TMEM): 16 x kind::f8f6f4 (K = 32) over the 512 content dims,
// then 4 x kind::f16 (K = 16) over the 64 RoPE dims, accumulating into the same S;
// commit to `bar`.  One elect for the whole block.  Descriptor start addresses
// advance in 16-byte units: content step kk at byte (kk / 4) * 8192 + (kk % 4) * 32.
#define SNAPMLA_QK8(ta, bo, acc)                                                               \
  "add.u32 t, %1, " #ta ";\n\tadd.s64 b, %2, " #bo ";\n\t"                                     \
  "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [t], b, %3, " acc ";\n\t"
#define SNAPMLA_QK16(ao)                                                                       \
  "add.s64 a, %4, " #ao ";\n\tadd.s64 b, %5, " #ao ";\n\t"                                     \
  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %6, pt;\n\t"
// The content A operand (q_c codes) lives in TMEM: step kk reads columns tQ + 8 kk.
__device__ __forceinline__ void qk_issue(uint32_t dS, uint32_t tQ, uint64_t dK, uint64_t dQr, uint64_t dKr,
                                         uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e, pf, pt;\n\t.reg .b64 a, b;\n\t.reg .b32 z, t;\n\t"
      "mov.b32 z, 0;\n\tsetp.ne.b32 pf, z, 0;\n\tsetp.eq.b32 pt, z, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      SNAPMLA_QK8(0, 0, "pf") SNAPMLA_QK8(8, 2, "pt") SNAPMLA_QK8(16, 4, "pt") SNAPMLA_QK8(24, 6, "pt")
      SNAPMLA_QK8(32, 512, "pt") SNAPMLA_QK8(40, 514, "pt") SNAPMLA_QK8(48, 516, "pt") SNAPMLA_QK8(56, 518, "pt")
      SNAPMLA_QK8(64, 1024, "pt") SNAPMLA_QK8(72, 1026, "pt") SNAPMLA_QK8(80, 1028, "pt") SNAPMLA_QK8(88, 1030, "pt")
      SNAPMLA_QK8(96, 1536, "pt") SNAPMLA_QK8(104, 1538, "pt") SNAPMLA_QK8(112, 1540, "pt") SNAPMLA_QK8(120, 1542, "pt")
      SNAPMLA_QK16(0) SNAPMLA_QK16(2) SNAPMLA_QK16(4) SNAPMLA_QK16(6)
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%7];\n\t}"
      ::"r"(dS), "r"(tQ), "l"(dK), "r"(kIdescQk8), "l"(dQr), "l"(dKr), "r"(kIdescQk16), "r"(bar)
      : "memory");
}

// One PV half: T = P' (64 x 64 tokens, K-major) x V (64 tokens x 256 dims, MN-major),
// 2 x kind::f8f6f4 (K = 32); commit to t_full, p_empty and kv_empty.
__device__ __forceinline__ void pv_issue(uint32_t dT, uint64_t dP, uint64_t dV, uint32_t bar_t, uint32_t bar_p,
                                         uint32_t bar_kv) {
  asm volatile(
      "{\n\t.reg .pred e, pf, pt;\n\t.reg .b64 a, b;\n\t.reg .b32 z;\n\t"
      "mov.b32 z, 0;\n\tsetp.ne.b32 pf, z, 0;\n\tsetp.eq.b32 pt, z, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
#ifndef SNAPMLA_SOL_NOPV
      "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, pf;\n\t"
      "add.s64 a, %1, 128;\n\tadd.s64 b, %2, 256;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], a, b, %3, pt;\n\t"
#endif
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%4];\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%6];\n\t}"
      ::"r"(dT), "l"(dP), "l"(dV), "r"(kIdescPv), "r"(bar_t), "r"(bar_p), "r"(bar_kv)
      : "memory");
}

// One swapped PV half (dim tiles 2 half, 2 half + 1): 2 tiles x 2 K-steps of M = 128, N = 64, K = 32;
// tile t at TMEM columns dT + 64 t; commit to t_full, p_empty and kv_empty.
__device__ __forceinline__ void pv_issue_swt(uint32_t dT, uint64_t dV, uint64_t dP, uint32_t bar_t, uint32_t bar_p,
                                             uint32_t bar_kv) {
  asm volatile(
      "{\n\t.reg .pred e, pf, pt;\n\t.reg .b64 a, b;\n\t.reg .b32 z, d;\n\t"
      "mov.b32 z, 0;\n\tsetp.ne.b32 pf, z, 0;\n\tsetp.eq.b32 pt, z, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, pf;\n\t"
      "add.s64 a, %1, 256;\n\tadd.s64 b, %2, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], a, b, %3, pt;\n\t"
      "add.u32 d, %0, 64;\n\tadd.s64 a, %1, 512;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [d], a, %2, %3, pf;\n\t"
      "add.s64 a, %1, 768;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [d], a, b, %3, pt;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%4];\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%6];\n\t}"
      ::"r"(dT), "l"(dV), "l"(dP), "r"(kIdescPvSw), "r"(bar_t), "r"(bar_p), "r"(bar_kv)
      : "memory");
}

// TMEM map (M = 64 data-path layout: row m at lane (m % 16) + 32 (m / 16), +16 for the
// upper half-subpartitions).  Lanes 0-15: S slots 0 / 1 (cols 0 / 64), the Q content codes
// (cols 128-255, the QK A operand: A-in-TMEM must start at lane 0, scripts/tmem_a_check.cu),
// T slot 0 (cols 256-511).  Lanes 16-31: T slots 1 / 2 (cols 0 / 256).
constexpr uint32_t kTmemQ = 128;
__device__ __forceinline__ uint32_t t_slot_addr(uint32_t tmem, uint32_t s) {
  return tmem + (s == 0 ? 256u : (16u << 16) + 256u * (s - 1));
}

// Per-variant layout: FP8 (the method) and the BF16 baseline variant (NEXT-2, same skeleton,
// unquantized cache / Q / P).  BF16: 8 content boxes + RoPE = 72 KB per block (two slots fit),
// q content (1 KB per row) in TMEM columns 128-383 of lanes 0-15, so only the two T half-slots
// of lanes 16-31 remain; P' is BF16 (8 KB per slot).
#ifndef SNAPMLA_SPF
#define SNAPMLA_SPF 1   // FP8 kernel: S(n+1) TMEM load issued before block n's P' stores
#endif
template <bool kBf> struct Variant;
template <> struct Variant<false> {
  static constexpr int kSlots = 5, kTSlots = 3, kBoxes = 4;
  static constexpr uint32_t kTx = kKvTx, kStage = 41984, kPBytes = 4096, kOffKv = 16384;
  static constexpr uint32_t kOffBar = kOffKv + kSlots * kStage, kSmem = kOffBar + 5120 + 1024;
  static __device__ __forceinline__ uint32_t t_slot(uint32_t tmem, uint32_t s) { return t_slot_addr(tmem, s); }
};
template <> struct Variant<true> {
  static constexpr int kSlots = 2, kTSlots = 2, kBoxes = 8;
  static constexpr uint32_t kTx = 9 * kBoxBytes, kStage = 9 * kBoxBytes, kPBytes = 8192, kOffKv = 8192 + 2 * 8192;
  static constexpr uint32_t kOffBar = kOffKv + kSlots * kStage, kSmem = kOffBar + 5120 + 1024;
  static __device__ __forceinline__ uint32_t t_slot(uint32_t tmem, uint32_t s) {
    return tmem + (16u << 16) + 256u * s;
  }
};
static_assert(Variant<false>::kSmem <= 232448 && Variant<true>::kSmem <= 232448, "shared memory budget");

// BF16 variant QK: 32 x kind::f16 (K = 16) over the content (A = q in TMEM, columns tQ + 8 kk)
// + 4 x kind::f16 over the RoPE, one accumulator; commit to `bar`.
#define SNAPMLA_QKB(ta, bo, acc)                                                               \
  "add.u32 t, %1, " #ta ";\n\tadd.s64 b, %2, " #bo ";\n\t"                                     \
  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t], b, %3, " acc ";\n\t"
__device__ __forceinline__ void qk_issue_bf16(uint32_t dS, uint32_t tQ, uint64_t dK, uint64_t dQr, uint64_t dKr,
                                              uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e, pf, pt;\n\t.reg .b64 a, b;\n\t.reg .b32 z, t;\n\t"
      "mov.b32 z, 0;\n\tsetp.ne.b32 pf, z, 0;\n\tsetp.eq.b32 pt, z, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      SNAPMLA_QKB(0, 0, "pf") SNAPMLA_QKB(8, 2, "pt") SNAPMLA_QKB(16, 4, "pt") SNAPMLA_QKB(24, 6, "pt")
      SNAPMLA_QKB(32, 512, "pt") SNAPMLA_QKB(40, 514, "pt") SNAPMLA_QKB(48, 516, "pt") SNAPMLA_QKB(56, 518, "pt")
      SNAPMLA_QKB(64, 1024, "pt") SNAPMLA_QKB(72, 1026, "pt") SNAPMLA_QKB(80, 1028, "pt") SNAPMLA_QKB(88, 1030, "pt")
      SNAPMLA_QKB(96, 1536, "pt") SNAPMLA_QKB(104, 1538, "pt") SNAPMLA_QKB(112, 1540, "pt") SNAPMLA_QKB(120, 1542, "pt")
      SNAPMLA_QKB(128, 2048, "pt") SNAPMLA_QKB(136, 2050, "pt") SNAPMLA_QKB(144, 2052, "pt") SNAPMLA_QKB(152, 2054, "pt")
      SNAPMLA_QKB(160, 2560, "pt") SNAPMLA_QKB(168, 2562, "pt") SNAPMLA_QKB(176, 2564, "pt") SNAPMLA_QKB(184, 2566, "pt")
      SNAPMLA_QKB(192, 3072, "pt") SNAPMLA_QKB(200, 3074, "pt") SNAPMLA_QKB(208, 3076, "pt") SNAPMLA_QKB(216, 3078, "pt")
      SNAPMLA_QKB(224, 3584, "pt") SNAPMLA_QKB(232, 3586, "pt") SNAPMLA_QKB(240, 3588, "pt") SNAPMLA_QKB(248, 3590, "pt")
      SNAPMLA_QK16(0) SNAPMLA_QK16(2) SNAPMLA_QK16(4) SNAPMLA_QK16(6)
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%7];\n\t}"
      ::"r"(dS), "r"(tQ), "l"(dK), "r"(kIdescQkB), "l"(dQr), "l"(dKr), "r"(kIdescQk16), "r"(bar)
      : "memory");
}

// BF16 variant PV half: T = P (64 x 64 tokens, BF16 K-major) x V (64 tokens x 256 dims, BF16
// MN-major, 4 boxes of 64 dims), 4 x kind::f16 (K = 16: +2048 B in both operands per step).
__device__ __forceinline__ void pv_issue_bf16(uint32_t dT, uint64_t dP, uint64_t dV, uint32_t bar_t, uint32_t bar_p,
                                              uint32_t bar_kv) {
  asm volatile(
      "{\n\t.reg .pred e, pf, pt;\n\t.reg .b64 a, b;\n\t.reg .b32 z;\n\t"
      "mov.b32 z, 0;\n\tsetp.ne.b32 pf, z, 0;\n\tsetp.eq.b32 pt, z, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, pf;\n\t"
      "add.s64 a, %1, 128;\n\tadd.s64 b, %2, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, pt;\n\t"
      "add.s64 a, %1, 256;\n\tadd.s64 b, %2, 256;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, pt;\n\t"
      "add.s64 a, %1, 384;\n\tadd.s64 b, %2, 384;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, pt;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%4];\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%6];\n\t}"
      ::"r"(dT), "l"(dP), "l"(dV), "r"(kIdescPvB), "r"(bar_t), "r"(bar_p), "r"(bar_kv)
      : "memory");
}

template <bool kBf>
__global__ void __launch_bounds__(kThreads, 1)
    mla_decode_kernel(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_rope,
                      const DecodeParams p) {
  using V = Variant<kBf>;
  constexpr bool kSwPv = !kBf && SNAPMLA_SC_SWAPPV;   // FP8: PV with swapped operands (T^T, M = 128 dims)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t bar0 = sbase + V::kOffBar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) TRACE(TR_C2, 250u);   // prologue stamps (trace builds): kernel entry

  // ---- setup overlaps the plan kernel (programmatic dependent launch)
  if (threadIdx.x == 0) {
    for (int i = 0; i < V::kSlots; ++i) {
      mbar_init(BAR(kv_full) + 8 * i, 1);
      mbar_init(BAR(kv_empty) + 8 * i, 2);
    }
    for (int i = 0; i < kPSlots; ++i) {
      mbar_init(BAR(p_full) + 8 * i, 4 * kArriveMul);
      // PV_L + PV_R commits, and the stats readers: the 8 accumulator warps (swapped PV: warp 11)
      mbar_init(BAR(p_empty) + 8 * i, kSwPv ? 2 + 1 : 2 + 8 * kArriveMul);
    }
    for (int i = 0; i < kSSlots; ++i) {
      mbar_init(BAR(s_full) + 8 * i, 1);
      mbar_init(BAR(s_empty) + 8 * i, 4);
    }
    for (int i = 0; i < V::kTSlots; ++i) {
      mbar_init(BAR(t_full) + 8 * i, 1);
      mbar_init(BAR(t_free) + 8 * i, 4);
    }
    mbar_init(BAR(q_full), 4);
    mbar_init(BAR(q_free), 1);
    mbar_init(BAR(fin_full), 1);   // swapped PV: warp 11 (the recurrence warp)
    mbar_init(BAR(fin_empty), 8);  // swapped PV: the 8 accumulator warps
    for (int i = 0; i < 4; ++i) {
      mbar_init(BAR(gam_full) + 8 * i, 1);
      mbar_init(BAR(gam_empty) + 8 * i, 8);
    }
    fence_barrier_init();
  }
  if (warp == kWarpTma && lane == 0) {
    tma_prefetch_desc(&tm_kv);
    tma_prefetch_desc(&tm_rope);
  }
  if (warp == kWarpQk) tmem_alloc(BAR(tmem_base), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = lds_u32(BAR(tmem_base));
  const uint32_t tmem_S = tmem;                       // lanes 0-15 (+32k): S slot s at cols 64 s

  if (threadIdx.x == 0) TRACE(TR_C2, 251u);   // setup done
  pdl_wait();   // plan (and the appends before it) visible from here on
  pdl_launch_dependents();   // the combine may be scheduled as CTAs retire (it waits for completion)
  if (threadIdx.x == 0) TRACE(TR_C2, 252u);   // plan visible
  const int ht = blockIdx.x % p.n_ht;
  const int g = blockIdx.x / p.n_ht;
  const int per = p.ws_hdr[H_PER], total = p.ws_hdr[H_TOTAL], groups = p.ws_hdr[H_GROUPS];
  const int lo = g * per;
  const bool has_work = g < groups && lo < total;
  const int hi = min(total, lo + per);
#ifdef SNAPMLA_TRACE
  if (p.trace != nullptr && threadIdx.x == 0) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(gt));
    p.trace[TR_NEV * kTraceN + 2 * blockIdx.x] = gt;
  }
#endif

  UnitIter it{p.cum, lo, hi, g, has_work ? __ldg(p.first_req + g) : 0, has_work ? p.batch : 0};
  Unit u;

  if (warp >= kWarpTma && warp < kWarpSoftmax) {
    regs_dec<kRegsIssue>();
    if (warp == kWarpTma) {
      // ============================ TMA producer ============================
      if (lane == 0) {
        const uint64_t pol = l2_policy_evict_first();
        uint32_t n = 0;
        while (it.next(u)) {
          const int32_t* bt = p.block_table + (int64_t)u.b * p.max_pages;
          prefetch_block_table(bt, u.k0, u.k1);
          for (int j = u.k0; j < u.k1; ++j, ++n) {
            const uint32_t st = n % V::kSlots;
            mbar_wait_backoff(BAR(kv_empty) + 8 * st, ((n / V::kSlots) & 1) ^ 1);
            TRACE(TR_TMA, n);
            const int row = __ldg(bt + j) * kPage;
            const uint32_t dst = sbase + V::kOffKv + st * V::kStage;
            const uint32_t full = BAR(kv_full) + 8 * st;
            mbar_arrive_expect_tx(full, V::kTx);
#pragma unroll
            for (int c = 0; c < V::kBoxes; ++c)   // content boxes of 128 B (128 E4M3 / 64 BF16 values) x 64 tokens
              tma_load_2d(dst + c * kBoxBytes, &tm_kv, full, c * (kBf ? 64 : 128), row, pol);
            tma_load_2d(dst + V::kBoxes * kBoxBytes, &tm_rope, full, 0, row, pol);
            if constexpr (!kBf) {
              bulk_load(dst + 5 * kBoxBytes, p.kv_scale + (int64_t)row, 128, full, pol);
              bulk_load(dst + kOffScaleHi, p.kv_scale + (int64_t)row + 32, 128, full, pol);
            }
          }
        }
      }
    } else if (warp == kWarpQk) {
      // ================================ QK issuer ================================
      const uint64_t dQr = make_smem_desc(sbase + kOffQr, 16, 1024, LAYOUT_SW128);
      uint32_t n = 0, unit = 0;
      while (it.next(u)) {
        mbar_wait_sleep(BAR(q_full), unit & 1);
        if (lane == 0 && unit == 0) TRACE(TR_C2, 254u);   // QK warp: q_full seen
        for (int j = u.k0; j < u.k1; ++j, ++n) {
          const uint32_t st = n % V::kSlots, ss = n % kSSlots;
          mbar_wait_sleep(BAR(kv_full) + 8 * st, (n / V::kSlots) & 1);
          mbar_wait_sleep(BAR(s_empty) + 8 * ss, ((n / kSSlots) & 1) ^ 1);
          tc_fence_after();
          if (lane == 0) TRACE(TR_QK, n);
          const uint32_t kv = sbase + V::kOffKv + st * V::kStage;
          if constexpr (kBf)
            qk_issue_bf16(tmem_S + 64 * ss, tmem + kTmemQ, make_smem_desc(kv, 16, 1024, LAYOUT_SW128), dQr,
                          make_smem_desc(kv + 8 * kBoxBytes, 16, 1024, LAYOUT_SW128), BAR(s_full) + 8 * ss);
          else
            qk_issue(tmem_S + 64 * ss, tmem + kTmemQ, make_smem_desc(kv, 16, 1024, LAYOUT_SW128), dQr,
                     make_smem_desc(kv + 4 * kBoxBytes, 16, 1024, LAYOUT_SW128), BAR(s_full) + 8 * ss);
        }
        mma_commit_ws(BAR(q_free));   // Q (TMEM + SMEM) reusable once this unit's QK MMAs completed
        ++unit;
      }
    } else {
      // =============================== PV_L / PV_R ===============================
      const uint32_t half = warp - kWarpPv;
      uint32_t n = 0;
      // swapped PV: warp 11 also runs the per-row recurrence (rows lane, lane + 32)
      float rc_m_ref[2] = {-INFINITY, -INFINITY}, rc_m_O[2] = {0.f, 0.f}, rc_sig_O[2] = {1.f, 1.f}, rc_l[2] = {0.f, 0.f};
      uint32_t rc_unit = 0;
      while (it.next(u)) {
        for (int j = u.k0; j < u.k1; ++j, ++n) {
          const uint32_t st = n % V::kSlots, ps = n % kPSlots;
          if constexpr (kSwPv) {   // T^T half `half` (dims 256 half + [0, 256)) -> TMEM cols 256 + 128 half, all lanes
            mbar_wait_sleep(BAR(p_full) + 8 * ps, (n / kPSlots) & 1);
            if (half == 1) {
              // Alg.1 steps 4, 8-10 for rows lane and lane + 32 (as the accumulators of the M = 64 PV
              // run them per row): gamma / delta into a 4-block ring for the accumulators, whose
              // threads each need all 64 rows' factors
              const uint32_t gs = n % 4;
              if (n >= 4) mbar_wait_sleep(BAR(gam_empty) + 8 * gs, (n / 4 - 1) & 1);
              bool sk = false;
#pragma unroll
              for (int i = 0; i < 2; ++i) {
                const int row = lane + 32 * i;
                const uint32_t sa = BAR(stat) + 4 * row + ps * (3 * 64 * 4);
                const float mb = lds_f32(sa), sb = lds_f32(sa + 256), lb = lds_f32(sa + 512);
                const float m_new = fmaxf(rc_m_ref[i], mb);
                const bool first = j == u.k0;
                const bool skip = !first && ((mb == -INFINITY) || (mb < m_new - 64.f));
                float gamma = 0.f, delta = 1.f;
                if (first) {
                  rc_m_O[i] = mb;
                  rc_sig_O[i] = sb;
                  rc_l[i] = lb;
                  rc_m_ref[i] = mb;
                } else if (!skip) {
                  gamma = ex2_approx(rc_m_O[i] - mb) * __fdividef(rc_sig_O[i], sb);
                  rc_l[i] = rc_l[i] * ex2_approx(rc_m_ref[i] - m_new) + lb * ex2_approx(mb - m_new);
                  rc_m_ref[i] = m_new;
                  rc_m_O[i] = mb;
                  rc_sig_O[i] = sb;
                } else {
                  gamma = 1.f;
                  delta = 0.f;
                }
                sts_f32(BAR(gam) + 4 * (gs * 64 + row), gamma);
                sts_f32(BAR(del) + 4 * (gs * 64 + row), delta);
                sk |= skip;
              }
              const unsigned any = __ballot_sync(0xffffffffu, sk);
              if (lane < 4) sts_f32(BAR(skipw) + 4 * (gs * 4 + lane), (lane == 0 && any != 0u) ? 1.f : 0.f);
              __syncwarp();
              if (lane == 0) {
                mbar_arrive(BAR(gam_full) + 8 * gs);
                mbar_arrive(BAR(p_empty) + 8 * ps);   // stats of this slot consumed
              }
              if (j + 1 == u.k1) {   // epilogue factors (a9): o = sigma_O 2^{m_O - m_ref} O / l, natural-log LSE
                if (rc_unit > 0) mbar_wait_sleep(BAR(fin_empty), (rc_unit - 1) & 1);
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                  const int row = lane + 32 * i;
                  sts_f32(BAR(fin) + 4 * row, rc_l[i] > 0.f ? rc_sig_O[i] * ex2_approx(rc_m_O[i] - rc_m_ref[i]) / rc_l[i] : 0.f);
                  if (ht * kHeadTile + row < p.num_heads)
                    p.lse_part[((int64_t)u.slot * p.n_ht + ht) * kHeadTile + row] =
                        rc_l[i] > 0.f ? (rc_m_ref[i] + log2f(rc_l[i])) * 0.69314718055994531f : -INFINITY;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(BAR(fin_full));
                ++rc_unit;
              }
            }
            if (n >= 1) mbar_wait_sleep(BAR(t_free) + 8 * half, (n - 1) & 1);
            tc_fence_after();
            const uint32_t kvb = sbase + V::kOffKv + st * V::kStage + 2 * half * kBoxBytes;
            if (lane == 0) TRACE(half == 0 ? TR_PVL : TR_PVR, n);
            pv_issue_swt(tmem + 256 + 128 * half, make_smem_desc(kvb, kBoxBytes, 1024, LAYOUT_SW128),
                         make_smem_desc(sbase + kOffP + ps * V::kPBytes, 1024, 128, LAYOUT_NONE),
                         BAR(t_full) + 8 * half, BAR(p_empty) + 8 * ps, BAR(kv_empty) + 8 * st);
            continue;
          }
          const uint32_t h = 2 * n + half, ts = h % V::kTSlots;
          mbar_wait_sleep(BAR(p_full) + 8 * ps, (n / kPSlots) & 1);                  // P'(n) in SMEM
          if (h >= V::kTSlots) mbar_wait_sleep(BAR(t_free) + 8 * ts, (h / V::kTSlots - 1) & 1);   // slot read
          tc_fence_after();
          if (lane == 0) TRACE(half == 0 ? TR_PVL : TR_PVR, n);
          const uint32_t pA = sbase + kOffP + ps * V::kPBytes;
          const uint32_t vb = sbase + V::kOffKv + st * V::kStage + (V::kBoxes / 2 * half) * kBoxBytes;
          if constexpr (kBf)
            pv_issue_bf16(V::t_slot(tmem, ts), make_smem_desc(pA, 1024, 128, LAYOUT_NONE),
                          make_smem_desc(vb, kBoxBytes, 1024, LAYOUT_SW128), BAR(t_full) + 8 * ts,
                          BAR(p_empty) + 8 * ps, BAR(kv_empty) + 8 * st);
          else
            pv_issue(V::t_slot(tmem, ts), make_smem_desc(pA, 1024, 128, LAYOUT_NONE),
                     make_smem_desc(vb, kBoxBytes, 1024, LAYOUT_SW128), BAR(t_full) + 8 * ts,
                     BAR(p_empty) + 8 * ps, BAR(kv_empty) + 8 * st);
        }
      }
    }
  } else if (warp >= kWarpSoftmax) {
    if constexpr (kRegsSoftmax > 128) regs_inc<kRegsSoftmax>();   // launch: 128 per thread
    else regs_dec<kRegsSoftmax>();
    // ======= softmax / scale fusion / P quantization: thread = (row, 32-token half) =======
    const int k = warp & 3;                  // TMEM subpartition of this warp
    const int t = lane & 15, hh = lane >> 4; // row-in-quarter, 32-token half
    const int r = 16 * k + t;                // query-head row inside the tile
    const int head = ht * kHeadTile + r;
    const bool row_ok = head < p.num_heads;
    const uint32_t lane_off = (uint32_t)(32 * k) << 16;
    const uint32_t stat0 = BAR(stat) + 4 * r;
    uint32_t n = 0, unit = 0;
    while (it.next(u)) {
      // ---------------- Fused-Q-Quant prologue (a2): row r, content half hh
      if (unit > 0) mbar_wait(BAR(q_free), (unit - 1) & 1, 11, unit);   // QK of the previous unit done
      float c_row;
      if constexpr (kBf) {
        // BF16 variant (NEXT-2): the unquantized q row goes to TMEM / SMEM as is; c = scale * log2(e)
        const uint4* qrow = reinterpret_cast<const uint4*>(p.q + ((int64_t)u.b * p.num_heads + head) * kDqk);
        c_row = p.scale_log2;
        // content elements [256 hh, 256 hh + 256) = TMEM columns kTmemQ + 128 hh + [0, 128), 2 per column
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint32_t qa[32];
#pragma unroll
          for (int g8 = 0; g8 < 8; ++g8) {
            const uint4 v = row_ok ? __ldg(qrow + 32 * hh + 8 * i + g8) : make_uint4(0, 0, 0, 0);
            qa[4 * g8] = v.x;
            qa[4 * g8 + 1] = v.y;
            qa[4 * g8 + 2] = v.z;
            qa[4 * g8 + 3] = v.w;
          }
          tmem_st_16x32bx2_x32<128>(tmem + lane_off + kTmemQ + 32 * i, qa);
        }
        tmem_wait_st();
#pragma unroll
        for (int gch = 0; gch < 4; ++gch) {
          const int c = 4 * hh + gch;
          const uint4 v = row_ok ? __ldg(qrow + 64 + c) : make_uint4(0, 0, 0, 0);
          sts_u4(sbase + kOffQr + r * 128 + ((c ^ (r & 7)) << 4), v.x, v.y, v.z, v.w);
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(BAR(q_full));
      } else {
        if (threadIdx.x == 32 * kWarpSoftmax && unit == 0) TRACE(TR_C2, 245u);   // Q load start
        // Fused-Q-Quant ran in the plan launch (q_quant_row): load this row's codes (content half hh)
        // into TMEM columns kTmemQ + 64 hh + [0, 64) (the QK A operand), q_r' into its SW128 SMEM row
        const int64_t qrow_i = (int64_t)u.b * p.num_heads + head;
        const uint4* qcr = reinterpret_cast<const uint4*>(p.qc + qrow_i * kDc) + 16 * hh;
        c_row = (row_ok ? __ldg(p.sq + qrow_i) : 1.f) * p.scale_log2;
#pragma unroll
        for (int half32 = 0; half32 < 2; ++half32) {
          uint32_t qa[32];
#pragma unroll
          for (int g8 = 0; g8 < 8; ++g8) {
            const uint4 v = row_ok ? __ldg(qcr + 8 * half32 + g8) : make_uint4(0, 0, 0, 0);
            qa[4 * g8] = v.x;
            qa[4 * g8 + 1] = v.y;
            qa[4 * g8 + 2] = v.z;
            qa[4 * g8 + 3] = v.w;
          }
          tmem_st_16x32bx2_x32<64>(tmem + lane_off + kTmemQ + 32 * half32, qa);
        }
        const uint4* qrr = reinterpret_cast<const uint4*>(p.qr + qrow_i * kDr);
#pragma unroll
        for (int gch = 0; gch < 4; ++gch) {
          const int c = 4 * hh + gch;   // 16-byte chunk of the 128-B RoPE row
          const uint4 v = row_ok ? __ldg(qrr + c) : make_uint4(0, 0, 0, 0);
          sts_u4(sbase + kOffQr + r * 128 + ((c ^ (r & 7)) << 4), v.x, v.y, v.z, v.w);
        }
        tmem_wait_st();
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(BAR(q_full));
        if (threadIdx.x == 32 * kWarpSoftmax && unit == 0) TRACE(TR_C2, 253u);   // Q-quant done (warp 12)
      }

      // visible keys of this row: query token t = head / heads of q_len sees the cache
      // up to its own position, L - (q_len - 1 - t) (causal MTP, reading R25)
      const int L = __ldg(p.seq_lens + u.b) - (p.q_len - 1 - head / p.heads);
      // S(n) is loaded from TMEM one block ahead: the load of S(n+1) is issued before
      // block n's P' / stats stores, fence and arrive, which hide its latency.
      float tt[32];
      for (int j = u.k0; j < u.k1; ++j, ++n) {
        const uint32_t st = n % V::kSlots, ss = n % kSSlots, ps = n % kPSlots;
        if (j == u.k0 || kBf || !SNAPMLA_SPF) {
          mbar_wait(BAR(s_full) + 8 * ss, (n / kSSlots) & 1, 7, n);
          tc_fence_after();
          tmem_ld_16x32bx2_x32<32>(tmem_S + lane_off + 64 * ss, *reinterpret_cast<uint32_t(*)[32]>(tt));
        }
        if (threadIdx.x == 32 * kWarpSoftmax) TRACE(TR_SM_IN, n);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(BAR(s_empty) + 8 * ss);
        if (threadIdx.x == 32 * kWarpSoftmax) TRACE(TR_S1, n);
        // sigma_K of my 32 tokens (from the TMA'd slot)
        const uint32_t sk = sbase + V::kOffKv + st * V::kStage + (hh ? kOffScaleHi : 5 * kBoxBytes);
        const int nvalid = L - (j * kBc + 32 * hh);   // tokens of my half inside the sequence
        float4 skv[8];                                                 // sigma_K of my 32 tokens, kept
#pragma unroll
        for (int e = 0; e < 8; ++e) skv[e] = kBf ? make_float4(1.f, 1.f, 1.f, 1.f) : lds_f4(sk + 16 * e);
#pragma unroll
        for (int e = 0; e < 32; e += 4) {                              // Alg.1 step 3 (descale)
          if constexpr (kBf) break;
          const float4 s4 = skv[e / 4];
          const float2 a = __fmul2_rn(make_float2(tt[e], tt[e + 1]), make_float2(s4.x, s4.y));
          const float2 b = __fmul2_rn(make_float2(tt[e + 2], tt[e + 3]), make_float2(s4.z, s4.w));
          tt[e] = a.x;
          tt[e + 1] = a.y;
          tt[e + 2] = b.x;
          tt[e + 3] = b.y;
        }
        if (nvalid < 32) {                                             // ragged tail block: mask (R19)
#pragma unroll
          for (int e = 0; e < 32; ++e) tt[e] = e < nvalid ? tt[e] : -INFINITY;
        }
        float mx0 = fmaxf(fmaxf(tt[0], tt[1]), tt[2]), mx1 = fmaxf(fmaxf(tt[3], tt[4]), tt[5]);
#pragma unroll
        for (int e = 6; e < 30; e += 4) {
          mx0 = fmaxf(fmaxf(mx0, tt[e]), tt[e + 1]);
          mx1 = fmaxf(fmaxf(mx1, tt[e + 2]), tt[e + 3]);
        }
        float mx = fmaxf(fmaxf(mx0, mx1), fmaxf(tt[30], tt[31]));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));          // block max of t (local m)
        if (threadIdx.x == 32 * kWarpSoftmax) TRACE(TR_S2, n);
        const float mc = mx == -INFINITY ? 0.f : mx * c_row;            // fully masked row block (MTP)
        float2 ls0 = make_float2(0.f, 0.f), ls1 = make_float2(0.f, 0.f);
        float mb0 = 0.f, mb1 = 0.f;
#pragma unroll
        for (int e = 0; e < 32; e += 4) {
          const float4 s4 = skv[e / 4];
          const float2 e0 = __ffma2_rn(make_float2(tt[e], tt[e + 1]), make_float2(c_row, c_row), make_float2(-mc, -mc));
          const float2 e1 = __ffma2_rn(make_float2(tt[e + 2], tt[e + 3]), make_float2(c_row, c_row), make_float2(-mc, -mc));
          const float2 p0 = make_float2(ex2_approx(e0.x), ex2_approx(e0.y));   // step 5 (block reference)
          const float2 p1 = make_float2(ex2_approx(e1.x), ex2_approx(e1.y));
          const float2 w0 = kBf ? p0 : __fmul2_rn(p0, make_float2(s4.x, s4.y));   // step 6: p * sigma_K
          const float2 w1 = kBf ? p1 : __fmul2_rn(p1, make_float2(s4.z, s4.w));
          ls0 = __fadd2_rn(ls0, p0);
          ls1 = __fadd2_rn(ls1, p1);
          tt[e] = w0.x;
          tt[e + 1] = w0.y;
          tt[e + 2] = w1.x;
          tt[e + 3] = w1.y;
          mb0 = fmaxf(fmaxf(mb0, w0.x), w0.y);
          mb1 = fmaxf(fmaxf(mb1, w1.x), w1.y);
        }
        float lsum = (ls0.x + ls0.y) + (ls1.x + ls1.y);
        float mb = fmaxf(mb0, mb1);
        mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 16));
        lsum += __shfl_xor_sync(0xffffffffu, lsum, 16);
        if (threadIdx.x == 32 * kWarpSoftmax) TRACE(TR_S3, n);
        // step 7: sigma_p = max/448, P' = E4M3(w * 448/max); a zero-max block gives
        // P' = 0 and is skipped by the recurrence (R11)
        // BF16 variant: P = BF16(p) with sigma_p = 1 (no P quantization)
        // sigma_p = M_b / 448 as one multiply by the rounded reciprocal (not bit-gated; as the block-pair kernel)
        const float st_m = mb > 0.f ? mc : -INFINITY, st_sig = kBf ? 1.f : mb * (1.0f / 448.0f);
        const float inv = mb > 0.f ? __fdividef(448.0f, mb) : 0.f;
        const float2 inv2 = make_float2(inv, inv);
        uint32_t pw[kBf ? 16 : 8];
        if constexpr (kBf) {
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            __nv_bfloat162 b2 = __floats2bfloat162_rn(tt[2 * e], tt[2 * e + 1]);
            pw[e] = *reinterpret_cast<uint32_t*>(&b2);
          }
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float2 a = __fmul2_rn(make_float2(tt[4 * e], tt[4 * e + 1]), inv2);
            const float2 b = __fmul2_rn(make_float2(tt[4 * e + 2], tt[4 * e + 3]), inv2);
            pw[e] = cvt4_e4m3(a.x, a.y, b.x, b.y);
          }
        }
        if (threadIdx.x == 32 * kWarpSoftmax) TRACE(TR_S4, n);
        // prefetch S(n+1) (FP8 only: with the BF16 variant's 2-slot ring it ties P'(n) to the TMA
        // of block n+1 and serialises the pipeline, measured 4x slower per block)
        if (!kBf && SNAPMLA_SPF && j + 1 < u.k1) {
          const uint32_t ss1 = (n + 1) % kSSlots;
          mbar_wait(BAR(s_full) + 8 * ss1, ((n + 1) / kSSlots) & 1, 7, n + 1);
          tc_fence_after();
          tmem_ld_16x32bx2_x32<32>(tmem_S + lane_off + 64 * ss1, *reinterpret_cast<uint32_t(*)[32]>(tt));
        }
        // P' / stats slot free once PV_L and PV_R of block n - kPSlots completed and the
        // eight accumulator warps read its stats
        mbar_wait(BAR(p_empty) + 8 * ps, ((n / kPSlots) & 1) ^ 1, 8, n);
        if (threadIdx.x == 32 * kWarpSoftmax) TRACE(TR_S5, n);
        // K-major core matrices: byte(row, tok) = (tok/16)*1024 + row*16 + tok%16 (E4M3);
        // BF16: (tok/8)*1024 + row*16 + 2 (tok%8)
        if (hh == 0) {
          const uint32_t sa = stat0 + ps * (3 * 64 * 4);
          sts_f32(sa, st_m);
          sts_f32(sa + 256, st_sig);
          sts_f32(sa + 512, lsum);
        }
        const uint32_t pdst = sbase + kOffP + ps * V::kPBytes + r * 16;
        if constexpr (kBf) {
#pragma unroll
          for (int c = 0; c < 4; ++c) sts_u4(pdst + (4 * hh + c) * 1024, pw[4 * c], pw[4 * c + 1], pw[4 * c + 2], pw[4 * c + 3]);
        } else {
          sts_u4(pdst + (2 * hh) * 1024, pw[0], pw[1], pw[2], pw[3]);
          sts_u4(pdst + (2 * hh + 1) * 1024, pw[4], pw[5], pw[6], pw[7]);
        }
        if (threadIdx.x == 32 * kWarpSoftmax) TRACE(TR_C2, n);
        fence_proxy_async_smem();
        warp_arrive(BAR(p_full) + 8 * ps, lane);
        if (threadIdx.x == 32 * kWarpSoftmax) TRACE(TR_SM_OUT, n);
      }
      ++unit;
    }
  } else if constexpr (kSwPv) {
    if constexpr (kRegsAcc > 128) regs_inc<kRegsAcc>();
    else regs_dec<kRegsAcc>();
    // ==== accumulators (swapped PV): thread = (dim, 64 rows) for dim tiles 2 w, 2 w + 1; O^T in registers ====
    const int q4 = warp & 3, w = warp >> 2;
    const uint32_t lane_off = (uint32_t)(32 * q4) << 16;
    uint32_t n = 0, unit = 0;
    while (it.next(u)) {
      float o[2][64];
#pragma unroll
      for (int d = 0; d < 2; ++d)
#pragma unroll
        for (int h = 0; h < 64; ++h) o[d][h] = 0.f;   // the first block enters with gamma = 0
      for (int j = u.k0; j < u.k1; ++j, ++n) {
        const uint32_t gs = n % 4;
        mbar_wait_sleep(BAR(gam_full) + 8 * gs, (n / 4) & 1);            // gamma / delta of block n
        const float4 sk4 = lds_f4(BAR(skipw) + 16 * gs);
        const bool anyskip = (sk4.x + sk4.y + sk4.z + sk4.w) != 0.f;
        if (threadIdx.x == 128 * w) TRACE(w == 0 ? TR_C0 : TR_C1, n);
        mbar_wait_sleep(BAR(t_full) + 8 * w, n & 1);                     // T^T half w = V^T P'^T (n) complete
        tc_fence_after();
        if (threadIdx.x == 128 * w) TRACE(w == 0 ? TR_C1 : TR_C2, n);
        const uint32_t gb = BAR(gam) + 4 * (gs * 64), db = BAR(del) + 4 * (gs * 64);
#pragma unroll
        for (int c = 0; c < 4; ++c) {   // 16 rows (heads) at a time: their gammas serve both dim tiles
          float g[16];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float4 g4 = lds_f4(gb + 4 * (16 * c + 4 * i));
            g[4 * i] = g4.x;
            g[4 * i + 1] = g4.y;
            g[4 * i + 2] = g4.z;
            g[4 * i + 3] = g4.w;
          }
#pragma unroll
          for (int d = 0; d < 2; ++d) {
            uint32_t tv[16];
            tmem_ld_32x32b_x16(tmem + lane_off + 256 + 128 * w + 64 * d + 16 * c, tv);
            tmem_wait_ld();
            if (c == 3 && d == 1) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(BAR(t_free) + 8 * w);            // PV(n + 1) may overwrite the half
            }
            if (anyskip) {   // a row whose block is negligible keeps O (delta = 0)
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float4 d4 = lds_f4(db + 4 * (16 * c + 4 * i));
                tv[4 * i] = __float_as_uint(__uint_as_float(tv[4 * i]) * d4.x);
                tv[4 * i + 1] = __float_as_uint(__uint_as_float(tv[4 * i + 1]) * d4.y);
                tv[4 * i + 2] = __float_as_uint(__uint_as_float(tv[4 * i + 2]) * d4.z);
                tv[4 * i + 3] = __float_as_uint(__uint_as_float(tv[4 * i + 3]) * d4.w);
              }
            }
#pragma unroll
            for (int e = 0; e < 16; e += 2) {
              const int h = 16 * c + e;
              const float2 r2 = __ffma2_rn(make_float2(o[d][h], o[d][h + 1]), make_float2(g[e], g[e + 1]),
                                           make_float2(__uint_as_float(tv[e]), __uint_as_float(tv[e + 1])));
              o[d][h] = r2.x;
              o[d][h + 1] = r2.y;
            }
          }
        }
        warp_arrive(BAR(gam_empty) + 8 * gs, lane);                       // this block's factors read
        if (threadIdx.x == 128 * w) TRACE(w == 0 ? TR_C_L : TR_C_R, n);
      }
      // ---------------- epilogue (a9): o_part[row h][dim] = O^T[dim][h] f_h (f from the softmax warps)
      mbar_wait(BAR(fin_full), unit & 1);
      const int64_t prow0 = ((int64_t)u.slot * p.n_ht + ht) * kHeadTile;
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        const int dim = 128 * (2 * w + d) + 32 * q4 + lane;
#pragma unroll
        for (int h = 0; h < 64; ++h)
          if (ht * kHeadTile + h < p.num_heads) p.o_part[(prow0 + h) * kDc + dim] = o[d][h] * lds_f32(BAR(fin) + 4 * h);
      }
      warp_arrive(BAR(fin_empty), lane);
      ++unit;
    }
  } else {
    if constexpr (kRegsAcc > 128) regs_inc<kRegsAcc>();
    else regs_dec<kRegsAcc>();
    // ========= accumulators: Alg.1 recurrence per row, O <- gamma O + T in registers =========
    const uint32_t w = warp >> 2;            // 0: O cols 0-255 (L halves), 1: cols 256-511 (R halves)
    const int k = warp & 3;
    const int t = lane & 15, hh = lane >> 4;
    const int r = 16 * k + t;
    const int head = ht * kHeadTile + r;
    const bool row_ok = head < p.num_heads;
    const uint32_t lane_off = (uint32_t)(32 * k) << 16;
    const uint32_t stat0 = BAR(stat) + 4 * r;
    uint32_t n = 0;
    while (it.next(u)) {
      const uint32_t n0 = n;
      // O holds sum_b (sig_b 2^{m_b - m_O}) P'_b V in units of sig_O 2^{m_O} (log2 units);
      // l_run = sum_b l_b 2^{m_b - m_ref}.  This thread: row r, cols 256 w + 128 hh + [0, 128).
      float o[128];
#pragma unroll
      for (int e = 0; e < 128; ++e) o[e] = 0.f;   // the first block enters with gamma = 0
      float m_ref = -INFINITY, m_O = 0.f, sig_O = 1.f, l_run = 0.f;
      for (int j = u.k0; j < u.k1; ++j, ++n) {
        const uint32_t ps = n % kPSlots;
        mbar_wait_sleep(BAR(p_full) + 8 * ps, (n / kPSlots) & 1);
        const uint32_t sa = stat0 + ps * (3 * 64 * 4);
        const float mb = lds_f32(sa), sb = lds_f32(sa + 256), lb = lds_f32(sa + 512);
        warp_arrive(BAR(p_empty) + 8 * ps, lane);                      // stats of this slot consumed
        const float m_new = fmaxf(m_ref, mb);                          // step 4 (running max)
        // a block whose contributions are < 2^-64 of the running total is dropped
        // (Alg.1 loses it to fp32 underflow of exp(s - m)); so is a zero-max block
        const bool first = n == n0;
        const bool skip = !first && ((mb == -INFINITY) || (mb < m_new - 64.f));
        float gamma = 0.f;
        if (first) {
          m_O = mb;
          sig_O = sb;
          l_run = lb;
          m_ref = mb;
        } else if (!skip) {
          gamma = ex2_approx(m_O - mb) * __fdividef(sig_O, sb);        // steps 9-10
          l_run = l_run * ex2_approx(m_ref - m_new) + lb * ex2_approx(mb - m_new);
          m_ref = m_new;
          m_O = mb;
          sig_O = sb;
        }
        const uint32_t h = 2 * n + w, ts = h % V::kTSlots;
        mbar_wait_sleep(BAR(t_full) + 8 * ts, (h / V::kTSlots) & 1);      // T half = P'(n) V complete
        tc_fence_after();
        if (threadIdx.x == 128 * w) TRACE(w == 0 ? TR_C0 : TR_C1, n);
        const uint32_t taddr = V::t_slot(tmem, ts) + lane_off;
        const float2 g2 = make_float2(gamma, gamma);
        // software-pipelined T reads (8 chunks of 16 columns)
        uint32_t tv[2][16];
        tmem_ld_16x32bx2_x16<128>(taddr, tv[0]);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          tmem_wait_ld();
          if (c < 7) tmem_ld_16x32bx2_x16<128>(taddr + 16 * (c + 1), tv[(c + 1) & 1]);
          else {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(BAR(t_free) + 8 * ts);           // PV may overwrite the slot
          }
          const uint32_t* cur = tv[c & 1];
          if (!skip) {   // first block: gamma = 0 on a zeroed O
#pragma unroll
            for (int e = 0; e < 16; e += 2) {
              const float2 a = __ffma2_rn(make_float2(o[16 * c + e], o[16 * c + e + 1]), g2,
                                          make_float2(__uint_as_float(cur[e]), __uint_as_float(cur[e + 1])));
              o[16 * c + e] = a.x;
              o[16 * c + e + 1] = a.y;
            }
          }
        }
        if (threadIdx.x == 128 * w) TRACE(w == 0 ? TR_C_L : TR_C_R, n);
      }
      // ---------------- epilogue (a9): o = sig_O 2^{m_O - m_ref} O / l ; L = (m_ref + log2 l) ln 2
      // a row that saw no key in this split (MTP: the split holds only keys after its
      // query token) leaves o = 0, lse = -inf, which the combine weighs by zero
      const float f = l_run > 0.f ? sig_O * ex2_approx(m_O - m_ref) / l_run : 0.f;
      const int64_t prow = ((int64_t)u.slot * p.n_ht + ht) * kHeadTile + r;
      if (row_ok) {
        float* dst = p.o_part + prow * kDc + 256 * w + 128 * hh;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
#pragma unroll
          for (int e = 0; e < 32; e += 4)
            *reinterpret_cast<float4*>(dst + 32 * c + e) =
                make_float4(o[32 * c + e] * f, o[32 * c + e + 1] * f, o[32 * c + e + 2] * f, o[32 * c + e + 3] * f);
        }
        if (w == 0 && hh == 0)
          p.lse_part[prow] = l_run > 0.f ? (m_ref + log2f(l_run)) * 0.69314718055994531f : -INFINITY;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kWarpQk) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
#ifdef SNAPMLA_TRACE
  if (p.trace != nullptr && threadIdx.x == 0) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(gt));
    p.trace[TR_NEV * kTraceN + 2 * blockIdx.x + 1] = gt;
  }
#endif
}

// ===================================================================== cta_group::2 helpers
constexpr uint32_t kIdescPvS = make_idesc(0, 0, 0, 1, 128, 256);
#define SNAPMLA_QK8S(ta, bo, acc)                                                              \
  "add.u32 t, %1, " #ta ";\n\tadd.s64 b, %2, " #bo ";\n\t"                                     \
  "@e tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], [t], b, %3, " acc ";\n\t"
#define SNAPMLA_QK16S(ao)                                                                      \
  "add.s64 a, %4, " #ao ";\n\tadd.s64 b, %5, " #ao ";\n\t"                                     \
  "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a, b, %6, pt;\n\t"
// One PV half (cta_group::2, N = 256 = 128 dims from each CTA): 2 x K = 32; commits multicast
// to t_full, p_empty and kv_empty of both CTAs.
__device__ __forceinline__ void pv_issue_2sm(uint32_t dT, uint64_t dP, uint64_t dV, uint32_t bar_t, uint32_t bar_p,
                                             uint32_t bar_kv) {
  asm volatile(
      "{\n\t.reg .pred e, pf, pt;\n\t.reg .b64 a, b;\n\t.reg .b32 z;\n\t"
      "mov.b32 z, 0;\n\tsetp.ne.b32 pf, z, 0;\n\tsetp.eq.b32 pt, z, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, pf;\n\t"
      "add.s64 a, %1, 128;\n\tadd.s64 b, %2, 256;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], a, b, %3, pt;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%4], %7;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%5], %7;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%6], %7;\n\t}"
      ::"r"(dT), "l"(dP), "l"(dV), "r"(kIdescPvS), "r"(bar_t), "r"(bar_p), "r"(bar_kv), "h"((uint16_t)3)
      : "memory");
}

// ===================================================================== 2-SM block-pair kernel
// 64 < rows <= 128 (DeepSeek-R1's 128 heads; LongCat MTP-2).  The two 64-row head tiles of a
// key range are a CTA pair (cluster of 2) and every contraction is a cta_group::2 MMA at M = 128
// (64 rows per CTA), processed over PAIRS of key blocks (A, B) = (j, j + 1):
//   QK  N = 128: CTA 0 supplies block A's 64 tokens, CTA 1 block B's (each the full 576 dims:
//       4 FP8 boxes X = dims 0-255, Y = dims 256-511, and the RoPE box R).  Each CTA gets S for its
//       rows with block A on lanes 0-63 and block B on lanes 64-127 (scripts/pair_probe.cu), so a
//       softmax thread owns a whole row of ONE block: no cross-thread exchange (SMSPs 0-1 run
//       block A, SMSPs 2-3 block B of the same rows at the same time).
//   PV  N = 256 per half: CTA 0 supplies V dims 256-511, CTA 1 dims 0-255 of the block, from the
//       same SMEM offset in both CTAs (the leader's descriptor addresses both): once QK(pair) has
//       completed, CTA 0 reloads X <- B dims 256-511 and CTA 1 reloads Y <- A dims 0-255
//       ("phase 2", an L2 hit: the peer loaded those bytes in phase 1); PV(A) then reads Y and
//       PV(B) reads X in both CTAs.  T lanes 0-63 = dims 256-511, lanes 64-127 = dims 0-255.
// 40.5 KB per pair per CTA in SMEM (4 pairs = 8 blocks in flight per cluster), DRAM bytes stay
// algorithmic.  A unit with an odd block count ends in a half pair: block B is absent (no loads,
// softmax writes m = -inf, the accumulators skip it; the QK / PV MMAs still run on stale SMEM
// and their outputs are never read).  Cross-CTA signals as in §7.8: the peer's phase-1/2 TMA
// complete on the leader's kv_full / v_full (cta_group::2 TMA), its S-slot and T-half releases
// and P' readiness are forwarded to the leader by its idle issue warps.
constexpr int kBpSlots = 4;
#ifndef SNAPMLA_BP_PSLOTS
#define SNAPMLA_BP_PSLOTS 2
#endif
constexpr int kBpPSlots = SNAPMLA_BP_PSLOTS;   // P' + stats ring depth (block pairs)
// 16 warps: 0-7 accumulators (2 per SMSP), 8 TMA, 9 QK, 10 / 11 PV_L / PV_R (peer CTA: 9-11
// forward its signals), 12-15 softmax.  setmaxnreg only redistributes the CTA's launch
// allocation (512 x 128), so per SMSP 2 x 176 + 40 + 120 = 512 = 4 x 128.  (A 20-warp layout
// with two token-half softmax warps per SMSP measured slower: its 480-register budget per SMSP
// starves the accumulators.)
constexpr int kBpThreads = 512, kBpWarpTma = 8, kBpWarpQk = 9, kBpWarpPv = 10, kBpWarpSm = 12;
constexpr uint32_t kBpRegsAcc = 176, kBpRegsSm = 120, kBpRegsIssue = 40;
static_assert(2 * kBpRegsAcc + kBpRegsSm + kBpRegsIssue <= 4 * 128, "setmaxnreg budget per SMSP (block-pair kernel)");
constexpr uint32_t kBpStage = 41984;   // X 16 KB | Y 16 KB | RoPE 8 KB | sigma_K of A (256 B) and B (256 B)
constexpr uint32_t kBpOffX = 0, kBpOffY = 16384, kBpOffR = 32768, kBpOffSc = 40960;
constexpr uint32_t kBpTx1 = 40960, kBpTx2 = 16384;   // TMA bytes per CTA: phase 1 (own block), phase 2 (V half)
constexpr uint32_t kBpOffQr = 0, kBpOffP = 8192, kBpOffKv = 8192 + kBpPSlots * 8192;
constexpr uint32_t kBpOffBar = kBpOffKv + kBpSlots * kBpStage;
constexpr uint32_t kBpBarBytes = 8192;
constexpr uint32_t kBpSmem = kBpOffBar + kBpBarBytes + 1024;
static_assert(kBpSmem <= 232448, "shared memory budget (block-pair kernel)");
constexpr uint32_t kIdescQk8P = make_idesc(0, 0, 0, 0, 128, 128);
constexpr uint32_t kIdescQk16P = make_idesc(1, 1, 0, 0, 128, 128);
// TMEM: S pair slot ss at cols 64 ss; q codes (QK A operand, both lane halves) at cols 128-255;
// T half slot h (L = 0, R = 1) at cols 256 + 128 h.
constexpr uint32_t kBpTmemQ = 128, kBpTmemT = 256;

// The block-pair kernel's MMA issuers and the peer's forwarding warps share SMSPs with the softmax
// warps; SNAPMLA_BP_SLEEP makes their waits suspend instead of spin (A/B: profiles/r2w_*).
// SNAPMLA_BP_DIRECT (default 0): the peer CTA's softmax and accumulator warps arrive on the leader's
// s_empty / t_free themselves (relaxed remote arrives after their TMEM reads completed) instead of
// arriving locally and having an idle issue warp forward one arrive.  Measured slower on DS-R1
// (0.503-0.513 vs 0.482 ms decode: 8 remote arrives per T half cost more than the forwarding hop;
// profiles/r2w_bp_direct_ab_dsr1.txt).
#ifndef SNAPMLA_BP_DIRECT
#define SNAPMLA_BP_DIRECT 0
#endif
#ifdef SNAPMLA_BP_SLEEP
#define SNAPMLA_BP_ISSUE_WAIT(bar, par) mbar_wait_sleep((bar), (par))
#else
#define SNAPMLA_BP_ISSUE_WAIT(bar, par) mbar_wait((bar), (par))
#endif
struct BarsP {
  alignas(16) uint8_t sink[kBpPSlots + 1][16];   // landing bytes of the peer's P' / Q signals
  uint64_t kv_full[kBpSlots];    // leader: phase-1 TMA of both CTAs
  uint64_t v_full[kBpSlots];     // leader: phase-2 TMA of both CTAs
  uint64_t sc_full[kBpSlots];    // local: sigma_K of A and B
  uint64_t qk_done[kBpSlots];    // both: QK(pair) complete (multicast commit) -> phase 2 may overwrite
  uint64_t kv_empty[kBpSlots];   // both: PV_L(B) + PV_R(B) complete (multicast commits)
  uint64_t s_full[kSSlots], s_empty[kSSlots];
  uint64_t p_full[kBpPSlots], pp_full[kBpPSlots], p_empty[kBpPSlots];
  uint64_t t_full[2], t_free[2];
  uint64_t q_full, q_free;
  uint32_t tmem_base;
  float crow[64];
  float stat[kBpPSlots][2][3][64];   // [pair slot][block A / B][m, sigma_p, l][row]
};
static_assert(sizeof(BarsP) <= kBpBarBytes, "barrier region (block-pair kernel)");
#define BP(field) (bar0 + (uint32_t)offsetof(BarsP, field))

// QK of a block pair: 16 x kind::f8f6f4 + 4 x kind::f16, cta_group::2, N = 128; commits
// multicast to s_full (softmax) and qk_done (phase-2 TMA) of both CTAs.
__device__ __forceinline__ void qk_issue_bp(uint32_t dS, uint32_t tQ, uint64_t dK, uint64_t dQr, uint64_t dKr,
                                            uint32_t bar_s, uint32_t bar_q) {
  asm volatile(
      "{\n\t.reg .pred e, pf, pt;\n\t.reg .b64 a, b;\n\t.reg .b32 z, t;\n\t"
      "mov.b32 z, 0;\n\tsetp.ne.b32 pf, z, 0;\n\tsetp.eq.b32 pt, z, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      SNAPMLA_QK8S(0, 0, "pf") SNAPMLA_QK8S(8, 2, "pt") SNAPMLA_QK8S(16, 4, "pt") SNAPMLA_QK8S(24, 6, "pt")
      SNAPMLA_QK8S(32, 512, "pt") SNAPMLA_QK8S(40, 514, "pt") SNAPMLA_QK8S(48, 516, "pt") SNAPMLA_QK8S(56, 518, "pt")
      SNAPMLA_QK8S(64, 1024, "pt") SNAPMLA_QK8S(72, 1026, "pt") SNAPMLA_QK8S(80, 1028, "pt") SNAPMLA_QK8S(88, 1030, "pt")
      SNAPMLA_QK8S(96, 1536, "pt") SNAPMLA_QK8S(104, 1538, "pt") SNAPMLA_QK8S(112, 1540, "pt") SNAPMLA_QK8S(120, 1542, "pt")
      SNAPMLA_QK16S(0) SNAPMLA_QK16S(2) SNAPMLA_QK16S(4) SNAPMLA_QK16S(6)
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%7], %9;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%8], %9;\n\t}"
      ::"r"(dS), "r"(tQ), "l"(dK), "r"(kIdescQk8P), "l"(dQr), "l"(dKr), "r"(kIdescQk16P), "r"(bar_s), "r"(bar_q),
      "h"((uint16_t)3)
      : "memory");
}
// PV half of block A: 2 x K = 32, commit multicast to t_full only
__device__ __forceinline__ void pv_issue_bp_a(uint32_t dT, uint64_t dP, uint64_t dV, uint32_t bar_t) {
  asm volatile(
      "{\n\t.reg .pred e, pf, pt;\n\t.reg .b64 a, b;\n\t.reg .b32 z;\n\t"
      "mov.b32 z, 0;\n\tsetp.ne.b32 pf, z, 0;\n\tsetp.eq.b32 pt, z, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, pf;\n\t"
      "add.s64 a, %1, 128;\n\tadd.s64 b, %2, 256;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], a, b, %3, pt;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%4], %5;\n\t}"
      ::"r"(dT), "l"(dP), "l"(dV), "r"(kIdescPvS), "r"(bar_t), "h"((uint16_t)3)
      : "memory");
}

__device__ __forceinline__ uint64_t l2_policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kBpThreads, 1)
    mla_decode_bp_kernel(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_rope,
                         const DecodeParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t bar0 = sbase + kBpOffBar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cta = cluster_ctarank();
  const bool leader = cta == 0;
#ifdef SNAPMLA_TRACE
  if (p.trace != nullptr && threadIdx.x == 0) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(gt));
    p.trace[TR_NEV * kTraceN + 2 * blockIdx.x] = gt;
  }
#endif

  if (threadIdx.x == 0) {
    for (int i = 0; i < kBpSlots; ++i) {
      mbar_init(BP(kv_full) + 8 * i, 1);
      mbar_init(BP(v_full) + 8 * i, 1);
      mbar_init(BP(sc_full) + 8 * i, 1);
      mbar_init(BP(qk_done) + 8 * i, 1);
      mbar_init(BP(kv_empty) + 8 * i, 2);
    }
    for (int i = 0; i < kSSlots; ++i) {
      mbar_init(BP(s_full) + 8 * i, 1);
      mbar_init(BP(s_empty) + 8 * i, leader ? (SNAPMLA_BP_DIRECT ? 4 + 4 : 4 + 1) : 4);
    }
    for (int i = 0; i < kBpPSlots; ++i) {
      mbar_init(BP(p_full) + 8 * i, 4 * kArriveMul);
      mbar_init(BP(pp_full) + 8 * i, 1);
      mbar_init(BP(p_empty) + 8 * i, 2 + 8 * kArriveMul);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(BP(t_full) + 8 * i, 1);
      mbar_init(BP(t_free) + 8 * i, leader ? (SNAPMLA_BP_DIRECT ? 8 + 8 : 8 + 1) : 8);
    }
    mbar_init(BP(q_full), leader ? 12 + 1 : 12);
    mbar_init(BP(q_free), 1);
    fence_barrier_init();
  }
  if (warp == kBpWarpTma && lane == 0) {
    tma_prefetch_desc(&tm_kv);
    tma_prefetch_desc(&tm_rope);
  }
  if (warp == kBpWarpQk) tmem_alloc_pair(BP(tmem_base), 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = lds_u32(BP(tmem_base));

  pdl_wait();
  pdl_launch_dependents();
  const int ht = (int)cta;
  const int g = blockIdx.x / 2;
  const int per = p.ws_hdr[H_PER], total = p.ws_hdr[H_TOTAL], groups = p.ws_hdr[H_GROUPS];
  const int lo = g * per;
  const bool has_work = g < groups && lo < total;
  const int hi = min(total, lo + per);
  UnitIter it{p.cum, lo, hi, g, has_work ? __ldg(p.first_req + g) : 0, has_work ? p.batch : 0};
  Unit u;

  if (warp >= kBpWarpTma && warp < kBpWarpSm) {
    regs_dec<kBpRegsIssue>();
    if (warp == kBpWarpTma) {
      // ===================== TMA producer (both CTAs): phase 1 and phase 2 =====================
      // One thread serves two streams: phase 1 of pair n1 (slot free: kv_empty) and phase 2 of
      // pair n2 < n1 (QK(n2) complete: qk_done); it polls both so neither waits on the other.
      if (lane == 0) {
        const uint64_t pol = l2_policy_evict_first(), pol_keep = l2_policy_evict_normal();
        const uint32_t kv_full_leader = mapa_shared(BP(kv_full), 0), v_full_leader = mapa_shared(BP(v_full), 0);
        UnitIter it1 = it, it2 = it;
        Unit u1, u2;
        bool live1 = it1.next(u1), live2 = it2.next(u2);
        int j1 = live1 ? u1.k0 : 0, j2 = live2 ? u2.k0 : 0;
        if (live1) prefetch_block_table(p.block_table + (int64_t)u1.b * p.max_pages, u1.k0, u1.k1);
        uint32_t n1 = 0, n2 = 0;
        while (live2) {
          bool did = false;
          if (live1 && n1 < n2 + kBpSlots) {
            const uint32_t st = n1 % kBpSlots;
            if (mbar_try_wait_ns(BP(kv_empty) + 8 * st, ((n1 / kBpSlots) & 1) ^ 1, n2 < n1 ? 200u : 100000u)) {
              TRACE(TR_TMA, n1);
              const int32_t* bt = p.block_table + (int64_t)u1.b * p.max_pages;
              const bool hasB = j1 + 1 < u1.k1;
              const int rowA = __ldg(bt + j1) * kPage, rowB = hasB ? __ldg(bt + j1 + 1) * kPage : 0;
              const uint32_t slot = sbase + kBpOffKv + st * kBpStage;
              const uint32_t sc = BP(sc_full) + 8 * st;
              mbar_arrive_expect_tx(sc, hasB ? 512 : 256);
              bulk_load(slot + kBpOffSc, p.kv_scale + (int64_t)rowA, 256, sc, pol);
              if (hasB) bulk_load(slot + kBpOffSc + 256, p.kv_scale + (int64_t)rowB, 256, sc, pol);
              if (leader) mbar_arrive_expect_tx(BP(kv_full) + 8 * st, hasB ? 2 * kBpTx1 : kBpTx1);
              if (leader || hasB) {
                const int row = leader ? rowA : rowB;
                const uint32_t fb = kv_full_leader + 8 * st;
#pragma unroll
                for (int c = 0; c < 4; ++c)   // the half the peer reloads in phase 2 stays in L2 (evict_normal)
                  tma_load_2d_cg2(slot + c * kBoxBytes, &tm_kv, fb, c * 128, row,
                                  ((c >> 1) == (int)cta) ? pol_keep : pol);
                tma_load_2d_cg2(slot + kBpOffR, &tm_rope, fb, 0, row, pol);
              }
              ++n1;
              j1 += 2;
              if (j1 >= u1.k1) {
                live1 = it1.next(u1);
                if (live1) {
                  j1 = u1.k0;
                  prefetch_block_table(p.block_table + (int64_t)u1.b * p.max_pages, u1.k0, u1.k1);
                }
              }
              did = true;
            }
          }
          if (n2 < n1) {
            const uint32_t st = n2 % kBpSlots;
            if (mbar_try_wait_ns(BP(qk_done) + 8 * st, (n2 / kBpSlots) & 1, live1 && n1 < n2 + kBpSlots ? 200u : 100000u)) {
              const int32_t* bt = p.block_table + (int64_t)u2.b * p.max_pages;
              const bool hasB = j2 + 1 < u2.k1;
              const uint32_t slot = sbase + kBpOffKv + st * kBpStage;
              const uint32_t fb = v_full_leader + 8 * st;
              if (leader) mbar_arrive_expect_tx(BP(v_full) + 8 * st, hasB ? 2 * kBpTx2 : kBpTx2);
              if (!leader) {           // CTA 1: Y <- block A dims 0-255
                const int rowA = __ldg(bt + j2) * kPage;
                tma_load_2d_cg2(slot + kBpOffY, &tm_kv, fb, 0, rowA, pol);
                tma_load_2d_cg2(slot + kBpOffY + kBoxBytes, &tm_kv, fb, 128, rowA, pol);
              } else if (hasB) {       // CTA 0: X <- block B dims 256-511
                const int rowB = __ldg(bt + j2 + 1) * kPage;
                tma_load_2d_cg2(slot + kBpOffX, &tm_kv, fb, 256, rowB, pol);
                tma_load_2d_cg2(slot + kBpOffX + kBoxBytes, &tm_kv, fb, 384, rowB, pol);
              }
              ++n2;
              j2 += 2;
              if (j2 >= u2.k1) {
                live2 = it2.next(u2);
                if (live2) j2 = u2.k0;
              }
              did = true;
            }
          }
        }
      }
    } else if (warp == kBpWarpQk && leader) {
      // ================================ QK issuer (leader) ================================
      const uint64_t dQr = make_smem_desc(sbase + kBpOffQr, 16, 1024, LAYOUT_SW128);
      uint32_t n = 0, unit = 0;
      while (it.next(u)) {
        SNAPMLA_BP_ISSUE_WAIT(BP(q_full), unit & 1);
        for (int j = u.k0; j < u.k1; j += 2, ++n) {
          const uint32_t st = n % kBpSlots, ss = n % kSSlots;
          SNAPMLA_BP_ISSUE_WAIT(BP(kv_full) + 8 * st, (n / kBpSlots) & 1);
          if (lane == 0) TRACE(TR_C1, n);
          SNAPMLA_BP_ISSUE_WAIT(BP(s_empty) + 8 * ss, ((n / kSSlots) & 1) ^ 1);
          tc_fence_after();
          if (lane == 0) TRACE(TR_QK, n);
          const uint32_t kv = sbase + kBpOffKv + st * kBpStage;
          qk_issue_bp(tmem + 64 * ss, tmem + kBpTmemQ, make_smem_desc(kv + kBpOffX, 16, 1024, LAYOUT_SW128), dQr,
                      make_smem_desc(kv + kBpOffR, 16, 1024, LAYOUT_SW128), BP(s_full) + 8 * ss,
                      BP(qk_done) + 8 * st);
        }
        mma_commit_pair_ws(BP(q_free));
        ++unit;
      }
    } else if (leader) {
      // ============================ PV_L / PV_R issuers (leader) ============================
      const uint32_t half = warp - kBpWarpPv;
      const uint32_t dT = tmem + kBpTmemT + 128 * half;
      uint32_t n = 0;
      while (it.next(u)) {
        for (int j = u.k0; j < u.k1; j += 2, ++n) {
          const uint32_t st = n % kBpSlots, ps = n % kBpPSlots;
          SNAPMLA_BP_ISSUE_WAIT(BP(p_full) + 8 * ps, (n / kBpPSlots) & 1);
          SNAPMLA_BP_ISSUE_WAIT(BP(pp_full) + 8 * ps, (n / kBpPSlots) & 1);
          if (lane == 0 && half == 0) TRACE(TR_S5, n);
          SNAPMLA_BP_ISSUE_WAIT(BP(v_full) + 8 * st, (n / kBpSlots) & 1);
          if (lane == 0 && half == 0) TRACE(TR_C2, n);
          const uint32_t kv = sbase + kBpOffKv + st * kBpStage;
          const uint32_t pA = sbase + kBpOffP + ps * 8192;
#pragma unroll
          for (int blk = 0; blk < 2; ++blk) {
            const uint32_t nb = 2 * n + blk;
            if (nb >= 1) SNAPMLA_BP_ISSUE_WAIT(BP(t_free) + 8 * half, (nb - 1) & 1);
            tc_fence_after();
            if (lane == 0 && blk == 0) TRACE(half == 0 ? TR_PVL : TR_PVR, n);
            const uint64_t dP = make_smem_desc(pA + 4096 * blk, 1024, 128, LAYOUT_NONE);
            const uint64_t dV = make_smem_desc(kv + (blk ? kBpOffX : kBpOffY) + half * kBoxBytes, kBoxBytes, 1024,
                                               LAYOUT_SW128);
            if (blk == 0)
              pv_issue_bp_a(dT, dP, dV, BP(t_full) + 8 * half);
            else
              pv_issue_2sm(dT, dP, dV, BP(t_full) + 8 * half, BP(p_empty) + 8 * ps, BP(kv_empty) + 8 * st);
          }
        }
      }
    } else if (warp == kBpWarpQk) {
      // ======== peer: forward its Q readiness and "S slot read" to the leader ========
      const uint32_t s_empty_leader = mapa_shared(BP(s_empty), 0);
      const uint32_t q_full_leader = mapa_shared(BP(q_full), 0);
      uint32_t n = 0, unit = 0;
      while (it.next(u)) {
        SNAPMLA_BP_ISSUE_WAIT(BP(q_full), unit & 1);
        tc_fence_after();
        if (lane == 0) mbar_signal_peer_tx(q_full_leader, mapa_shared(BP(sink), 0) + 16 * kBpPSlots, sbase + kBpOffQr);
        __syncwarp();
        ++unit;
        for (int j = u.k0; j < u.k1; j += 2, ++n) {
          if (SNAPMLA_BP_DIRECT) continue;   // the softmax warps arrive on the leader themselves
          const uint32_t ss = n % kSSlots;
          SNAPMLA_BP_ISSUE_WAIT(BP(s_empty) + 8 * ss, (n / kSSlots) & 1);
          if (lane == 0) mbar_arrive_cluster_relaxed(s_empty_leader + 8 * ss);
          __syncwarp();
        }
      }
    } else if (warp == kBpWarpPv + 1 && !SNAPMLA_BP_DIRECT) {
      // ======== peer: forward "T half read" (its 8 accumulator warps) to the leader ========
      const uint32_t t_free_leader = mapa_shared(BP(t_free), 0);
      uint32_t nb = 0;
      while (it.next(u)) {
        for (int j = u.k0; j < u.k1; j += 2) {
#pragma unroll 1
          for (int blk = 0; blk < 2; ++blk, ++nb) {
#pragma unroll 1
            for (int hf = 0; hf < 2; ++hf) {
              SNAPMLA_BP_ISSUE_WAIT(BP(t_free) + 8 * hf, nb & 1);
              if (lane == 0) mbar_arrive_cluster_relaxed(t_free_leader + 8 * hf);
              __syncwarp();
            }
          }
        }
      }
    } else if (warp == kBpWarpPv) {
      // ======== peer: forward "P' written" to the leader's PV issue (16-byte bulk-copy signal) ========
      const uint32_t pp_leader = mapa_shared(BP(pp_full), 0);
      uint32_t n = 0;
      while (it.next(u)) {
        for (int j = u.k0; j < u.k1; j += 2, ++n) {
          const uint32_t ps = n % kBpPSlots;
          SNAPMLA_BP_ISSUE_WAIT(BP(p_full) + 8 * ps, (n / kBpPSlots) & 1);
          if (lane == 0)
            mbar_signal_peer_tx(pp_leader + 8 * ps, mapa_shared(BP(sink), 0) + 16 * ps, sbase + kBpOffP + ps * 8192);
          __syncwarp();
        }
      }
    }
  } else if (warp >= kBpWarpSm) {
    regs_dec<kBpRegsSm>();
    // ======== softmax / scale fusion / P quantization: thread = (row, block of the pair) ========
    const int k = warp & 3;                  // SMSP = TMEM lane quarter
    const int hk = k >> 1;                   // block of the pair: 0 = A (lanes 0-63), 1 = B (lanes 64-127)
    const int r = 32 * (k & 1) + lane;       // row inside the head tile
    const int head = ht * kHeadTile + r;
    const bool row_ok = head < p.num_heads;
    const uint32_t lane_base = (uint32_t)(32 * k) << 16;
    uint32_t n = 0, unit = 0;
    while (it.next(u)) {
      // ---------------- Fused-Q-Quant prologue (a2): as in the 2-SM kernel (codes by the
      // accumulator warps into every lane quarter; q_r' / sigma_q and c by SMSPs 0-1)
      if (unit > 0) {
        mbar_wait(BP(q_free), (unit - 1) & 1, 11, unit);
        named_bar_sync(1, 128);
      }
      {   // Fused-Q-Quant ran in the plan launch: q_r' to its SW128 SMEM row, c = sigma_q scale log2(e)
        if (hk == 0) {
          const int64_t qrow_i = (int64_t)u.b * p.num_heads + head;
          const uint4* qrr = reinterpret_cast<const uint4*>(p.qr + qrow_i * kDr);
          sts_f32(BP(crow) + 4 * r, (row_ok ? __ldg(p.sq + qrow_i) : 1.f) * p.scale_log2);
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint4 v = row_ok ? __ldg(qrr + c) : make_uint4(0, 0, 0, 0);
            sts_u4(sbase + kBpOffQr + r * 128 + ((c ^ (r & 7)) << 4), v.x, v.y, v.z, v.w);
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(BP(q_full));
      }
      named_bar_sync(1, 128);
      const float c_row = lds_f32(BP(crow) + 4 * r);
      const int L = __ldg(p.seq_lens + u.b) - (p.q_len - 1 - head / p.heads);
      float tt[64];
      for (int j = u.k0; j < u.k1; j += 2, ++n) {
        const uint32_t st = n % kBpSlots, ss = n % kSSlots, ps = n % kBpPSlots;
        const int blk = j + hk;
        const bool valid = blk < u.k1;
        if (j == u.k0) {   // first pair of the unit; later pairs were prefetched (below)
          mbar_wait(BP(s_full) + 8 * ss, (n / kSSlots) & 1, 7, n);
          tc_fence_after();
          tmem_ld_32x32b_x32(tmem + lane_base + 64 * ss, *reinterpret_cast<uint32_t(*)[32]>(tt));
          tmem_ld_32x32b_x32(tmem + lane_base + 64 * ss + 32, *reinterpret_cast<uint32_t(*)[32]>(tt + 32));
        }
        tmem_wait_ld();
        if (threadIdx.x == 32 * kBpWarpSm) TRACE(TR_SM_IN, n);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (SNAPMLA_BP_DIRECT && !leader) mbar_arrive_cluster_relaxed(mapa_shared(BP(s_empty), 0) + 8 * ss);
          else mbar_arrive(BP(s_empty) + 8 * ss);   // peer (SNAPMLA_BP_DIRECT 0): forwarded by its warp 9
        }
        float st_m = -INFINITY, st_sig = 1.f, lsum = 0.f;
        uint32_t pw[16];
        if (valid) {
          mbar_wait(BP(sc_full) + 8 * st, (n / kBpSlots) & 1, 12, n);
          if (threadIdx.x == 32 * kBpWarpSm) TRACE(TR_S1, n);
          // sigma_K of the block, 16 tokens per batch of loads: the four loads of a batch issue
          // back to back (one exposed shared-load latency per batch, ~16 extra registers live)
          const uint32_t sk = sbase + kBpOffKv + st * kBpStage + kBpOffSc + 256 * hk;
#pragma unroll
          for (int e0 = 0; e0 < 64; e0 += 16) {                           // step 3 (descale)
            float4 s4[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) s4[i] = lds_f4(sk + 4 * (e0 + 4 * i));
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int e = e0 + 4 * i;
              const float2 a = __fmul2_rn(make_float2(tt[e], tt[e + 1]), make_float2(s4[i].x, s4[i].y));
              const float2 b = __fmul2_rn(make_float2(tt[e + 2], tt[e + 3]), make_float2(s4[i].z, s4[i].w));
              tt[e] = a.x;
              tt[e + 1] = a.y;
              tt[e + 2] = b.x;
              tt[e + 3] = b.y;
            }
          }
          const int nvalid = L - blk * kBc;
          if (nvalid < 64) {                                              // ragged tail (R19)
#pragma unroll
            for (int e = 0; e < 64; ++e) tt[e] = e < nvalid ? tt[e] : -INFINITY;
          }
          float m0 = fmax3(tt[0], tt[1], tt[2]), m1 = fmax3(tt[3], tt[4], tt[5]);
          float m2 = fmax3(tt[6], tt[7], tt[8]), m3 = fmax3(tt[9], tt[10], tt[11]);
#pragma unroll
          for (int e = 12; e < 60; e += 8) {
            m0 = fmax3(m0, tt[e], tt[e + 1]);
            m1 = fmax3(m1, tt[e + 2], tt[e + 3]);
            m2 = fmax3(m2, tt[e + 4], tt[e + 5]);
            m3 = fmax3(m3, tt[e + 6], tt[e + 7]);
          }
          const float mx = fmax3(fmax3(m0, m1, m2), fmax3(m3, tt[60], tt[61]), fmaxf(tt[62], tt[63]));
          const float mc = mx == -INFINITY ? 0.f : mx * c_row;
          if (threadIdx.x == 32 * kBpWarpSm) TRACE(TR_S2, n);
          float2 ls0 = make_float2(0.f, 0.f), ls1 = make_float2(0.f, 0.f);
          float mb0 = 0.f, mb1 = 0.f;
          float4 s4b[4];
#pragma unroll
          for (int e = 0; e < 64; e += 4) {
            if ((e & 15) == 0) {   // next batch of 16 sigma_K
#pragma unroll
              for (int i = 0; i < 4; ++i) s4b[i] = lds_f4(sk + 4 * (e + 4 * i));
            }
            const float4 s4 = s4b[(e & 15) / 4];
            const float2 e0 = __ffma2_rn(make_float2(tt[e], tt[e + 1]), make_float2(c_row, c_row), make_float2(-mc, -mc));
            const float2 e1 = __ffma2_rn(make_float2(tt[e + 2], tt[e + 3]), make_float2(c_row, c_row), make_float2(-mc, -mc));
#ifdef SNAPMLA_SOL_NOEXP   // speed-of-light experiment only (wrong results): MUFU-free softmax
            const float2 p0 = __fmul2_rn(e0, make_float2(0.5f, 0.5f)), p1 = __fmul2_rn(e1, make_float2(0.5f, 0.5f));
#else
            const float2 p0 = make_float2(ex2_approx(e0.x), ex2_approx(e0.y));   // step 5
            const float2 p1 = make_float2(ex2_approx(e1.x), ex2_approx(e1.y));
#endif
            ls0 = __fadd2_rn(ls0, p0);
            ls1 = __fadd2_rn(ls1, p1);
            const float2 w0 = __fmul2_rn(p0, make_float2(s4.x, s4.y));   // step 6: w = p sigma_K
            const float2 w1 = __fmul2_rn(p1, make_float2(s4.z, s4.w));
            tt[e] = w0.x;
            tt[e + 1] = w0.y;
            tt[e + 2] = w1.x;
            tt[e + 3] = w1.y;
            mb0 = fmax3(mb0, w0.x, w0.y);
            mb1 = fmax3(mb1, w1.x, w1.y);
          }
          lsum = (ls0.x + ls0.y) + (ls1.x + ls1.y);
          const float mb = fmaxf(mb0, mb1);
          if (threadIdx.x == 32 * kBpWarpSm) TRACE(TR_S3, n);
          // step 7: sigma_p = max/448, P' = E4M3(w * 448/max); a zero-max block is skipped (R11)
          st_m = mb > 0.f ? mc : -INFINITY;
          st_sig = mb * (1.0f / 448.0f);   // sigma_p = M_b / 448 (one rounding; not bit-gated)
          const float inv = mb > 0.f ? __fdividef(448.0f, mb) : 0.f;
          const float2 inv2 = make_float2(inv, inv);
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float2 a = __fmul2_rn(make_float2(tt[4 * e], tt[4 * e + 1]), inv2);
            const float2 b = __fmul2_rn(make_float2(tt[4 * e + 2], tt[4 * e + 3]), inv2);
            pw[e] = cvt4_e4m3(a.x, a.y, b.x, b.y);
          }
        }
        if (j + 2 < u.k1) {   // prefetch S(n+1): its TMEM load overlaps this pair's P' / stats stores
          const uint32_t ss1 = (n + 1) % kSSlots;
          mbar_wait(BP(s_full) + 8 * ss1, ((n + 1) / kSSlots) & 1, 7, n + 1);
          tc_fence_after();
          tmem_ld_32x32b_x32(tmem + lane_base + 64 * ss1, *reinterpret_cast<uint32_t(*)[32]>(tt));
          tmem_ld_32x32b_x32(tmem + lane_base + 64 * ss1 + 32, *reinterpret_cast<uint32_t(*)[32]>(tt + 32));
        }
        mbar_wait(BP(p_empty) + 8 * ps, ((n / kBpPSlots) & 1) ^ 1, 8, n);
        if (threadIdx.x == 32 * kBpWarpSm) TRACE(TR_S4, n);
        {
          const uint32_t sa = BP(stat) + ((ps * 2 + hk) * 3 * 64 + r) * 4;
          sts_f32(sa, st_m);
          sts_f32(sa + 256, st_sig);
          sts_f32(sa + 512, lsum);
        }
        if (valid) {   // K-major core matrices: byte(row, tok) = (tok / 16) * 1024 + row * 16 + tok % 16
          const uint32_t pdst = sbase + kBpOffP + ps * 8192 + hk * 4096 + r * 16;
#pragma unroll
          for (int c = 0; c < 4; ++c) sts_u4(pdst + c * 1024, pw[4 * c], pw[4 * c + 1], pw[4 * c + 2], pw[4 * c + 3]);
        }
        fence_proxy_async_smem();
        warp_arrive(BP(p_full) + 8 * ps, lane);
        if (threadIdx.x == 32 * kBpWarpSm) TRACE(TR_SM_OUT, n);
      }
      ++unit;
    }
  } else {
    regs_inc<kBpRegsAcc>();
    // ========= accumulators: thread = (row, CTA dims half of T), two warps per SMSP split columns =========
    const int k = warp & 3, cg = warp >> 2;
    const int r = 32 * (k & 1) + lane;
    const int head = ht * kHeadTile + r;
    const bool row_ok = head < p.num_heads;
    const uint32_t lane_base = (uint32_t)(32 * k) << 16;
    const int dbase = (k < 2 ? 256 : 0) + 64 * cg;   // lanes 0-63: CTA 0's V columns = dims 256-511
    uint32_t n = 0, unit = 0;
    while (it.next(u)) {
      if (unit > 0) mbar_wait(BP(q_free), (unit - 1) & 1, 19, unit);
      {
        // Fused-Q-Quant ran in the plan launch: this thread's 256 codes (dims 256 cg + [0, 256)) into
        // both TMEM lane halves (the cta_group::2 datapath reads A per N half)
        const uint4* qcr = reinterpret_cast<const uint4*>(p.qc + ((int64_t)u.b * p.num_heads + head) * kDc) + 16 * cg;
#pragma unroll
        for (int ci = 0; ci < 2; ++ci) {
          uint32_t qa[32];
#pragma unroll
          for (int g8 = 0; g8 < 8; ++g8) {
            const uint4 v = row_ok ? __ldg(qcr + 8 * ci + g8) : make_uint4(0, 0, 0, 0);
            qa[4 * g8] = v.x;
            qa[4 * g8 + 1] = v.y;
            qa[4 * g8 + 2] = v.z;
            qa[4 * g8 + 3] = v.w;
          }
          tmem_st_32x32b_x32(tmem + lane_base + kBpTmemQ + 32 * (2 * cg + ci), qa);
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(BP(q_full));
      }
      ++unit;
      float o[128];
#pragma unroll
      for (int e = 0; e < 128; ++e) o[e] = 0.f;
      float m_ref = -INFINITY, m_O = 0.f, sig_O = 1.f, l_run = 0.f;
      for (int j = u.k0; j < u.k1; j += 2, ++n) {
        const uint32_t ps = n % kBpPSlots;
        mbar_wait(BP(p_full) + 8 * ps, (n / kBpPSlots) & 1, 9, n);
        if (threadIdx.x == 0) TRACE(TR_C0, n);
        const uint32_t sa = BP(stat) + (ps * 2 * 3 * 64 + r) * 4;
        const float mbA = lds_f32(sa), sbA = lds_f32(sa + 256), lbA = lds_f32(sa + 512);
        const float mbB = lds_f32(sa + 768), sbB = lds_f32(sa + 1024), lbB = lds_f32(sa + 1280);
        warp_arrive(BP(p_empty) + 8 * ps, lane);
#pragma unroll 1
        for (int blk = 0; blk < 2; ++blk) {
          const uint32_t nb = 2 * n + blk;
          const float mb = blk ? mbB : mbA, sb = blk ? sbB : sbA, lb = blk ? lbB : lbA;
          const float m_new = fmaxf(m_ref, mb);
          const bool first = j == u.k0 && blk == 0;
#ifdef SNAPMLA_SOL_NOACC   // speed-of-light experiment only (wrong results): no accumulate FMAs
          const bool skip = true;
#else
          const bool skip = !first && ((mb == -INFINITY) || (mb < m_new - 64.f));
#endif
          float gamma = 0.f;
          if (first) {
            m_O = mb;
            sig_O = sb;
            l_run = lb;
            m_ref = mb;
          } else if (!skip) {
            gamma = ex2_approx(m_O - mb) * __fdividef(sig_O, sb);
            l_run = l_run * ex2_approx(m_ref - m_new) + lb * ex2_approx(mb - m_new);
            m_ref = m_new;
            m_O = mb;
            sig_O = sb;
          }
          const float2 g2 = make_float2(gamma, gamma);
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            mbar_wait(BP(t_full) + 8 * hf, nb & 1, 10, nb);
            tc_fence_after();
            const uint32_t taddr = tmem + lane_base + kBpTmemT + 128 * hf + 64 * cg;
            uint32_t tv[2][16];   // T in 16-column chunks, software-pipelined
            tmem_ld_32x32b_x16(taddr, tv[0]);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              tmem_wait_ld();
              if (c < 3) tmem_ld_32x32b_x16(taddr + 16 * (c + 1), tv[(c + 1) & 1]);
              else {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                  if (SNAPMLA_BP_DIRECT && !leader) mbar_arrive_cluster_relaxed(mapa_shared(BP(t_free), 0) + 8 * hf);
                  else mbar_arrive(BP(t_free) + 8 * hf);   // peer (SNAPMLA_BP_DIRECT 0): forwarded by its warp 11
                }
              }
              const uint32_t* cur = tv[c & 1];
              if (!skip) {
#pragma unroll
                for (int e = 0; e < 16; e += 2) {
                  const int oi = 64 * hf + 16 * c + e;
                  const float2 a = __ffma2_rn(make_float2(o[oi], o[oi + 1]), g2,
                                              make_float2(__uint_as_float(cur[e]), __uint_as_float(cur[e + 1])));
                  o[oi] = a.x;
                  o[oi + 1] = a.y;
                }
              }
            }
            if (threadIdx.x == 0 && blk == 0) TRACE(hf == 0 ? TR_C_L : TR_C_R, n);
          }
        }
      }
      const float f = l_run > 0.f ? sig_O * ex2_approx(m_O - m_ref) / l_run : 0.f;
      const int64_t prow = ((int64_t)u.slot * p.n_ht + ht) * kHeadTile + r;
      if (row_ok) {
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          float* dst = p.o_part + prow * kDc + dbase + 128 * hf;
#pragma unroll
          for (int e = 0; e < 64; e += 4)
            *reinterpret_cast<float4*>(dst + e) = make_float4(o[64 * hf + e] * f, o[64 * hf + e + 1] * f,
                                                              o[64 * hf + e + 2] * f, o[64 * hf + e + 3] * f);
        }
        if (k < 2 && cg == 0)
          p.lse_part[prow] = l_run > 0.f ? (m_ref + log2f(l_run)) * 0.69314718055994531f : -INFINITY;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == kBpWarpQk) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 512);
  }
#ifdef SNAPMLA_TRACE
  if (p.trace != nullptr && threadIdx.x == 0) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(gt));
    p.trace[TR_NEV * kTraceN + 2 * blockIdx.x + 1] = gt;
  }
#endif
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

static bool encode_2d(CUtensorMap* m, CUtensorMapDataType dt, const void* base, uint64_t inner, uint64_t rows,
                      uint64_t row_bytes, uint32_t box_inner, uint32_t box_rows) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_inner, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ---- process-wide host state (thread-safe): the debug switches below, a per-device
// record of one-time launch attributes, and a small cache of encoded tensor maps keyed by
// (device, pool base, rows, kind).  Nothing else is global.
std::atomic<unsigned long long*> g_trace{nullptr};
static std::atomic<int> g_kernel{-1};   // 64 < rows <= 128: -1 auto, 0 single-CTA, 1 block-pair (debug override)
static std::atomic<int> g_small{-1};    // rows <= 32: -1 auto (swapped for <= 16), 1 swapped, 0 single-CTA (debug)

struct DeviceInfo {
  int sms = 0;
  bool attr_done[3] = {false, false, false};   // MaxDynamicSharedMemorySize set: FP8, BF16, block-pair
  int bp_max_clusters = -1;
};
constexpr int kMaxDevices = 64;
static std::mutex g_host_mu;
static DeviceInfo g_dev[kMaxDevices];

struct TmapEntry {
  int dev;
  const void* base;
  uint64_t rows;
  int kind;   // 0 FP8 content, 1 BF16 content (baseline), 2 RoPE
  CUtensorMap map;
};
constexpr int kTmapCache = 32;
static TmapEntry g_tmap[kTmapCache];
static int g_tmap_n = 0, g_tmap_next = 0;

int current_device() {
  int dev = 0;
  return cudaGetDevice(&dev) == cudaSuccess && dev >= 0 && dev < kMaxDevices ? dev : -1;
}

int device_num_sms() {
  const int dev = current_device();
  if (dev < 0) return 0;
  std::lock_guard<std::mutex> lk(g_host_mu);
  if (g_dev[dev].sms == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    g_dev[dev].sms = n;
  }
  return g_dev[dev].sms;
}

// the encoded map for (current device, base, rows, kind), encoding it on first use
bool cached_tmap(int dev, const void* base, uint64_t rows, int kind, CUtensorMap* out) {
  std::lock_guard<std::mutex> lk(g_host_mu);
  for (int i = 0; i < g_tmap_n; ++i) {
    const TmapEntry& e = g_tmap[i];
    if (e.dev == dev && e.base == base && e.rows == rows && e.kind == kind) {
      *out = e.map;
      return true;
    }
  }
  CUtensorMap m;
  const bool ok = kind == 0   ? encode_2d(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, base, kDc, rows, kDc, 128, 64)
                  : kind == 1 ? encode_2d(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, base, kDc, rows, kDc * 2, 64, 64)
                              : encode_2d(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, base, kDr, rows, kDr * 2, 64, 64);
  if (!ok) return false;
  TmapEntry& e = g_tmap[g_tmap_next];
  e = TmapEntry{dev, base, rows, kind, m};
  g_tmap_next = (g_tmap_next + 1) % kTmapCache;
  if (g_tmap_n < kTmapCache) ++g_tmap_n;
  *out = m;
  return true;
}

mla_status launch_plan(const int32_t* seq_lens, int batch, int num_heads, int groups, int32_t* hdr, int32_t* cum,
                       int32_t* first_req, int num_sms, cudaStream_t st, const __nv_bfloat16* q, uint8_t* qc,
                       __nv_bfloat16* qr, float* sq) {
  cudaLaunchAttribute pdl_attr[1];
  pdl_attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl_attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t pc = {};
  pc.gridDim = dim3(1 + (q ? (batch * num_heads + 31) / 32 : 0));   // CTA 0 plans, the others quantize q
  pc.blockDim = dim3(1024);
  pc.stream = st;
  pc.attrs = pdl_attr;
  pc.numAttrs = 1;
  return cudaLaunchKernelEx(&pc, plan_kernel, seq_lens, batch, num_heads, groups, hdr, cum, first_req, num_sms, q, qc,
                            qr, sq) ==
                 cudaSuccess
             ? MLA_OK
             : MLA_ERR_CUDA;
}

// one-time per device: dynamic SMEM attribute of a kernel (and the block-pair cluster occupancy)
template <typename K>
static bool ensure_attr(int dev, int which, K kernel, uint32_t smem) {
  std::lock_guard<std::mutex> lk(g_host_mu);
  if (g_dev[dev].attr_done[which]) return true;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return false;
  g_dev[dev].attr_done[which] = true;
  return true;
}

}  // namespace snapmla

using namespace snapmla;

// Debug only (include/snapmla_debug.h): subsequent decodes record a CTA-0 event timeline.
extern "C" void mla_debug_set_trace(unsigned long long* dev_buf) { g_trace.store(dev_buf); }
// Debug / test only: force the kernel for 64 < rows <= 128 (-1 = automatic, the default).
extern "C" void mla_debug_set_pair(int v) { g_kernel.store(v); }
// Debug / test only: rows <= 32 run the swapped-operand kernel (1; -1, the default: for rows <= 16, where it
// is measured faster -- scripts/cmp_small.py) or the single-CTA one (0).
extern "C" void mla_debug_set_small(int v) { g_small.store(v); }
extern "C" size_t mla_decode_workspace_bytes(int batch, int num_heads, int num_sms) {
  if (batch < 0 || num_heads <= 0) return 0;
  if (num_sms <= 0) num_sms = device_num_sms();
  if (num_sms <= 0) num_sms = 148;
  return ws_layout(batch, num_heads, num_sms).total;
}

// The block-pair kernel wins once each cluster streams enough pairs to amortise its longer
// start-up; the host cannot read seq_lens (device-resident), so it decides on the block
// table's extent, an upper bound of the work (scripts/cmp_kernels.py, re-measured after the
// Q-quant moved into the plan launch: crossover at ~8K blocks on the DeepSeek-R1 shape --
// 4K blocks tie or favour the single-CTA kernel, 8K+ the block-pair one;
// profiles/r2x_cmp_kernels_sweep.txt).
constexpr int64_t kBpMinBlocks = 8192;

static mla_status decode_launch(bool bf16, const void* q, const void* kv_fp8, const void* kv_rope,
                                const float* kv_scale, const int32_t* block_table, const int32_t* seq_lens,
                                int batch, int num_heads, int q_len, int kv_lora_rank, int rope_dim,
                                int page_size, int max_pages_per_seq, int64_t num_pages, float softmax_scale,
                                void* workspace, size_t workspace_bytes, mla_stream_t stream) {
  if (batch < 0 || num_heads <= 0 || q_len <= 0 || max_pages_per_seq < 0 || num_pages < 0) return MLA_ERR_SHAPE;
  if (kv_lora_rank != kDc || rope_dim != kDr || page_size != kPage) return MLA_ERR_UNSUPPORTED;
  const int heads = num_heads;
  if ((int64_t)num_heads * q_len > kMaxRows) return MLA_ERR_UNSUPPORTED;
  num_heads *= q_len;   // rows per request from here on
  if (num_pages * kPage >= (int64_t)INT32_MAX) return MLA_ERR_UNSUPPORTED;   // TMA row coordinate is int32
  if (!workspace) return MLA_ERR_WORKSPACE;
  if (batch == 0) return MLA_OK;
  if (!q || !kv_fp8 || !kv_rope || (!bf16 && !kv_scale) || !block_table || !seq_lens) return MLA_ERR_NULL;
  if (!aligned(q, 16) || !aligned(kv_fp8, 128) || !aligned(kv_rope, 128) || (!bf16 && !aligned(kv_scale, 16)) ||
      !aligned(workspace, 256))
    return MLA_ERR_ALIGN;
  if (num_pages == 0) return MLA_ERR_SHAPE;
  const int dev = current_device();
  const int sms = device_num_sms();
  if (dev < 0 || sms <= 0) return MLA_ERR_CUDA;
  const WsLayout wl = ws_layout(batch, num_heads, sms);
  if (workspace_bytes < wl.total) return MLA_ERR_WORKSPACE;
  const int n_ht = (num_heads + kHeadTile - 1) / kHeadTile;
  const int force = g_kernel.load();
  const bool bp = !bf16 && n_ht == 2 &&
                  (force == 1 || (force < 0 && (int64_t)batch * max_pages_per_seq >= kBpMinBlocks));
  const int small = g_small.load();
  const bool sw = !bf16 && num_heads <= 32 && (small == 1 || (small < 0 && num_heads <= 16));
  int groups = sms / n_ht;
  if (bp) {
    if (!ensure_attr(dev, 2, mla_decode_bp_kernel, kBpSmem)) return MLA_ERR_CUDA;
    std::lock_guard<std::mutex> lk(g_host_mu);
    if (g_dev[dev].bp_max_clusters < 0) {
      cudaLaunchConfig_t oc = {};
      oc.gridDim = dim3(2 * groups);
      oc.blockDim = dim3(kBpThreads);
      oc.dynamicSmemBytes = kBpSmem;
      int nc = 0;
      if (cudaOccupancyMaxActiveClusters(&nc, mla_decode_bp_kernel, &oc) != cudaSuccess) return MLA_ERR_CUDA;
      g_dev[dev].bp_max_clusters = nc;
    }
    const int nc = g_dev[dev].bp_max_clusters;
    if (nc > 0 && nc < groups) groups = nc;
  } else if (!sw && !(bf16 ? ensure_attr(dev, 1, mla_decode_kernel<true>, Variant<true>::kSmem)
                    : ensure_attr(dev, 0, mla_decode_kernel<false>, Variant<false>::kSmem))) {
    return MLA_ERR_CUDA;
  }
  CUtensorMap tm_kv, tm_rope;
  const uint64_t rows = (uint64_t)num_pages * kPage;
  if (!cached_tmap(dev, kv_fp8, rows, bf16 ? 1 : 0, &tm_kv) || !cached_tmap(dev, kv_rope, rows, 2, &tm_rope))
    return MLA_ERR_CUDA;

  char* ws = static_cast<char*>(workspace);
  int32_t* hdr = reinterpret_cast<int32_t*>(ws);
  int32_t* cum = reinterpret_cast<int32_t*>(ws + wl.cum);
  int32_t* first = reinterpret_cast<int32_t*>(ws + wl.first);
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* qc = reinterpret_cast<uint8_t*>(ws + wl.qc);
  __nv_bfloat16* qrp = reinterpret_cast<__nv_bfloat16*>(ws + wl.qr);
  float* sqp = reinterpret_cast<float*>(ws + wl.sq);
  if (launch_plan(seq_lens, batch, num_heads, groups, hdr, cum, first, sms, st,
                  bf16 ? nullptr : static_cast<const __nv_bfloat16*>(q), qc, qrp, sqp) != MLA_OK)
    return MLA_ERR_CUDA;

  const uint32_t smem = bp ? kBpSmem : bf16 ? Variant<true>::kSmem : Variant<false>::kSmem;
  DecodeParams prm;
  prm.q = (const __nv_bfloat16*)q;
  prm.kv_fp8 = static_cast<const uint8_t*>(kv_fp8);
  prm.kv_rope = (const __nv_bfloat16*)kv_rope;
  prm.kv_scale = kv_scale;
  prm.block_table = block_table;
  prm.seq_lens = seq_lens;
  prm.ws_hdr = hdr;
  prm.cum = cum;
  prm.first_req = first;
  prm.lse_part = reinterpret_cast<float*>(ws + wl.lse);
  prm.o_part = reinterpret_cast<float*>(ws + wl.o);
  prm.qc = qc;
  prm.qr = qrp;
  prm.sq = sqp;
  prm.batch = batch;
  prm.num_heads = num_heads;
  prm.n_ht = n_ht;
  prm.q_len = q_len;
  prm.heads = heads;
  prm.max_pages = max_pages_per_seq;
  prm.scale_log2 = softmax_scale * 1.4426950408889634f;
  prm.trace = g_trace.load();
  if (sw) return launch_decode_sw(tm_kv, tm_rope, prm, dev, sms, st) == MLA_OK && cudaGetLastError() == cudaSuccess
                     ? MLA_OK
                     : MLA_ERR_CUDA;
  // programmatic dependent launch: the decode CTAs start (barrier init, TMEM
  // alloc, descriptor prefetch) while the plan kernel runs; griddepcontrol.wait
  // in the kernel orders every read of the plan / cache after it.
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(groups * n_ht);
  cfg.blockDim = dim3(bp ? kBpThreads : kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (bp) {
    if (cudaLaunchKernelEx(&cfg, mla_decode_bp_kernel, tm_kv, tm_rope, prm) != cudaSuccess) return MLA_ERR_CUDA;
  } else if (cudaLaunchKernelEx(&cfg, bf16 ? mla_decode_kernel<true> : mla_decode_kernel<false>, tm_kv, tm_rope,
                                prm) != cudaSuccess) {
    return MLA_ERR_CUDA;
  }
  return cudaGetLastError() == cudaSuccess ? MLA_OK : MLA_ERR_CUDA;
}

extern "C" mla_status mla_decode_fp8_ex(const void* q, const uint8_t* kv_fp8, const void* kv_rope,
                                        const float* kv_scale, const int32_t* block_table, const int32_t* seq_lens,
                                        int batch, int num_heads, int q_len, int kv_lora_rank, int rope_dim,
                                        int page_size, int max_pages_per_seq, int64_t num_pages, float softmax_scale,
                                        void* workspace, size_t workspace_bytes, mla_stream_t stream) {
  return decode_launch(false, q, kv_fp8, kv_rope, kv_scale, block_table, seq_lens, batch, num_heads, q_len,
                       kv_lora_rank, rope_dim, page_size, max_pages_per_seq, num_pages, softmax_scale, workspace,
                       workspace_bytes, stream);
}

extern "C" mla_status mla_decode_bf16(const void* q, const void* kv_c, const void* kv_rope,
                                      const int32_t* block_table, const int32_t* seq_lens, int batch, int num_heads,
                                      int q_len, int kv_lora_rank, int rope_dim, int page_size,
                                      int max_pages_per_seq, int64_t num_pages, float softmax_scale, void* workspace,
                                      size_t workspace_bytes, mla_stream_t stream) {
  return decode_launch(true, q, kv_c, kv_rope, nullptr, block_table, seq_lens, batch, num_heads, q_len,
                       kv_lora_rank, rope_dim, page_size, max_pages_per_seq, num_pages, softmax_scale, workspace,
                       workspace_bytes, stream);
}

extern "C" mla_status mla_decode_fp8(const void* q, const uint8_t* kv_fp8, const void* kv_rope,
                                     const float* kv_scale, const int32_t* block_table, const int32_t* seq_lens,
                                     int batch, int num_heads, int kv_lora_rank, int rope_dim, int page_size,
                                     int max_pages_per_seq, int64_t num_pages, float softmax_scale,
                                     void* workspace, size_t workspace_bytes, mla_stream_t stream) {
  if (num_heads > 2 * kHeadTile) return MLA_ERR_UNSUPPORTED;
  return mla_decode_fp8_ex(q, kv_fp8, kv_rope, kv_scale, block_table, seq_lens, batch, num_heads, 1, kv_lora_rank,
                           rope_dim, page_size, max_pages_per_seq, num_pages, softmax_scale, workspace,
                           workspace_bytes, stream);
}
