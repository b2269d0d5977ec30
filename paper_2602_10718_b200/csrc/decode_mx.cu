// NEXT-4(b): the MX-scaled P variant of the decode -- NOT the paper's method.
//
// The paper quantizes P' per 64-token block with sigma_p = M_b / 448 (Algorithm 1
// P:695-696), a non-power-of-two scale, so every block's P'V product must be rescaled into the
// running output by the CUDA cores (O <- gamma O + T: one FMA per output element per block).
// B200's kind::mxf8f6f4.block_scale MMA applies a per-(row, 32-K-chunk) UE8M0 power-of-two scale
// to A inside the tensor core.  With P'_j = E4M3(w_j / 2^e_b), 2^e_b = 2^ceil(log2(M_b / 448))
// (oracle.snapmla.decode_mx), and the exponentials taken against an integer reference per block
// (p_j = 2^(L2_j - R_b), R_b = ceil(max_j L2_j), L2 = logit * log2 e), each block's contribution
// is 2^(e_b + R_b) * P'_b V_b: an exact power of two, absolute (no running max).  O therefore
// accumulates in TMEM through the MMA itself, block after block in increasing order (Appendix C),
// and the only per-row scalar work left is l = sum_b l_b 2^(R_b).  There are no accumulator warps.
//
// Layout: a cluster of two CTAs per key range (64 < rows <= 128 or fewer, padded to M = 128).
// CTA c owns the blocks n of the range with n % 2 == c: it loads their full K tile, runs their
// QK (cta_group::1, M = 128 rows, N = 64, A = q codes in TMEM) and their softmax, writes P' (+ the
// per-row scale bytes) to SMEM and copies it to the peer's SMEM (bulk copy).  Every CTA runs the
// PV of EVERY block for its half of the output dims (CTA c: dims [256c, 256c + 256), N = 256,
// M = 128, K = 64), so O is 128 lanes x 256 columns of its TMEM; a peer block's V half is a 16 KB
// TMA load (an L2 hit: the owner loaded the block).  Both CTAs normalise their O half by the total
// l at the end of a unit (l partials exchanged through DSMEM).
// Warps: 0 TMA, 1 QK, 2 PV, 3 P' export, 4-7 / 8-11 two softmax warpgroups taking the CTA's
// own blocks alternately (ping-pong: each has two block periods for its chain); the 8 softmax
// warps also run the Fused-Q-Quant prologue and the epilogue.
// Limits (documented in snapmla.h): |logit| * log2 e must stay below ~90 so 2^(e_b + R_b) fits
// UE8M0 and the fp32 accumulator; beyond that the scale is clamped.
#include "decode_common.cuh"

namespace snapmla {

constexpr int kMxThreads = 384;
constexpr int kMxWarpTma = 0, kMxWarpQk = 1, kMxWarpPv = 2, kMxWarpX = 3, kMxWarpSm = 4;
// launch 384 x 168 registers; setmaxnreg per SMSP: 40 + 2 x 232 = 504 = 3 x 168
constexpr uint32_t kMxRegsIssue = 40, kMxRegsSm = 232;
constexpr int kMxOwn = 3, kMxPeer = 2, kMxPSlots = 4;
constexpr uint32_t kMxOwnStage = 41984;   // K 32 KB | RoPE 8 KB | sigma_K 256 B
constexpr uint32_t kMxOffR = 32768, kMxOffSc = 40960, kMxOwnTx = 40960 + 256;
constexpr uint32_t kMxPeerStage = 16384;  // V half: two 64-token x 128-dim boxes
constexpr uint32_t kMxPStage = 9216;      // P' 128 x 64 E4M3 (K-major core matrices) | SF tile 512 B
constexpr uint32_t kMxPSf = 8192, kMxPCopy = 8704;
constexpr uint32_t kMxOffBar = 0;                                   // barriers + row scalars first
constexpr uint32_t kMxBarBytes = 6144;
constexpr uint32_t kMxOffQr = kMxOffBar + kMxBarBytes;              // q_r' 128 rows x 128 B, SW128
constexpr uint32_t kMxOffP = kMxOffQr + 16384;
constexpr uint32_t kMxOffOwn = kMxOffP + kMxPSlots * kMxPStage;
constexpr uint32_t kMxOffPeer = kMxOffOwn + kMxOwn * kMxOwnStage;
constexpr uint32_t kMxSmem = kMxOffPeer + kMxPeer * kMxPeerStage + 1024;
static_assert(kMxSmem <= 232448, "shared memory budget (MX kernel)");
// TMEM: O cols 0-255 | q codes 256-383 | S 384-447 | SFA ring 448 + 4 i | SFB 464-471 (all 2^0)
constexpr uint32_t kMxTQ = 256, kMxTS = 384, kMxTSfa = 448, kMxTSfb = 464;

struct BarsMx {
  uint64_t kv_full[kMxOwn], kv_empty[kMxOwn];   // own blocks: TMA -> QK / softmax; PV -> TMA
  uint64_t v_full[kMxPeer], v_empty[kMxPeer];   // peer blocks' V half: TMA -> PV; PV -> TMA
  uint64_t s_full[2], s_empty;                  // QK -> softmax warpgroup (no % 2); softmax -> QK
  // (one s_full per warpgroup: the two warpgroups take alternate phases of the S slot, and a parity
  // wait is only unambiguous for a waiter at most one phase behind)
  uint64_t p_full[kMxPSlots];                   // own P' + scales written (softmax warpgroup)
  uint64_t pp_full[kMxPSlots];                  // peer P' + scales arrived (bulk copy)
  uint64_t p_empty[kMxPSlots];                  // PV of the slot's block done in both CTAs
  uint64_t q_full, q_free, xa_full;
  uint64_t o_ready, o_free;                     // unit's last PV done -> epilogue; epilogue -> PV
  uint64_t lx_full;                             // the peer's l partials of the unit written
  uint32_t tmem_base;
  float crow[128];
  float xa[2][128];
  float lpart[2][128];                          // own-block l of warpgroup 0 / 1 (unit)
  float lpeer[2][2][128];                       // [unit parity][peer warpgroup][row]
};
static_assert(sizeof(BarsMx) <= kMxBarBytes, "barrier region (MX kernel)");
#define BM(field) (bar0 + (uint32_t)offsetof(BarsMx, field))

constexpr uint32_t kIdescQk8M = make_idesc(0, 0, 0, 0, 128, 64);
constexpr uint32_t kIdescQk16M = make_idesc(1, 1, 0, 0, 128, 64);
// block-scaled E4M3 x E4M3 -> F32, scale format E8M0, A K-major, B MN-major, M = 128, N = 256
constexpr uint32_t kIdescPvMx = (1u << 16) | ((256u >> 3) << 17) | (1u << 23) | ((128u >> 4) << 24);

// QK of one block, M = 128 (all rows), N = 64: 16 x f8f6f4 (A = q codes in TMEM) + 4 x f16 (RoPE)
__device__ __forceinline__ void qk_issue_mx(uint32_t dS, uint32_t tQ, uint64_t dK, uint64_t dQr, uint64_t dKr,
                                            uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e, pf, pt;\n\t.reg .b64 a, b;\n\t.reg .b32 z, t;\n\t"
      "mov.b32 z, 0;\n\tsetp.ne.b32 pf, z, 0;\n\tsetp.eq.b32 pt, z, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "add.u32 t, %1, 0;\n\tadd.s64 b, %2, 0;\n\t@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [t], b, %3, pf;\n\t"
      "add.u32 t, %1, 8;\n\tadd.s64 b, %2, 2;\n\t@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [t], b, %3, pt;\n\t"
      "add.u32 t, %1, 16;\n\tadd.s64 b, %2, 4;\n\t@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [t], b, %3, pt;\n\t"
      "add.u32 t, %1, 24;\n\tadd.s64 b, %2, 6;\n\t@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [t], b, %3, pt;\n\t"
      "add.u32 t, %1, 32;\n\tadd.s64 b, %2, 512;\n\t@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [t], b, %3, pt;\n\t"
      "add.u32 t, %1, 40;\n\tadd.s64 b, %2, 514;\n\t@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [t], b, %3, pt;\n\t"
      "add.u32 t, %1, 48;\n\tadd.s64 b, %2, 516;\n\t@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [t], b, %3, pt;\n\t"
      "add.u32 t, %1, 56;\n\tadd.s64 b, %2, 518;\n\t@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [t], b, %3, pt;\n\t"
      "add.u32 t, %1, 64;\n\tadd.s64 b, %2, 1024;\n\t@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [t], b, %3, pt;\n\t"
      "add.u32 t, %1, 72;\n\tadd.s64 b, %2, 1026;\n\t@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [t], b, %3, pt;\n\t"
      "add.u32 t, %1, 80;\n\tadd.s64 b, %2, 1028;\n\t@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [t], b, %3, pt;\n\t"
      "add.u32 t, %1, 88;\n\tadd.s64 b, %2, 1030;\n\t@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [t], b, %3, pt;\n\t"
      "add.u32 t, %1, 96;\n\tadd.s64 b, %2, 1536;\n\t@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [t], b, %3, pt;\n\t"
      "add.u32 t, %1, 104;\n\tadd.s64 b, %2, 1538;\n\t@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [t], b, %3, pt;\n\t"
      "add.u32 t, %1, 112;\n\tadd.s64 b, %2, 1540;\n\t@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [t], b, %3, pt;\n\t"
      "add.u32 t, %1, 120;\n\tadd.s64 b, %2, 1542;\n\t@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [t], b, %3, pt;\n\t"
      "add.s64 a, %4, 0;\n\tadd.s64 b, %5, 0;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %6, pt;\n\t"
      "add.s64 a, %4, 2;\n\tadd.s64 b, %5, 2;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %6, pt;\n\t"
      "add.s64 a, %4, 4;\n\tadd.s64 b, %5, 4;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %6, pt;\n\t"
      "add.s64 a, %4, 6;\n\tadd.s64 b, %5, 6;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %6, pt;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%7];\n\t}"
      ::"r"(dS), "r"(tQ), "l"(dK), "r"(kIdescQk8M), "l"(dQr), "l"(dKr), "r"(kIdescQk16M), "r"(bar)
      : "memory");
}

// PV of one block into O: the block's scale bytes SMEM -> TMEM (tcgen05.cp 32x128b.warpx4: row m
// at lane m % 32 of column m / 32, replicated to the four lane quarters; scripts/mx_probe.cu),
// then 2 x block-scaled MMAs (K = 32 each; A = P', B = V half MN-major, SFB = 2^0).  Commits:
// p_empty of both CTAs (multicast) and this CTA's KV / V slot barrier.
__device__ __forceinline__ void pv_issue_mx(uint32_t dO, uint64_t dP, uint64_t dV, uint64_t dSf, uint32_t tSfa,
                                            uint32_t tSfb, uint32_t acc, uint32_t bar_p, uint32_t bar_kv) {
  asm volatile(
      "{\n\t.reg .pred e, pacc, pt;\n\t.reg .b64 a, b;\n\t"
      "setp.ne.b32 pacc, %6, 0;\n\tsetp.eq.b32 pt, %6, %6;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.cp.cta_group::1.32x128b.warpx4 [%4], %3;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], %1, %2, %7, [%4], [%5], pacc;\n\t"
      "add.s64 a, %1, 256;\n\tadd.s64 b, %2, 256;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], a, b, %7, [%4], [%5], pt;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%8], %10;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%9];\n\t}"
      ::"r"(dO), "l"(dP), "l"(dV), "l"(dSf), "r"(tSfa), "r"(tSfb), "r"(acc), "r"(kIdescPvMx), "r"(bar_p),
      "r"(bar_kv), "h"((uint16_t)3)
      : "memory");
}

__device__ __forceinline__ void mma_commit_local(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
      : "memory");
}

// block ownership inside a CTA pair: block n (the pair's n-th block) is owned by CTA n % 2; the
// owner's own-block counter and the other CTA's peer-block counter are both n / 2.
#ifdef SNAPMLA_MX_OWN0   // debug: CTA 0 owns every block
__device__ __forceinline__ bool mx_own(uint32_t n, uint32_t cta) { return cta == 0; }
__device__ __forceinline__ uint32_t mx_idx(uint32_t n) { return n; }
#else
__device__ __forceinline__ bool mx_own(uint32_t n, uint32_t cta) { return (n & 1) == cta; }
__device__ __forceinline__ uint32_t mx_idx(uint32_t n) { return n >> 1; }
#endif

// 2^k for an integer k in [-126, 127] (exact)
__device__ __forceinline__ float exp2i(int k) { return __uint_as_float((uint32_t)(k + 127) << 23); }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kMxThreads, 1)
    mla_decode_mx_kernel(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_rope,
                         const DecodeParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t bar0 = sbase + kMxOffBar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cta = cluster_ctarank();

  if (threadIdx.x == 0) {
    for (int i = 0; i < kMxOwn; ++i) {
      mbar_init(BM(kv_full) + 8 * i, 1);
      mbar_init(BM(kv_empty) + 8 * i, 1);
    }
    for (int i = 0; i < kMxPeer; ++i) {
      mbar_init(BM(v_full) + 8 * i, 1);
      mbar_init(BM(v_empty) + 8 * i, 1);
    }
    mbar_init(BM(s_full), 1);
    mbar_init(BM(s_full) + 8, 1);
    mbar_init(BM(s_empty), 4 * kArriveMul);
    for (int i = 0; i < kMxPSlots; ++i) {
      mbar_init(BM(p_full) + 8 * i, 4 * kArriveMul);
      mbar_init(BM(pp_full) + 8 * i, 1);
      mbar_init(BM(p_empty) + 8 * i, 2);
    }
    mbar_init(BM(q_full), 8 * kArriveMul);
    mbar_init(BM(q_free), 1);
    mbar_init(BM(xa_full), 8 * kArriveMul);
    mbar_init(BM(o_ready), 1);
    mbar_init(BM(o_free), 8 * kArriveMul);
    mbar_init(BM(lx_full), 8);
    fence_barrier_init();
  }
  if (warp == kMxWarpTma && lane == 0) {
    tma_prefetch_desc(&tm_kv);
    tma_prefetch_desc(&tm_rope);
  }
  if (warp == kMxWarpQk) tmem_alloc(BM(tmem_base), 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = lds_u32(BM(tmem_base));

  pdl_wait();
  pdl_launch_dependents();
  const int g = blockIdx.x / 2;
  const int per = p.ws_hdr[H_PER], total = p.ws_hdr[H_TOTAL], groups = p.ws_hdr[H_GROUPS];
  const int lo = g * per;
  const bool has_work = g < groups && lo < total;
  const int hi = min(total, lo + per);
  UnitIter it{p.cum, lo, hi, g, has_work ? __ldg(p.first_req + g) : 0, has_work ? p.batch : 0};
  Unit u;

  if (warp < kMxWarpSm) {
    regs_dec<kMxRegsIssue>();
    if (warp == kMxWarpTma) {
      // ============================ TMA producer ============================
      if (lane == 0) {
        const uint64_t pol = l2_policy_evict_first();
        uint32_t n = 0;
        while (it.next(u)) {
          const int32_t* bt = p.block_table + (int64_t)u.b * p.max_pages;
          prefetch_block_table(bt, u.k0, u.k1);
          for (int j = u.k0; j < u.k1; ++j, ++n) {
            const int row = __ldg(bt + j) * kPage;
            if (mx_own(n, cta)) {   // own block: the full K tile (QK) + RoPE + sigma_K
              const uint32_t no = mx_idx(n), os = no % kMxOwn;
              mbar_wait_backoff(BM(kv_empty) + 8 * os, ((no / kMxOwn) & 1) ^ 1);
              const uint32_t slot = sbase + kMxOffOwn + os * kMxOwnStage, full = BM(kv_full) + 8 * os;
              mbar_arrive_expect_tx(full, kMxOwnTx);
#pragma unroll
              for (int c = 0; c < 4; ++c) tma_load_2d(slot + c * kBoxBytes, &tm_kv, full, c * 128, row, pol);
              tma_load_2d(slot + kMxOffR, &tm_rope, full, 0, row, pol);
              bulk_load(slot + kMxOffSc, p.kv_scale + (int64_t)row, 256, full, pol);
            } else {                // peer block: this CTA's dims half of V
              const uint32_t np = mx_idx(n), vs = np % kMxPeer;
              mbar_wait_backoff(BM(v_empty) + 8 * vs, ((np / kMxPeer) & 1) ^ 1);
              const uint32_t slot = sbase + kMxOffPeer + vs * kMxPeerStage, full = BM(v_full) + 8 * vs;
              mbar_arrive_expect_tx(full, kMxPeerStage);
              tma_load_2d(slot, &tm_kv, full, 256 * cta, row, pol);
              tma_load_2d(slot + kBoxBytes, &tm_kv, full, 256 * cta + 128, row, pol);
            }
          }
        }
      }
    } else if (warp == kMxWarpQk) {
      // ================================ QK (own blocks) ================================
      const uint64_t dQr = make_smem_desc(sbase + kMxOffQr, 16, 1024, LAYOUT_SW128);
      uint32_t n = 0, unit = 0;
      while (it.next(u)) {
        mbar_wait(BM(q_full), unit & 1, 2, unit);
        for (int j = u.k0; j < u.k1; ++j, ++n) {
          if (!mx_own(n, cta)) continue;
          const uint32_t no = mx_idx(n), os = no % kMxOwn;
          mbar_wait(BM(kv_full) + 8 * os, (no / kMxOwn) & 1, 3, n);
          if (lane == 0) TRACE(TR_C1, n);
#ifdef SNAPMLA_HANG_CHECK
          {   // debug: dump the barrier words if s_empty does not complete
            const long long t0 = clock64();
            while (!mbar_try_wait(BM(s_empty), (no & 1) ^ 1)) {
              if (clock64() - t0 > (1ll << 30)) {
                if (lane == 0) {
                  for (int i = 0; i < 32; ++i) {
                    unsigned long long raw;
                    asm volatile("ld.shared.b64 %0, [%1];" : "=l"(raw) : "r"(bar0 + 8 * i));
                    printf("MXDUMP blk %d n %d word %d off %d raw 0x%016llx\n", blockIdx.x, n, i, 8 * i, raw);
                  }
                }
                __syncwarp();
                __trap();
              }
            }
          }
#endif
          mbar_wait(BM(s_empty), (no & 1) ^ 1, 4, n);
          tc_fence_after();
          if (lane == 0) TRACE(TR_QK, n);
          const uint32_t kv = sbase + kMxOffOwn + os * kMxOwnStage;
          qk_issue_mx(tmem + kMxTS, tmem + kMxTQ, make_smem_desc(kv, 16, 1024, LAYOUT_SW128), dQr,
                      make_smem_desc(kv + kMxOffR, 16, 1024, LAYOUT_SW128), BM(s_full) + 8 * (no & 1));
        }
        mma_commit_local(BM(q_free));
        ++unit;
      }
    } else if (warp == kMxWarpPv) {
      // ============================ PV (every block, this CTA's dims half) ============================
      // SFB (all 2^0) once: 8 columns of every lane
      {
        uint32_t v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0x7F7F7F7Fu;
        // this warp (SMSP 2) reaches lanes 64-95 only: SFB is read per N column at lane n % 32
        // of column n / 32 with all four quarters replicated -> every quarter needs it; the
        // softmax warps of the other quarters write theirs in the prologue (below)
        tmem_st_32x32b_x32(tmem + ((uint32_t)(32 * (warp & 3)) << 16) + kMxTSfb, v);
        tmem_wait_st();
      }
      uint32_t n = 0, unit = 0;
      while (it.next(u)) {
        if (unit > 0) mbar_wait(BM(o_free), (unit - 1) & 1, 5, unit);   // epilogue read O
        mbar_wait(BM(q_full), unit & 1, 6, unit);                         // SFB quarters written (first unit)
        tc_fence_after();
        for (int j = u.k0; j < u.k1; ++j, ++n) {
          const uint32_t ps = n % kMxPSlots;
          uint32_t dv, bar_kv;
          if (mx_own(n, cta)) {
            const uint32_t no = mx_idx(n), os = no % kMxOwn;
            mbar_wait(BM(p_full) + 8 * ps, (n / kMxPSlots) & 1, 7, n);
            dv = sbase + kMxOffOwn + os * kMxOwnStage + 2 * cta * kBoxBytes;
            bar_kv = BM(kv_empty) + 8 * os;
          } else {
            const uint32_t np = mx_idx(n), vs = np % kMxPeer;
            mbar_wait(BM(pp_full) + 8 * ps, (n / kMxPSlots) & 1, 8, n);
            mbar_wait(BM(v_full) + 8 * vs, (np / kMxPeer) & 1, 9, n);
            dv = sbase + kMxOffPeer + vs * kMxPeerStage;
            bar_kv = BM(v_empty) + 8 * vs;
          }
          tc_fence_after();
          if (lane == 0) TRACE(TR_PVL, n);
          if (lane == 0) TRACE(TR_C2, n);
          const uint32_t pslot = sbase + kMxOffP + ps * kMxPStage;
          pv_issue_mx(tmem, make_smem_desc(pslot, 2048, 128, LAYOUT_NONE),
                      make_smem_desc(dv, kBoxBytes, 1024, LAYOUT_SW128),
                      make_smem_desc(pslot + kMxPSf, 16, 128, LAYOUT_NONE), tmem + kMxTSfa + 4 * (n % 4),
                      tmem + kMxTSfb, j > u.k0 ? 1u : 0u, BM(p_empty) + 8 * ps, bar_kv);
        }
        mma_commit_local(BM(o_ready));
        ++unit;
      }
    } else {
      // ============ P' export: own block's P' + scale bytes -> the peer's slot (bulk copy) ============
      const uint32_t peer = cta ^ 1u;
      uint32_t n = 0;
      while (it.next(u)) {
        for (int j = u.k0; j < u.k1; ++j, ++n) {
          if (!mx_own(n, cta)) continue;
          const uint32_t ps = n % kMxPSlots;
          mbar_wait(BM(p_full) + 8 * ps, (n / kMxPSlots) & 1, 10, n);
          if (lane == 0) {
            const uint32_t src = sbase + kMxOffP + ps * kMxPStage;
            const uint32_t pbar = mapa_shared(BM(pp_full) + 8 * ps, peer);
            mbar_arrive_expect_tx_cluster(pbar, kMxPCopy);
            bulk_copy_s2c(mapa_shared(src, peer), src, kMxPCopy, pbar);
          }
          __syncwarp();
        }
      }
    }
  } else {
    regs_inc<kMxRegsSm>();
    // ===== softmax warpgroups (own blocks, alternately), Q-quant prologue, epilogue =====
    const int w = (warp - kMxWarpSm) >> 2;   // warpgroup
    const int k = warp & 3;                  // TMEM lane quarter
    const int r = 32 * k + lane;             // query row (M = 128 layout: lane = row)
    const bool row_ok = r < p.num_heads;
    const uint32_t lane_base = (uint32_t)(32 * k) << 16;
    const uint32_t peer = cta ^ 1u;
    uint32_t n = 0, unit = 0;
    // SFB: this thread's quarter of the (replicated) 2^0 scale columns
    if (w == 0) {
      uint32_t v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = 0x7F7F7F7Fu;
      tmem_st_32x32b_x32(tmem + lane_base + kMxTSfb, v);
      tmem_wait_st();
    }
    while (it.next(u)) {
      // ---------------- Fused-Q-Quant prologue (a2): warpgroup w quantizes codes [256 w, 256 w + 256)
      if (unit > 0) mbar_wait(BM(q_free), (unit - 1) & 1, 11, unit);   // previous unit's QK done
      const uint4* qrow = reinterpret_cast<const uint4*>(p.q + ((int64_t)u.b * p.num_heads + (row_ok ? r : 0)) * kDqk);
      {
        float amax = 0.f;
#pragma unroll 4
        for (int i = 0; i < 32; ++i) {
          const uint4 v = row_ok ? __ldg(qrow + 32 * w + i) : make_uint4(0, 0, 0, 0);
          const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(hv[e]);
            amax = fmaxf(amax, fmaxf(fabsf(f.x), fabsf(f.y)));
          }
        }
        sts_f32(BM(xa) + 512 * w + 4 * r, amax);
        warp_arrive(BM(xa_full), lane);
        mbar_wait(BM(xa_full), unit & 1, 12, unit);
        const float am = fmaxf(lds_f32(BM(xa) + 4 * r), lds_f32(BM(xa) + 512 + 4 * r));
        const float sq = fmaxf(__fdiv_rn(am, 448.0f), kSigmaMin);
        const float rsq = __frcp_rn(sq);
#pragma unroll 1
        for (int ci = 0; ci < 2; ++ci) {   // 128 codes per store: TMEM columns kMxTQ + 64 w + 32 ci
          uint32_t qa[32];
#pragma unroll
          for (int g8 = 0; g8 < 8; ++g8) {
            uint4 v2[2];
            v2[0] = row_ok ? __ldg(qrow + 32 * w + 16 * ci + 2 * g8) : make_uint4(0, 0, 0, 0);
            v2[1] = row_ok ? __ldg(qrow + 32 * w + 16 * ci + 2 * g8 + 1) : make_uint4(0, 0, 0, 0);
            const __nv_bfloat162* a = reinterpret_cast<const __nv_bfloat162*>(v2);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f0 = __bfloat1622float2(a[2 * e]), f1 = __bfloat1622float2(a[2 * e + 1]);
              const float2 d0 = div_by2(f0, sq, rsq), d1 = div_by2(f1, sq, rsq);
              qa[4 * g8 + e] = cvt4_e4m3(d0.x, d0.y, d1.x, d1.y);
            }
          }
          tmem_st_32x32b_x32(tmem + lane_base + kMxTQ + 64 * w + 32 * ci, qa);
        }
        tmem_wait_st();
        if (w == 0) {   // q_r' = bf16(q_r / sigma_q) (SW128 rows of 128 B) and c = sigma_q scale log2(e)
          sts_f32(BM(crow) + 4 * r, sq * p.scale_log2);
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint4 v = row_ok ? __ldg(qrow + 64 + c) : make_uint4(0, 0, 0, 0);
            const __nv_bfloat162* a = reinterpret_cast<const __nv_bfloat162*>(&v);
            uint32_t wd[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = __bfloat1622float2(a[e]);
              __nv_bfloat162 o2 = __halves2bfloat162(__float2bfloat16_rn(div_by(f.x, sq, rsq)),
                                                     __float2bfloat16_rn(div_by(f.y, sq, rsq)));
              wd[e] = *reinterpret_cast<uint32_t*>(&o2);
            }
            sts_u4(sbase + kMxOffQr + r * 128 + ((c ^ (r & 7)) << 4), wd[0], wd[1], wd[2], wd[3]);
          }
        }
        fence_proxy_async_smem();
        tc_fence_before();
        warp_arrive(BM(q_full), lane);
      }
      named_bar_sync(1, 256);   // crow of every row written (softmax warps only)
      const float c_row = lds_f32(BM(crow) + 4 * r);
      const int L = __ldg(p.seq_lens + u.b) - (p.q_len - 1 - (row_ok ? r : 0) / p.heads);
      float lown = 0.f;   // this warpgroup's sum over its blocks of l_b 2^R_b
      float tt[64];
      for (int j = u.k0; j < u.k1; ++j, ++n) {
        if (!mx_own(n, cta)) continue;
        const uint32_t no = mx_idx(n);
        if ((int)(no & 1) != w) continue;   // the other warpgroup's block
        const uint32_t os = no % kMxOwn, ps = n % kMxPSlots;
        mbar_wait(BM(s_full) + 8 * w, (no >> 1) & 1, 13, n);
        tc_fence_after();
        tmem_ld_32x32b_x32(tmem + lane_base + kMxTS, *reinterpret_cast<uint32_t(*)[32]>(tt));
        tmem_ld_32x32b_x32(tmem + lane_base + kMxTS + 32, *reinterpret_cast<uint32_t(*)[32]>(tt + 32));
        tmem_wait_ld();
        if ((threadIdx.x & 127) == 0) TRACE(TR_SM_IN, n);
        tc_fence_before();
        warp_arrive(BM(s_empty), lane);
        mbar_wait(BM(kv_full) + 8 * os, (no / kMxOwn) & 1, 14, n);   // sigma_K visible (complete long ago)
        const uint32_t sk = sbase + kMxOffOwn + os * kMxOwnStage + kMxOffSc;
#pragma unroll
        for (int e0 = 0; e0 < 64; e0 += 16) {
          float4 s4[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) s4[i] = lds_f4(sk + 4 * (e0 + 4 * i));
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int e = e0 + 4 * i;
            const float2 a = __fmul2_rn(make_float2(tt[e], tt[e + 1]), make_float2(s4[i].x, s4[i].y));
            const float2 b = __fmul2_rn(make_float2(tt[e + 2], tt[e + 3]), make_float2(s4[i].z, s4[i].w));
            tt[e] = a.x * c_row;
            tt[e + 1] = a.y * c_row;
            tt[e + 2] = b.x * c_row;
            tt[e + 3] = b.y * c_row;
          }
        }
        const int nvalid = L - j * kBc;
        if (nvalid < 64) {
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
        const float mx = fmax3(fmax3(m0, m1, m2), fmax3(m3, tt[60], tt[61]), fmaxf(tt[62], tt[63]));   // max L2
        // integer reference R_b = ceil(max L2) (clamped; a fully masked row block gives R = 0, P' = 0)
        const float Rb = mx == -INFINITY ? 0.f : fminf(fmaxf(ceilf(mx), -100.f), 100.f);
        float2 ls0 = make_float2(0.f, 0.f), ls1 = make_float2(0.f, 0.f);
        float mb0 = 0.f, mb1 = 0.f;
        float4 s4b[4];
#pragma unroll
        for (int e = 0; e < 64; e += 4) {
          if ((e & 15) == 0) {
#pragma unroll
            for (int i = 0; i < 4; ++i) s4b[i] = lds_f4(sk + 4 * (e + 4 * i));
          }
          const float4 s4 = s4b[(e & 15) / 4];
          const float2 a0 = __fadd2_rn(make_float2(tt[e], tt[e + 1]), make_float2(-Rb, -Rb));
          const float2 a1 = __fadd2_rn(make_float2(tt[e + 2], tt[e + 3]), make_float2(-Rb, -Rb));
          const float2 p0 = make_float2(ex2_approx(a0.x), ex2_approx(a0.y));
          const float2 p1 = make_float2(ex2_approx(a1.x), ex2_approx(a1.y));
          ls0 = __fadd2_rn(ls0, p0);
          ls1 = __fadd2_rn(ls1, p1);
          const float2 w0 = __fmul2_rn(p0, make_float2(s4.x, s4.y));
          const float2 w1 = __fmul2_rn(p1, make_float2(s4.z, s4.w));
          tt[e] = w0.x;
          tt[e + 1] = w0.y;
          tt[e + 2] = w1.x;
          tt[e + 3] = w1.y;
          mb0 = fmax3(mb0, w0.x, w0.y);
          mb1 = fmax3(mb1, w1.x, w1.y);
        }
        const float lb = (ls0.x + ls0.y) + (ls1.x + ls1.y);
        const float mb = fmaxf(mb0, mb1);
        // 2^e = 2^ceil(log2(M_b / 448)): M_b / 448 <= 2^e, so P' = E4M3(w 2^-e) <= 448
        int eb = 0;
        if (mb > 0.f) {
          const uint32_t xb = __float_as_uint(__fdiv_rn(mb, 448.0f));
          eb = (int)((xb >> 23) & 0xFF) - 127 + ((xb & 0x7FFFFF) != 0 ? 1 : 0);
        }
        const float inv = exp2i(-eb);
        uint32_t pw[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float2 a = __fmul2_rn(make_float2(tt[4 * e], tt[4 * e + 1]), make_float2(inv, inv));
          const float2 b = __fmul2_rn(make_float2(tt[4 * e + 2], tt[4 * e + 3]), make_float2(inv, inv));
          pw[e] = cvt4_e4m3(a.x, a.y, b.x, b.y);
        }
        const int Ri = (int)Rb;
        const int E = max(-127, min(127, eb + Ri));   // this block's power-of-two scale of P'_b V
        lown += lb * exp2i(Ri);
        if ((threadIdx.x & 127) == 0) TRACE(TR_S3, n);
        mbar_wait(BM(p_empty) + 8 * ps, ((n / kMxPSlots) & 1) ^ 1, 15, n);
        if ((threadIdx.x & 127) == 0) TRACE(TR_S4, n);
        const uint32_t pslot = sbase + kMxOffP + ps * kMxPStage;
        const uint32_t pdst = pslot + r * 16;   // byte(row, tok) = (tok / 16) * 2048 + row * 16 + tok % 16
#pragma unroll
        for (int c = 0; c < 4; ++c) sts_u4(pdst + c * 2048, pw[4 * c], pw[4 * c + 1], pw[4 * c + 2], pw[4 * c + 3]);
        sts_f32(pslot + kMxPSf + lane * 16 + k * 4, __uint_as_float((uint32_t)(E + 127) * 0x01010101u));
        fence_proxy_async_smem();
        warp_arrive(BM(p_full) + 8 * ps, lane);
        if ((threadIdx.x & 127) == 0) TRACE(TR_SM_OUT, n);
      }
      // ---------------- epilogue (a9): l partials -> local SMEM and the peer's SMEM; O / l
      const uint32_t par = unit & 1;
      sts_f32(BM(lpart) + 512 * w + 4 * r, lown);
      st_cluster_f32(mapa_shared(BM(lpeer) + (par * 2 + w) * 512 + 4 * r, peer), lown);
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa_shared(BM(lx_full), peer));   // release: publishes the stores
      named_bar_sync(1, 256);
      mbar_wait(BM(o_ready), par, 16, unit);
      mbar_wait_cluster(BM(lx_full), par, 17, unit);
      tc_fence_after();
      const float ltot = lds_f32(BM(lpart) + 4 * r) + lds_f32(BM(lpart) + 512 + 4 * r) +
                         lds_f32(BM(lpeer) + (par * 2) * 512 + 4 * r) + lds_f32(BM(lpeer) + (par * 2 + 1) * 512 + 4 * r);
      const float f = ltot > 0.f ? 1.0f / ltot : 0.f;
      const int ht = r / kHeadTile;
      const int64_t prow = ((int64_t)u.slot * p.n_ht + ht) * kHeadTile + (r % kHeadTile);
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {   // this warpgroup's 128 of the CTA's 256 output dims
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem + lane_base + 128 * w + 32 * c, v);
        tmem_wait_ld();
        if (row_ok) {
          float* dst = p.o_part + prow * kDc + 256 * cta + 128 * w + 32 * c;
#pragma unroll
          for (int e = 0; e < 32; e += 4)
            *reinterpret_cast<float4*>(dst + e) =
                make_float4(__uint_as_float(v[e]) * f, __uint_as_float(v[e + 1]) * f, __uint_as_float(v[e + 2]) * f,
                            __uint_as_float(v[e + 3]) * f);
        }
      }
      if (row_ok && cta == 0 && w == 0) p.lse_part[prow] = ltot > 0.f ? log2f(ltot) * 0.69314718055994531f : -INFINITY;
      tc_fence_before();
      warp_arrive(BM(o_free), lane);
      ++unit;
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == kMxWarpQk) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace snapmla

using namespace snapmla;

extern "C" mla_status mla_decode_fp8_mx(const void* q, const uint8_t* kv_fp8, const void* kv_rope,
                                        const float* kv_scale, const int32_t* block_table, const int32_t* seq_lens,
                                        int batch, int num_heads, int q_len, int kv_lora_rank, int rope_dim,
                                        int page_size, int max_pages_per_seq, int64_t num_pages, float softmax_scale,
                                        void* workspace, size_t workspace_bytes, mla_stream_t stream) {
  if (batch < 0 || num_heads <= 0 || q_len <= 0 || max_pages_per_seq < 0 || num_pages < 0) return MLA_ERR_SHAPE;
  if (kv_lora_rank != kDc || rope_dim != kDr || page_size != kPage) return MLA_ERR_UNSUPPORTED;
  const int heads = num_heads;
  if ((int64_t)num_heads * q_len > 2 * kHeadTile) return MLA_ERR_UNSUPPORTED;   // one 128-row tile
  num_heads *= q_len;
  if (num_pages * kPage >= (int64_t)INT32_MAX) return MLA_ERR_UNSUPPORTED;
  if (!workspace) return MLA_ERR_WORKSPACE;
  if (batch == 0) return MLA_OK;
  if (!q || !kv_fp8 || !kv_rope || !kv_scale || !block_table || !seq_lens) return MLA_ERR_NULL;
  if (!aligned(q, 16) || !aligned(kv_fp8, 128) || !aligned(kv_rope, 128) || !aligned(kv_scale, 16) ||
      !aligned(workspace, 256))
    return MLA_ERR_ALIGN;
  if (num_pages == 0) return MLA_ERR_SHAPE;
  const int dev = current_device();
  const int sms = device_num_sms();
  if (dev < 0 || sms <= 0) return MLA_ERR_CUDA;
  const WsLayout wl = ws_layout(batch, num_heads, sms);
  if (workspace_bytes < wl.total) return MLA_ERR_WORKSPACE;
  const int n_ht = (num_heads + kHeadTile - 1) / kHeadTile;
  static std::atomic<int> max_clusters[64];
  static std::atomic<bool> attr_done[64];
  if (!attr_done[dev].load()) {
    if (cudaFuncSetAttribute(mla_decode_mx_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMxSmem) !=
        cudaSuccess)
      return MLA_ERR_CUDA;
    cudaLaunchConfig_t oc = {};
    oc.gridDim = dim3(sms);
    oc.blockDim = dim3(kMxThreads);
    oc.dynamicSmemBytes = kMxSmem;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, mla_decode_mx_kernel, &oc) != cudaSuccess) return MLA_ERR_CUDA;
    max_clusters[dev].store(nc);
    attr_done[dev].store(true);
  }
  int groups = sms / 2;
  const int nc = max_clusters[dev].load();
  if (nc > 0 && nc < groups) groups = nc;
  CUtensorMap tm_kv, tm_rope;
  const uint64_t rows = (uint64_t)num_pages * kPage;
  if (!cached_tmap(dev, kv_fp8, rows, 0, &tm_kv) || !cached_tmap(dev, kv_rope, rows, 2, &tm_rope)) return MLA_ERR_CUDA;
  char* ws = static_cast<char*>(workspace);
  int32_t* hdr = reinterpret_cast<int32_t*>(ws);
  int32_t* cum = reinterpret_cast<int32_t*>(ws + wl.cum);
  int32_t* first = reinterpret_cast<int32_t*>(ws + wl.first);
  cudaStream_t st = (cudaStream_t)stream;
  if (launch_plan(seq_lens, batch, num_heads, groups, hdr, cum, first, sms, st) != MLA_OK) return MLA_ERR_CUDA;
  DecodeParams prm;
  prm.q = (const __nv_bfloat16*)q;
  prm.kv_fp8 = kv_fp8;
  prm.kv_rope = (const __nv_bfloat16*)kv_rope;
  prm.kv_scale = kv_scale;
  prm.block_table = block_table;
  prm.seq_lens = seq_lens;
  prm.ws_hdr = hdr;
  prm.cum = cum;
  prm.first_req = first;
  prm.lse_part = reinterpret_cast<float*>(ws + wl.lse);
  prm.o_part = reinterpret_cast<float*>(ws + wl.o);
  prm.qc = nullptr;   // the MX kernel quantizes q in its own prologue
  prm.qr = nullptr;
  prm.sq = nullptr;
  prm.batch = batch;
  prm.num_heads = num_heads;
  prm.n_ht = n_ht;
  prm.q_len = q_len;
  prm.heads = heads;
  prm.max_pages = max_pages_per_seq;
  prm.scale_log2 = softmax_scale * 1.4426950408889634f;
  prm.trace = g_trace.load();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * groups);
  cfg.blockDim = dim3(kMxThreads);
  cfg.dynamicSmemBytes = kMxSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, mla_decode_mx_kernel, tm_kv, tm_rope, prm) != cudaSuccess) return MLA_ERR_CUDA;
  return cudaGetLastError() == cudaSuccess ? MLA_OK : MLA_ERR_CUDA;
}
