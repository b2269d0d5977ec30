// a2-a9 for few query rows (rows = q_len x heads <= 32, e.g. DeepSeek-R1 TP8: 16 heads per rank):
// the same method as decode.cu (Alg.1, block-wise P quantization P:237-249, Appendix C
// order P:759-764), with the MMA operand roles swapped so that the head count is the MMA's N:
//
//   QK   S^T (64 tokens x N heads) = K (64 x 576, the TMA'd tile) . Q^T      M = 64, N = 16 / 32
//   PV   O^T (512 dims x N heads)  = V^T (4 x 128 dims, the SAME FP8 tile read MN-major) . P'^T
//                                                                             M = 128, N = 16 / 32
// The decode.cu kernels put the rows on M (>= 64), so 16 heads pad 48 of every 64 MMA rows and
// the accumulators / softmax carry 4x the work.  Here the tensor core does N/64 of that work and
// one thread owns ONE token (softmax) or one output dim (accumulators) across the heads.
//
// DESIGN.md §7.11.  Warp roles (16 warps, one CTA per SM, a contiguous range of key blocks from
// the plan kernel with one head tile):
//   warps 0-3    softmax (a second group, warps 8-11, takes every other block, so two blocks'
//   (8-11)       reductions are in flight): thread = (token 16 w + lane % 16, heads (lane / 16) N/2 + [0, N/2)):
//                Q-quant prologue (Fused-Q-Quant), descale, per-head block max and M_b by
//                in-warp transpose-butterfly reductions + one SMEM exchange across the 4 warps,
//                p, w = p sigma_K, P'^T = E4M3(w 448 / M_b) bytes; warp 0 lane h runs head h's
//                Alg.1 recurrence (m, sigma, l, gamma; state chained in SMEM across the groups in
//                block order) and the epilogue factors
//   warps 4-7    accumulators: O^T <- gamma O^T + T^T per head column; thread = (dim, N heads)
//                for all 4 dim tiles; epilogue o = O f
//   warp 12      TMA producer (as decode.cu: 4 FP8 boxes + RoPE box + sigma_K per block)
//   warp 13      QK issuer (A = K tile, B = q codes / q_r' from SMEM)
//   warp 14      PV issuer (A = V^T MN-major, B = P'^T K-major), 3-slot TMEM ring of T^T
#include "decode_common.cuh"

namespace snapmla {

constexpr int kSwThreads = 512;
constexpr int kSwWarpAcc = 4, kSwWarpTma = 12, kSwWarpQk = 13, kSwWarpPv = 14;
constexpr int kSwSSlots = 4, kSwPSlots = 4, kSwTSlots = 3;
constexpr uint32_t kSwStage = 41984;                 // as decode.cu: 4 FP8 boxes | RoPE box | sigma_K
constexpr uint32_t kSwTx = kBc * (kDc + 2 * kDr + 4);
constexpr uint32_t kSwOffScLo = 5 * kBoxBytes, kSwOffScHi = 5 * kBoxBytes + 144;

template <int N> struct SwCfg {
  static constexpr int kSlots = N == 16 ? 5 : 4;     // KV ring depth (SMEM budget)
  static constexpr uint32_t kQcBox = N * 128;        // q codes: 4 SW128 boxes of N rows x 128 B
  static constexpr uint32_t kOffQc = kSlots * kSwStage;
  static constexpr uint32_t kOffQr = kOffQc + 4 * kQcBox;
  static constexpr uint32_t kPBytes = N * 64;        // P'^T: N heads x 64 tokens, K-major core matrices
  static constexpr uint32_t kOffP = kOffQr + N * 128;
  static constexpr uint32_t kOffBar = kOffP + kSwPSlots * kPBytes;
  static constexpr uint32_t kSmem = kOffBar + 6144 + 1024;
  // TMEM: S^T slot s at cols N s (M = 64 layout: token m at lane m % 16 + 32 (m / 16)), then the
  // T^T ring, slot t at cols 4 N + 4 N t (dim tile d at + N d; lane = dim % 128)
  static constexpr uint32_t kTmemT = 4 * N;
  static constexpr uint32_t kIdescQk8 = make_idesc(0, 0, 0, 0, 64, N);
  static constexpr uint32_t kIdescQk16 = make_idesc(1, 1, 0, 0, 64, N);
  static constexpr uint32_t kIdescPv = make_idesc(0, 0, 1, 0, 128, N);   // V^T MN-major, P'^T K-major
};
static_assert(SwCfg<16>::kSmem <= 232448 && SwCfg<32>::kSmem <= 232448, "shared memory budget (swapped kernel)");

struct BarsW {
  uint64_t kv_full[5], kv_empty[5];
  uint64_t s_full[kSwSSlots], s_empty[kSwSSlots];
  uint64_t p_full[kSwPSlots], p_empty[kSwPSlots];
  uint64_t t_full[kSwTSlots], t_free[kSwTSlots];
  uint64_t q_full, q_free, fin_full, fin_empty, bk_done;
  uint32_t tmem_base;
  alignas(16) float cq[32];                  // c = sigma_q * scale * log2(e) per row
  alignas(16) float red[2][3][4][32];        // [softmax group][block max of t, M_b, l_b][softmax warp][head]
  alignas(16) float bks[4][32];              // Alg.1 state per head between blocks: m_ref, m_O, sigma_O, l_run
  alignas(16) float gam[kSwPSlots][32];      // O <- gamma O + delta T per head
  alignas(16) float del[kSwPSlots][32];
  alignas(16) float skip[kSwPSlots];         // 1: some head of the block is skipped (delta = 0)
  alignas(16) float fin[32];                 // epilogue factor per head
};
constexpr uint32_t kSwBarBytes = 6144;
static_assert(sizeof(BarsW) <= kSwBarBytes, "barrier region (swapped kernel)");
#define BW(field) (bar0 + (uint32_t)offsetof(BarsW, field))

// Reduce NH per-thread values over the 16 lanes of a half warp (transpose butterfly: each stage
// hands half of the remaining heads to the partner lane).  Returns lane's result for head `head`
// (lanes l and l ^ (16 / NH - 1) ... share a head when NH < 16).
template <int NH, bool kMax>
__device__ __forceinline__ float tb_reduce(float (&v)[NH], int lane, int& head) {
  int base = 0;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int o = 8 >> s;
    const int cnt = NH >> s;   // values still held (compile-time after unrolling)
    if (cnt > 1) {
      const int half = cnt >> 1;
      const bool hi = (lane & o) != 0;
#pragma unroll
      for (int i = 0; i < half; ++i) {
        const float send = hi ? v[i] : v[i + half];
        const float keep = hi ? v[i + half] : v[i];
        const float got = __shfl_xor_sync(0xffffffffu, send, o);
        v[i] = kMax ? fmaxf(keep, got) : keep + got;
      }
      if (hi) base += half;
    } else {
      const float got = __shfl_xor_sync(0xffffffffu, v[0], o);
      v[0] = kMax ? fmaxf(v[0], got) : v[0] + got;
    }
  }
  head = base;
  return v[0];
}

template <int N>
__global__ void __launch_bounds__(kSwThreads, 1)
    mla_decode_sw_kernel(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_rope,
                         const DecodeParams p) {
  using C = SwCfg<N>;
  constexpr int NH = N / 2;
  // two softmax groups (warps 0-3, 8-11) take alternate blocks, 4 accumulator warps (4-7) hold all
  // 4 dim tiles (N = 32: 128 O registers each, via setmaxnreg: per SMSP 2 x 144 + 184 + 40 = 512)
  constexpr int kGroups = 2;
  constexpr int kAccW = 4;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t bar0 = sbase + C::kOffBar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool is_sm = warp < 4 || (kGroups == 2 && warp >= 8 && warp < 12);
  const int grp = warp < 4 ? 0 : 1;

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::kSlots; ++i) {
      mbar_init(BW(kv_full) + 8 * i, 1);
      mbar_init(BW(kv_empty) + 8 * i, 1);
    }
    for (int i = 0; i < kSwSSlots; ++i) {
      mbar_init(BW(s_full) + 8 * i, 1);
      mbar_init(BW(s_empty) + 8 * i, 4);
    }
    for (int i = 0; i < kSwPSlots; ++i) {
      mbar_init(BW(p_full) + 8 * i, 4);
      mbar_init(BW(p_empty) + 8 * i, 1 + kAccW);   // PV commit + accumulator warps (gamma read)
    }
    for (int i = 0; i < kSwTSlots; ++i) {
      mbar_init(BW(t_full) + 8 * i, 1);
      mbar_init(BW(t_free) + 8 * i, kAccW);
    }
    mbar_init(BW(q_full), 4);
    mbar_init(BW(q_free), 1);
    mbar_init(BW(fin_full), 1);
    mbar_init(BW(fin_empty), kAccW);
    mbar_init(BW(bk_done), 1);
    fence_barrier_init();
  }
  if (warp == kSwWarpTma && lane == 0) {
    tma_prefetch_desc(&tm_kv);
    tma_prefetch_desc(&tm_rope);
  }
  if (warp == kSwWarpQk) tmem_alloc(BW(tmem_base), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = lds_u32(BW(tmem_base));

  pdl_wait();
  pdl_launch_dependents();
  const int g = blockIdx.x;   // one head tile: a CTA group is one CTA
  const int per = p.ws_hdr[H_PER], total = p.ws_hdr[H_TOTAL], groups = p.ws_hdr[H_GROUPS];
  const int lo = g * per;
  const bool has_work = g < groups && lo < total;
  const int hi = min(total, lo + per);
  UnitIter it{p.cum, lo, hi, g, has_work ? __ldg(p.first_req + g) : 0, has_work ? p.batch : 0};
  Unit u;

  if (warp >= kSwWarpTma) {
    if constexpr (N == 32) regs_dec<40>();
    if (warp == kSwWarpTma) {
      // ============================ TMA producer ============================
      if (lane == 0) {
        const uint64_t pol = l2_policy_evict_first();
        uint32_t n = 0;
        while (it.next(u)) {
          const int32_t* bt = p.block_table + (int64_t)u.b * p.max_pages;
          prefetch_block_table(bt, u.k0, u.k1);
          for (int j = u.k0; j < u.k1; ++j, ++n) {
            const uint32_t st = n % C::kSlots;
            mbar_wait_backoff(BW(kv_empty) + 8 * st, ((n / C::kSlots) & 1) ^ 1);
            const int row = __ldg(bt + j) * kPage;
            const uint32_t dst = sbase + st * kSwStage;
            const uint32_t full = BW(kv_full) + 8 * st;
            mbar_arrive_expect_tx(full, kSwTx);
#pragma unroll
            for (int c = 0; c < 4; ++c) tma_load_2d(dst + c * kBoxBytes, &tm_kv, full, c * 128, row, pol);
            tma_load_2d(dst + 4 * kBoxBytes, &tm_rope, full, 0, row, pol);
            bulk_load(dst + kSwOffScLo, p.kv_scale + (int64_t)row, 128, full, pol);
            bulk_load(dst + kSwOffScHi, p.kv_scale + (int64_t)row + 32, 128, full, pol);
          }
        }
      }
    } else if (warp == kSwWarpQk) {
      // ================================ QK issuer ================================
      uint32_t n = 0, unit = 0;
      while (it.next(u)) {
        mbar_wait_sleep(BW(q_full), unit & 1);
        for (int j = u.k0; j < u.k1; ++j, ++n) {
          const uint32_t st = n % C::kSlots, ss = n % kSwSSlots;
          mbar_wait_sleep(BW(kv_full) + 8 * st, (n / C::kSlots) & 1);
          mbar_wait_sleep(BW(s_empty) + 8 * ss, ((n / kSwSSlots) & 1) ^ 1);
          tc_fence_after();
          const uint32_t kv = sbase + st * kSwStage, dS = tmem + N * ss;
#pragma unroll
          for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)   // K = 32 FP8 per step: +32 B inside the 128-B swizzled row
              mma_f8_ws(dS, make_smem_desc(kv + b * kBoxBytes + 32 * ks, 16, 1024, LAYOUT_SW128),
                        make_smem_desc(sbase + C::kOffQc + b * C::kQcBox + 32 * ks, 16, 1024, LAYOUT_SW128),
                        C::kIdescQk8, (b | ks) != 0);
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)     // RoPE: K = 16 BF16 per step (Eq.6 pre-scaled q_r')
            mma_bf16_ws(dS, make_smem_desc(kv + 4 * kBoxBytes + 32 * ks, 16, 1024, LAYOUT_SW128),
                        make_smem_desc(sbase + C::kOffQr + 32 * ks, 16, 1024, LAYOUT_SW128), C::kIdescQk16, 1);
          mma_commit_ws(BW(s_full) + 8 * ss);
        }
        mma_commit_ws(BW(q_free));
        ++unit;
      }
    } else if (warp == kSwWarpPv) {
      // ================================ PV issuer ================================
      uint32_t n = 0;
      while (it.next(u)) {
        for (int j = u.k0; j < u.k1; ++j, ++n) {
          const uint32_t st = n % C::kSlots, ps = n % kSwPSlots, ts = n % kSwTSlots;
          mbar_wait_sleep(BW(p_full) + 8 * ps, (n / kSwPSlots) & 1);
          if (n >= (uint32_t)kSwTSlots) mbar_wait_sleep(BW(t_free) + 8 * ts, (n / kSwTSlots - 1) & 1);
          tc_fence_after();
          const uint32_t kv = sbase + st * kSwStage, pb = sbase + C::kOffP + ps * C::kPBytes;
          const uint32_t dT = tmem + C::kTmemT + 4 * N * ts;
#pragma unroll
          for (int d = 0; d < 4; ++d)        // dim tile d = content box d (128 dims)
#pragma unroll
            for (int ks = 0; ks < 2; ++ks)   // K = 32 tokens: +4 KB in V^T (32 rows of 128 B), +2 core-matrix columns in P'^T
              mma_f8_ws(dT + N * d, make_smem_desc(kv + d * kBoxBytes + 4096 * ks, kBoxBytes, 1024, LAYOUT_SW128),
                        make_smem_desc(pb + 32 * N * ks, 16 * N, 128, LAYOUT_NONE), C::kIdescPv, ks);
          mma_commit_ws(BW(t_full) + 8 * ts);
          mma_commit_ws(BW(p_empty) + 8 * ps);
          mma_commit_ws(BW(kv_empty) + 8 * st);
        }
      }
    }
  } else if (is_sm) {
    if constexpr (N == 32) regs_inc<144>();
    // ================= softmax: thread = (token, N/2 heads); group grp takes blocks n % kGroups == grp =================
    const int w = warp & 3, hh = lane >> 4, tq = lane & 15;
    const int tok = 16 * w + tq;
    const uint32_t lane_base = (uint32_t)(32 * w) << 16;
    const uint32_t nbar = 1 + grp;                    // this group's named barrier (128 threads)
    const uint32_t red = BW(red) + grp * (3 * 4 * 32 * 4);
    const int tid = threadIdx.x & 127;
    constexpr int kTpr = 128 / N;                     // Q-quant: threads per row
    const int qr = tid / kTpr, qpart = tid % kTpr;
    const bool bk = w == 0 && lane < N;              // head `lane`'s Alg.1 bookkeeping (for this group's blocks)
    uint32_t n = 0, unit = 0;
    while (it.next(u)) {
      // ---------------- Fused-Q-Quant (a2) by group 0: row qr, content chunks of qpart
      if (grp == 0) {
        if (unit > 0) mbar_wait(BW(q_free), (unit - 1) & 1);
        // Fused-Q-Quant ran in the plan launch: copy row qr's codes (chunks of qpart) into the SW128
        // B-operand boxes, q_r' into its SW128 row, c = sigma_q scale log2(e)
        const bool rok = qr < p.num_heads;
        const int64_t qrow_i = (int64_t)u.b * p.num_heads + qr;
        const uint4* qcr = reinterpret_cast<const uint4*>(p.qc + qrow_i * kDc);
        const uint4* qrr = reinterpret_cast<const uint4*>(p.qr + qrow_i * kDr);
        constexpr int kCh = 32 / kTpr;               // 16-code chunks of this thread
#pragma unroll
        for (int i = 0; i < kCh; ++i) {
          const int cg = kCh * qpart + i, box = cg >> 3, c16 = cg & 7;
          const uint4 v = rok ? __ldg(qcr + cg) : make_uint4(0, 0, 0, 0);
          sts_u4(sbase + C::kOffQc + box * C::kQcBox + qr * 128 + ((c16 ^ (qr & 7)) << 4), v.x, v.y, v.z, v.w);
        }
#pragma unroll
        for (int i = 0; i < 8 / kTpr; ++i) {
          const int c = (8 / kTpr) * qpart + i;
          const uint4 v = rok ? __ldg(qrr + c) : make_uint4(0, 0, 0, 0);
          sts_u4(sbase + C::kOffQr + qr * 128 + ((c ^ (qr & 7)) << 4), v.x, v.y, v.z, v.w);
        }
        const float sq = rok ? __ldg(p.sq + qrow_i) : 1.f;
        if (qpart == 0) sts_f32(BW(cq) + 4 * qr, sq * p.scale_log2);
        fence_proxy_async_smem();
        named_bar_sync(nbar, 128);
        warp_arrive(BW(q_full), lane);
      }
      mbar_wait(BW(q_full), unit & 1);                // group 1: c is in SMEM from here on
      float c[NH];
#pragma unroll
      for (int i = 0; i < NH; ++i) c[i] = lds_f32(BW(cq) + 4 * (hh * NH + i));
      const float c_bk = bk ? lds_f32(BW(cq) + 4 * lane) : 0.f;
      // rows see the cache up to their own query token (causal MTP, reading R25)
      const int sl = __ldg(p.seq_lens + u.b);
      const int lmin = sl - (p.q_len - 1);
      for (int j = u.k0; j < u.k1; ++j, ++n) {
        if ((int)(n % kGroups) != grp) continue;
        const uint32_t st = n % C::kSlots, ss = n % kSwSSlots, ps = n % kSwPSlots;
        mbar_wait(BW(s_full) + 8 * ss, (n / kSwSSlots) & 1);
        tc_fence_after();
        float x[NH];
        if constexpr (NH == 8) tmem_ld_16x32bx2_x8<8>(tmem + lane_base + N * ss, *reinterpret_cast<uint32_t(*)[8]>(x));
        else tmem_ld_16x32bx2_x16<16>(tmem + lane_base + N * ss, *reinterpret_cast<uint32_t(*)[16]>(x));
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(BW(s_empty) + 8 * ss);
        mbar_wait(BW(kv_full) + 8 * st, (n / C::kSlots) & 1);   // sigma_K landed (already complete)
        const uint32_t kv = sbase + st * kSwStage;
        const float sk = lds_f32(kv + (tok < 32 ? kSwOffScLo + 4 * tok : kSwOffScHi + 4 * (tok - 32)));
        const int pos = j * kBc + tok;
#pragma unroll
        for (int i = 0; i < NH; ++i) x[i] *= sk;                     // step 3 (descale)
        if (pos >= lmin) {                                           // ragged tail / causal MTP (R19, R25)
#pragma unroll
          for (int i = 0; i < NH; ++i) {
            const int h = hh * NH + i;
            const int Lh = sl - (p.q_len - 1 - h / p.heads);
            x[i] = (h < p.num_heads && pos < Lh) ? x[i] : -INFINITY;
          }
        }
        // ---- per-head block max over the 64 tokens: half-warp butterfly, then the 4 warps
        // (exchange buffers: red[0] is read between this block's two barriers, red[1] / red[2]
        // after the second and before the group's next first barrier, so one buffer suffices)
        float v[NH];
        int hd;
#pragma unroll
        for (int i = 0; i < NH; ++i) v[i] = x[i];
        float r0 = tb_reduce<NH, true>(v, lane, hd);
        if ((lane & (16 / NH - 1)) == 0) sts_f32(red + 4 * ((0 * 4 + w) * 32 + hh * NH + hd), r0);
        named_bar_sync(nbar, 128);
        float m[NH];
#pragma unroll
        for (int i = 0; i < NH; i += 4) {
          float4 a = lds_f4(red + 4 * ((0 * 4 + 0) * 32 + hh * NH + i));
#pragma unroll
          for (int ww = 1; ww < 4; ++ww) {
            const float4 b = lds_f4(red + 4 * ((0 * 4 + ww) * 32 + hh * NH + i));
            a = make_float4(fmaxf(a.x, b.x), fmaxf(a.y, b.y), fmaxf(a.z, b.z), fmaxf(a.w, b.w));
          }
          m[i] = a.x;
          m[i + 1] = a.y;
          m[i + 2] = a.z;
          m[i + 3] = a.w;
        }
        float mx_bk = -INFINITY;
        if (bk) {
#pragma unroll
          for (int ww = 0; ww < 4; ++ww) mx_bk = fmaxf(mx_bk, lds_f32(red + 4 * ((0 * 4 + ww) * 32 + lane)));
        }
        // ---- steps 5-6: p = 2^(t c - m c), w = p sigma_K; M_b and l_b per head
        float pw[NH], pp[NH];
#pragma unroll
        for (int i = 0; i < NH; ++i) {
          const float mc = m[i] == -INFINITY ? 0.f : m[i] * c[i];
          pp[i] = ex2_approx(fmaf(x[i], c[i], -mc));
          pw[i] = pp[i] * sk;
          v[i] = pw[i];
        }
        float r1 = tb_reduce<NH, true>(v, lane, hd);
#pragma unroll
        for (int i = 0; i < NH; ++i) v[i] = pp[i];
        float r2 = tb_reduce<NH, false>(v, lane, hd);
        if ((lane & (16 / NH - 1)) == 0) {
          sts_f32(red + 4 * ((1 * 4 + w) * 32 + hh * NH + hd), r1);
          sts_f32(red + 4 * ((2 * 4 + w) * 32 + hh * NH + hd), r2);
        }
        named_bar_sync(nbar, 128);
        // ---- step 7: sigma_p = M_b / 448, P' = E4M3(w 448 / M_b), one byte per head into P'^T
        mbar_wait(BW(p_empty) + 8 * ps, ((n / kSwPSlots) & 1) ^ 1);
        const uint32_t pb = sbase + C::kOffP + ps * C::kPBytes + (tok >> 4) * (16 * N) + (tok & 15);
#pragma unroll
        for (int i = 0; i < NH; i += 4) {
          float4 a = lds_f4(red + 4 * ((1 * 4 + 0) * 32 + hh * NH + i));
#pragma unroll
          for (int ww = 1; ww < 4; ++ww) {
            const float4 b = lds_f4(red + 4 * ((1 * 4 + ww) * 32 + hh * NH + i));
            a = make_float4(fmaxf(a.x, b.x), fmaxf(a.y, b.y), fmaxf(a.z, b.z), fmaxf(a.w, b.w));
          }
          const float mbv[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int h = hh * NH + i + e;
            const float inv = mbv[e] > 0.f ? __fdividef(448.0f, mbv[e]) : 0.f;
            const uint32_t code = cvt_e4m3x2(pw[i + e] * inv, 0.f);
            asm volatile("st.shared.u8 [%0], %1;" ::"r"(pb + (h >> 3) * 128 + (h & 7) * 16), "r"(code) : "memory");
          }
        }
        if (w == 0) {
          // Alg.1 steps 4, 8-10 for head `lane`: the recurrence runs in block order across the
          // groups, its state chained through SMEM by bk_done (the decode.cu accumulator recurrence)
          if (n > 0) mbar_wait(BW(bk_done), (n - 1) & 1);
          const bool last = j + 1 == u.k1;
          if (bk) {
            const int h = lane;
            float mb = 0.f, lb = 0.f;
#pragma unroll
            for (int ww = 0; ww < 4; ++ww) {
              mb = fmaxf(mb, lds_f32(red + 4 * ((1 * 4 + ww) * 32 + h)));
              lb += lds_f32(red + 4 * ((2 * 4 + ww) * 32 + h));
            }
            const float mst = mb > 0.f ? (mx_bk == -INFINITY ? 0.f : mx_bk * c_bk) : -INFINITY;   // R11
            const float sb = mb * (1.0f / 448.0f);   // sigma_p = M_b / 448 (one rounding; not bit-gated)
            const bool first = j == u.k0;
            float m_ref = -INFINITY, m_O = 0.f, sig_O = 1.f, l_run = 0.f;
            if (!first) {
              m_ref = lds_f32(BW(bks) + 4 * (0 * 32 + h));
              m_O = lds_f32(BW(bks) + 4 * (1 * 32 + h));
              sig_O = lds_f32(BW(bks) + 4 * (2 * 32 + h));
              l_run = lds_f32(BW(bks) + 4 * (3 * 32 + h));
            }
            const float m_new = fmaxf(m_ref, mst);
            const bool skip = !first && ((mst == -INFINITY) || (mst < m_new - 64.f));
            float gamma = 0.f, delta = 1.f;
            if (first) {
              m_O = mst;
              sig_O = sb;
              l_run = lb;
              m_ref = mst;
            } else if (!skip) {
              gamma = ex2_approx(m_O - mst) * __fdividef(sig_O, sb);
              l_run = l_run * ex2_approx(m_ref - m_new) + lb * ex2_approx(mst - m_new);
              m_ref = m_new;
              m_O = mst;
              sig_O = sb;
            } else {
              gamma = 1.f;
              delta = 0.f;
            }
            sts_f32(BW(bks) + 4 * (0 * 32 + h), m_ref);
            sts_f32(BW(bks) + 4 * (1 * 32 + h), m_O);
            sts_f32(BW(bks) + 4 * (2 * 32 + h), sig_O);
            sts_f32(BW(bks) + 4 * (3 * 32 + h), l_run);
            sts_f32(BW(gam) + 4 * (ps * 32 + h), gamma);
            sts_f32(BW(del) + 4 * (ps * 32 + h), delta);
            const unsigned any = __ballot_sync(N == 32 ? 0xffffffffu : (1u << (N & 31)) - 1u, skip);
            if (h == 0) sts_f32(BW(skip) + 4 * ps, any != 0u ? 1.f : 0.f);
            if (last) {   // epilogue factors (a9): o = sigma_O 2^{m_O - m_ref} O / l, LSE natural log
              if (unit > 0) mbar_wait(BW(fin_empty), (unit - 1) & 1);
              const float f = l_run > 0.f ? sig_O * ex2_approx(m_O - m_ref) / l_run : 0.f;
              sts_f32(BW(fin) + 4 * h, f);
              if (h < p.num_heads)
                p.lse_part[(int64_t)u.slot * kHeadTile + h] =
                    l_run > 0.f ? (m_ref + log2f(l_run)) * 0.69314718055994531f : -INFINITY;
            }
          }
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(BW(bk_done));
            if (last) mbar_arrive(BW(fin_full));
          }
        }
        fence_proxy_async_smem();
        warp_arrive(BW(p_full) + 8 * ps, lane);
      }
      ++unit;
    }
  } else {
    // ============ accumulators: thread = (dim, N heads) for kTiles of the 4 dim tiles ============
    if constexpr (N == 32) regs_inc<184>();
    const int a = warp - kSwWarpAcc, q4 = a & 3, tp = a >> 2;
    constexpr int kTiles = 4 / (kAccW / 4);
    const uint32_t lane_base = (uint32_t)(32 * q4) << 16;
    uint32_t n = 0, unit = 0;
    while (it.next(u)) {
      float o[kTiles][N];
#pragma unroll
      for (int d = 0; d < kTiles; ++d)
#pragma unroll
        for (int h = 0; h < N; ++h) o[d][h] = 0.f;
      for (int j = u.k0; j < u.k1; ++j, ++n) {
        const uint32_t ps = n % kSwPSlots, ts = n % kSwTSlots;
        mbar_wait_sleep(BW(p_full) + 8 * ps, (n / kSwPSlots) & 1);
        const bool anyskip = lds_f32(BW(skip) + 4 * ps) != 0.f;
        mbar_wait_sleep(BW(t_full) + 8 * ts, (n / kSwTSlots) & 1);
        tc_fence_after();
#pragma unroll
        for (int d = 0; d < kTiles; ++d) {
          uint32_t tv[N];
          const uint32_t taddr = tmem + lane_base + C::kTmemT + 4 * N * ts + N * (kTiles * tp + d);
          if constexpr (N == 16) tmem_ld_32x32b_x16(taddr, *reinterpret_cast<uint32_t(*)[16]>(tv));
          else tmem_ld_32x32b_x32(taddr, *reinterpret_cast<uint32_t(*)[32]>(tv));
          tmem_wait_ld();
#pragma unroll
          for (int h = 0; h < N; h += 4) {
            const float4 g4 = lds_f4(BW(gam) + 4 * (ps * 32 + h));
            float4 t4 = make_float4(__uint_as_float(tv[h]), __uint_as_float(tv[h + 1]), __uint_as_float(tv[h + 2]),
                                    __uint_as_float(tv[h + 3]));
            if (anyskip) {   // a head whose block is negligible keeps O (delta = 0)
              const float4 d4 = lds_f4(BW(del) + 4 * (ps * 32 + h));
              t4 = make_float4(t4.x * d4.x, t4.y * d4.y, t4.z * d4.z, t4.w * d4.w);
            }
            const float2 r0 = __ffma2_rn(make_float2(o[d][h], o[d][h + 1]), make_float2(g4.x, g4.y), make_float2(t4.x, t4.y));
            const float2 r1 = __ffma2_rn(make_float2(o[d][h + 2], o[d][h + 3]), make_float2(g4.z, g4.w), make_float2(t4.z, t4.w));
            o[d][h] = r0.x;
            o[d][h + 1] = r0.y;
            o[d][h + 2] = r1.x;
            o[d][h + 3] = r1.y;
          }
        }
        tc_fence_before();
        warp_arrive(BW(t_free) + 8 * ts, lane);
        warp_arrive(BW(p_empty) + 8 * ps, lane);
      }
      // ---- epilogue (a9): o_part[row h][dim] = O^T[dim][h] f_h
      mbar_wait_sleep(BW(fin_full), unit & 1);
      const int64_t prow0 = (int64_t)u.slot * kHeadTile;
#pragma unroll
      for (int d = 0; d < kTiles; ++d) {
        const int dim = 128 * (kTiles * tp + d) + 32 * q4 + lane;
#pragma unroll
        for (int h = 0; h < N; ++h)
          if (h < p.num_heads) p.o_part[(prow0 + h) * kDc + dim] = o[d][h] * lds_f32(BW(fin) + 4 * h);
      }
      warp_arrive(BW(fin_empty), lane);
      ++unit;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kSwWarpQk) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// one-time per device and N: the dynamic SMEM attribute
static std::atomic<bool> g_sw_attr[2][64];

mla_status launch_decode_sw(const CUtensorMap& tm_kv, const CUtensorMap& tm_rope, const DecodeParams& prm, int dev,
                            int sms, cudaStream_t st) {
  const bool n16 = prm.num_heads <= 16;
  auto kern = n16 ? mla_decode_sw_kernel<16> : mla_decode_sw_kernel<32>;
  const uint32_t smem = n16 ? SwCfg<16>::kSmem : SwCfg<32>::kSmem;
  if (!g_sw_attr[n16 ? 0 : 1][dev].load()) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return MLA_ERR_CUDA;
    g_sw_attr[n16 ? 0 : 1][dev].store(true);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(kSwThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, tm_kv, tm_rope, prm) != cudaSuccess) return MLA_ERR_CUDA;
  return MLA_OK;
}

}  // namespace snapmla
