// a2-a9: absorbed-MLA FP8 decode with the reconstructed PV pipeline, sm_100a.
//
// Method (PAPER.md, arXiv 2602.10718): Eq.5 absorbed score, Eq.6
// pre-scaled RoPE alignment, scale fusion + block-wise dynamic P
// quantization + implicit dequantization, Algorithm 1
// with Appendix C's strictly monotonic accumulation order.
//
// B200 design: one persistent CTA per SM, one 64-row query-head
// tile per CTA (UMMA M = 64), split-KV over 64-token key blocks planned on the
// device, a 4-slot ring of KV blocks in SMEM.  Warp roles (16 warps; the SM
// schedulers prefer the highest eligible warp id, so latency-critical roles
// get the high ids):
//   warps 0-7    two accumulator warpgroups (O columns 0-255 / 256-511): the
//                scalar Alg.1 recurrence (m, sigma_p, l, gamma; steps 4, 8-10)
//                and O <- gamma O + T_n with O in REGISTERS (as Alg.1 keeps
//                o^L / o^R in registers), epilogue (fp32 split partials)
//   warp 8       TMA producer: per block 4 x 8 KB FP8 boxes + 8 KB BF16 RoPE box
//                (SWIZZLE_128B, row coordinate from the block table) + 256 B scales
//   warp 9       QK issuer (owns TMEM): 16 x kind::f8f6f4 (K=32) + 4 x kind::f16
//                (K=16) into ONE fp32 accumulator S (Eq.6 makes the domains agree)
//   warps 10, 11 PV_L / PV_R issuers: T_n = P'_n (SMEM, K-major) x V (the SAME
//                FP8 tile read MN-major: no transpose), a fresh TMEM tile per block
//   warps 12-15  Q-quant prologue (Fused-Q-Quant), softmax, scale fusion, block
//                P quantization; thread = (head row, 32-token half)
// Why O lives in registers (measured, scripts/tmem_bench.cu): TMEM stores run at
// ~235 B/cycle/SM, so rescaling a 64 x 512 fp32 O in TMEM every block costs
// >= 550 cycles and serialises PV(n-1) -> rescale -> PV(n).  Reading T_n (loads
// ~800 B/cycle) and FMA-ing into registers removes the stores and the chain.
// Each block's softmax is computed against its OWN max (the P' codes depend only
// on w / max_block(w)), and the accumulator warps, which see blocks in
// strictly increasing order, carry the running max, so blocks are independent.
// Issue warps run converged and elect one lane per tcgen05 op (measured: a
// tcgen05.commit stalls the issuing warp's next MMA until completion, so each
// committing MMA stream has its own warp).
// TMEM (512 cols): T_L / T_R in the lower half-subpartitions (lanes 0-15 of each
// 32, cols 0-255 / 256-511), four S slots (64 cols) in the upper (lanes 16-31).
#include "snapmla_internal.h"

namespace snapmla {

constexpr int kThreads = 512;     // 16 warps
constexpr int kWarpAcc = 0;       // 0-3  accumulator, O cols 0-255; 4-7 cols 256-511
constexpr int kWarpTma = 8;       // 8    TMA producer
constexpr int kWarpQk = 9;        // 9    QK issuer, owns TMEM
constexpr int kWarpPv = 10;       // 10-11 PV_L / PV_R issuers
constexpr int kWarpSoftmax = 12;  // 12-15 softmax
// register budget (setmaxnreg): 256 x 192 + 128 x 40 + 128 x 88 = 65,536
constexpr uint32_t kRegsAcc = 192, kRegsIssue = 40, kRegsSoftmax = 88;
constexpr int kSlots = 4;         // KV / S / P' ring depth (blocks)
constexpr uint32_t kBoxBytes = 8192;                        // 64 rows x 128 B
constexpr uint32_t kKvTx = kBc * (kDc + 2 * kDr + 4);       // 41216 B per block
constexpr uint32_t kStage = 41984;                          // kKvTx rounded up to 1024
constexpr uint32_t kOffQc = 0;                              // 4 x [64 rows x 128 B] SW128
constexpr uint32_t kOffQr = 32768;                          // [64 rows x 128 B] SW128
constexpr uint32_t kOffP = 40960;                           // 4 slots x 4096 B, K-major core matrices
constexpr uint32_t kOffKv = 57344;                          // 4 slots: 4 content boxes | RoPE box | scales
constexpr uint32_t kOffBar = kOffKv + kSlots * kStage;
constexpr uint32_t kSmemBytes = kOffBar + 4096 + 1024;      // barriers/stats + alignment slack
static_assert(kSmemBytes <= 232448, "shared memory budget");

// instruction descriptors (M = 64)
constexpr uint32_t kIdescQk8 = make_idesc(0, 0, 0, 0, 64, 64);      // E4M3 x E4M3, both K-major
constexpr uint32_t kIdescQk16 = make_idesc(1, 1, 0, 0, 64, 64);     // BF16 x BF16
constexpr uint32_t kIdescPv = make_idesc(0, 0, 0, 1, 64, 256);      // P' K-major, V MN-major

struct DecodeParams {
  const __nv_bfloat16* q;
  const float* kv_scale;
  const int32_t* block_table;
  const int32_t* seq_lens;
  const int32_t* ws_hdr;
  const int32_t* cum;
  const int32_t* first_req;
  float* lse_part;
  float* o_part;
  int batch, num_heads, n_ht, max_pages;
  float scale_log2;   // softmax_scale * log2(e)
  unsigned long long* trace;   // debug timeline (CTA 0), nullptr in production
};

// debug timeline: trace[ev * kTraceN + n] = clock64() of event ev at block n (CTA 0 only)
constexpr int kTraceN = 256;
enum TraceEv { TR_TMA = 0, TR_QK, TR_PVL, TR_PVR, TR_SM_IN, TR_SM_OUT, TR_C_L, TR_C_R, TR_S1, TR_S2, TR_S3, TR_S4, TR_S5, TR_C0, TR_C1, TR_C2, TR_NEV };
#define TRACE(ev, n)                                                                          \
  do {                                                                                        \
    if (p.trace != nullptr && blockIdx.x == 0 && (n) < (uint32_t)kTraceN)                     \
      p.trace[(ev) * kTraceN + (n)] = clock64();                                              \
  } while (0)

struct Bars {
  uint64_t kv_full[kSlots], kv_empty[kSlots];   // TMA -> QK / PV_L + PV_R -> TMA
  uint64_t s_full[kSlots], s_empty[kSlots];     // QK -> softmax / softmax -> QK
  uint64_t p_full[kSlots], p_empty[kSlots];     // P' + stats: softmax -> PV, acc / PV_L + PV_R -> softmax
  uint64_t t_full[2], t_free[2];                // T_L/T_R: PV -> acc / acc -> PV
  uint64_t q_full;                              // Q-quant prologue -> QK
  uint32_t tmem_base;
  float stat[kSlots][3][64];          // per block and row: max(t) * c (log2 units), sigma_loc, l_loc
};
static_assert(sizeof(Bars) <= 4096, "barrier region");

// ------------------------------------------------------------------ plan (a3)
// One CTA.  cum[b] = sum_{b'<b} ceil(L_b'/64) (exclusive scan), total T.
// Groups of n_ht CTAs share a contiguous range of `per` key blocks; group g
// covers blocks [g*per, (g+1)*per) of the concatenated request sequence.
// first_req[g] = request holding block g*per.  Splits fall on 64-token block
// boundaries, so the result is split-invariant (oracle test
// test_block_aligned_split_plus_combine_equals_unsplit).
__global__ void __launch_bounds__(1024) plan_kernel(const int32_t* __restrict__ seq_lens, int batch, int num_heads,
                                                    int groups, int32_t* __restrict__ hdr,
                                                    int32_t* __restrict__ cum, int32_t* __restrict__ first_req) {
  __shared__ int warp_sums[32];
  __shared__ int s_per;
  const int tid = threadIdx.x;
  pdl_launch_dependents();
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
    const int per = total > 0 ? (total + groups - 1) / groups : 1;
    s_per = per;
    hdr[H_TOTAL] = total;
    hdr[H_PER] = per;
    hdr[H_GROUPS] = groups;
    hdr[H_NHT] = (num_heads + kHeadTile - 1) / kHeadTile;
    hdr[H_BATCH] = batch;
    hdr[H_HEADS] = num_heads;
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
}

// ------------------------------------------------------------------- units
struct Unit {
  int b, k0, k1, slot;
};

struct UnitIter {
  const int32_t* cum;
  int lo, hi, g, b, batch;
  __device__ bool next(Unit& u) {
    while (b < batch) {
      const int c0 = __ldg(cum + b), c1 = __ldg(cum + b + 1);
      if (c0 >= hi) return false;
      const int k0 = max(lo, c0) - c0, k1 = min(hi, c1) - c0;
      const int bb = b++;
      if (k1 > k0) {
        u.b = bb;
        u.k0 = k0;
        u.k1 = k1;
        u.slot = bb + g;
        return true;
      }
    }
    return false;
  }
};

// ------------------------------------------------------------- decode kernel
// x / s for a row-constant s: rcp + one FMA correction of the quotient
// (Markstein); q codes are not bit-gated (the oracle re-quantizes q itself).
__device__ __forceinline__ float div_by(float x, float s, float rs) {
  const float q = x * rs;
  return fmaf(fmaf(-q, s, x), rs, q);
}

__device__ __forceinline__ uint32_t cvt4_e4m3(float a, float b, float c, float d) {
  return (uint32_t)cvt_e4m3x2(a, b) | ((uint32_t)cvt_e4m3x2(c, d) << 16);
}

__global__ void __launch_bounds__(kThreads, 1)
    mla_decode_kernel(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_rope,
                      const DecodeParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Bars& bars = *reinterpret_cast<Bars*>(smem + kOffBar);
  const uint32_t sbase = smem_u32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---- setup overlaps the plan kernel (programmatic dependent launch)
  if (threadIdx.x == 0) {
    for (int i = 0; i < kSlots; ++i) {
      mbar_init(&bars.kv_full[i], 1);
      mbar_init(&bars.kv_empty[i], 2);
      mbar_init(&bars.s_full[i], 1);
      mbar_init(&bars.s_empty[i], 128);
      mbar_init(&bars.p_full[i], 128);
      mbar_init(&bars.p_empty[i], 2);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars.t_full[i], 1);
      mbar_init(&bars.t_free[i], 128);
    }
    mbar_init(&bars.q_full, 128);
    fence_barrier_init();
  }
  if (warp == kWarpTma && lane == 0) {
    tma_prefetch_desc(&tm_kv);
    tma_prefetch_desc(&tm_rope);
  }
  if (warp == kWarpQk) tmem_alloc(&bars.tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars.tmem_base;
  const uint32_t tmem_T = tmem;                       // lanes 0-15 (+32k): T_L cols 0-255, T_R 256-511
  const uint32_t tmem_S = tmem + (16u << 16);         // lanes 16-31 (+32k): S slot s at cols 64 s

  pdl_wait();   // plan (and the appends before it) visible from here on
  const int ht = blockIdx.x % p.n_ht;
  const int g = blockIdx.x / p.n_ht;
  const int per = p.ws_hdr[H_PER], total = p.ws_hdr[H_TOTAL], groups = p.ws_hdr[H_GROUPS];
  const int lo = g * per;
  const bool has_work = g < groups && lo < total;
  const int hi = min(total, lo + per);
  if (p.trace != nullptr && threadIdx.x == 0) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(gt));
    p.trace[TR_NEV * kTraceN + 2 * blockIdx.x] = gt;
  }

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
          for (int j = u.k0; j < u.k1; ++j, ++n) {
            const uint32_t st = n % kSlots;
            mbar_wait(&bars.kv_empty[st], ((n / kSlots) & 1) ^ 1, 1, n);
            TRACE(TR_TMA, n);
            const int row = __ldg(bt + j) * kPage;
            const uint32_t dst = sbase + kOffKv + st * kStage;
            mbar_arrive_expect_tx(&bars.kv_full[st], kKvTx);
#pragma unroll
            for (int c = 0; c < 4; ++c)
              tma_load_2d(dst + c * kBoxBytes, &tm_kv, &bars.kv_full[st], c * 128, row, pol);
            tma_load_2d(dst + 4 * kBoxBytes, &tm_rope, &bars.kv_full[st], 0, row, pol);
            bulk_load(dst + 5 * kBoxBytes, p.kv_scale + (int64_t)row, 256, &bars.kv_full[st], pol);
          }
        }
      }
    } else if (warp == kWarpQk) {
      // ================================ QK issuer ================================
      uint32_t n = 0, unit = 0;
      while (it.next(u)) {
        mbar_wait(&bars.q_full, unit & 1, 2, unit);
        for (int j = u.k0; j < u.k1; ++j, ++n) {
          const uint32_t st = n % kSlots;
          mbar_wait(&bars.kv_full[st], (n / kSlots) & 1, 3, n);
          mbar_wait(&bars.s_empty[st], ((n / kSlots) & 1) ^ 1, 4, n);
          tc_fence_after();
          if (lane == 0) TRACE(TR_QK, n);
          const uint32_t kv = sbase + kOffKv + st * kStage;
          const uint32_t dS = tmem_S + 64 * st;
#pragma unroll
          for (int kk = 0; kk < 16; ++kk) {
            const uint32_t off = (kk >> 2) * kBoxBytes + (kk & 3) * 32;
            mma_f8_ws(dS, make_smem_desc(sbase + kOffQc + off, 16, 1024, LAYOUT_SW128),
                      make_smem_desc(kv + off, 16, 1024, LAYOUT_SW128), kIdescQk8, kk > 0);
          }
#pragma unroll
          for (int kr = 0; kr < 4; ++kr) {
            mma_bf16_ws(dS, make_smem_desc(sbase + kOffQr + kr * 32, 16, 1024, LAYOUT_SW128),
                        make_smem_desc(kv + 4 * kBoxBytes + kr * 32, 16, 1024, LAYOUT_SW128), kIdescQk16, 1u);
          }
          mma_commit_ws(&bars.s_full[st]);
        }
        ++unit;
      }
    } else {
      // =============================== PV_L / PV_R ===============================
      const uint32_t half = warp - kWarpPv;
      uint32_t n = 0;
      while (it.next(u)) {
        for (int j = u.k0; j < u.k1; ++j, ++n) {
          const uint32_t st = n % kSlots;
          mbar_wait(&bars.p_full[st], (n / kSlots) & 1, 5, n);              // P'(n) in SMEM
          if (n > 0) mbar_wait(&bars.t_free[half], (n - 1) & 1, 6, n);      // T half read by the acc warps
          tc_fence_after();
          if (lane == 0) TRACE(half == 0 ? TR_PVL : TR_PVR, n);
          const uint32_t pA = sbase + kOffP + st * 4096;
          const uint32_t vb = sbase + kOffKv + st * kStage + (2 * half) * kBoxBytes;
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            const uint64_t a = make_smem_desc(pA + ks * 2048, 1024, 128, LAYOUT_NONE);
            const uint64_t b = make_smem_desc(vb + ks * 4096, kBoxBytes, 1024, LAYOUT_SW128);
            mma_f8_ws(tmem_T + 256 * half, a, b, kIdescPv, ks);
          }
          mma_commit_ws(&bars.t_full[half]);
          mma_commit_ws(&bars.p_empty[st]);
          mma_commit_ws(&bars.kv_empty[st]);
        }
      }
    }
  } else if (warp >= kWarpSoftmax) {
    regs_dec<kRegsSoftmax>();
    // ======= softmax / scale fusion / P quantization: thread = (row, token half) =======
    const int k = warp & 3;                  // TMEM subpartition of this warp
    const int t = lane & 15, h = lane >> 4;  // row-in-quarter, 32-token half
    const int r = 16 * k + t;                // query-head row inside the tile
    const int head = ht * kHeadTile + r;
    const bool row_ok = head < p.num_heads;
    const uint32_t lane_base = (uint32_t)(32 * k) << 16;
    uint32_t n = 0;
    while (it.next(u)) {
      // ---------------- Fused-Q-Quant prologue (a2): row r, content half h
      float c_row;
      {
        const uint4* qrow = reinterpret_cast<const uint4*>(p.q + ((int64_t)u.b * p.num_heads + head) * kDqk);
        float amax = 0.f;
#pragma unroll
        for (int bh = 0; bh < 2; ++bh) {
          uint4 qv[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) qv[i] = row_ok ? __ldg(qrow + 32 * h + 16 * bh + i) : make_uint4(0, 0, 0, 0);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&qv[i]);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = __bfloat1622float2(hv[e]);
              amax = fmaxf(amax, fmaxf(fabsf(f.x), fabsf(f.y)));
            }
          }
        }
        amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 16));
        const float sq = fmaxf(__fdiv_rn(amax, 448.0f), kSigmaMin);
        const float rsq = __frcp_rn(sq);
        c_row = sq * p.scale_log2;
#pragma unroll 2
        for (int gch = 0; gch < 16; ++gch) {   // 16-byte chunk of codes (re-read: L1 hit)
          uint4 v2[2];
          v2[0] = row_ok ? __ldg(qrow + 32 * h + 2 * gch) : make_uint4(0, 0, 0, 0);
          v2[1] = row_ok ? __ldg(qrow + 32 * h + 2 * gch + 1) : make_uint4(0, 0, 0, 0);
          const __nv_bfloat162* a = reinterpret_cast<const __nv_bfloat162*>(v2);
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f0 = __bfloat1622float2(a[2 * e]), f1 = __bfloat1622float2(a[2 * e + 1]);
            w[e] = cvt4_e4m3(div_by(f0.x, sq, rsq), div_by(f0.y, sq, rsq), div_by(f1.x, sq, rsq),
                             div_by(f1.y, sq, rsq));
          }
          const int byte = 256 * h + 16 * gch;          // byte offset inside the 512-B row
          const int sub = byte >> 7, c = (byte >> 4) & 7;
          sts_u4(sbase + kOffQc + sub * 8192 + r * 128 + ((c ^ (r & 7)) << 4), w[0], w[1], w[2], w[3]);
        }
#pragma unroll
        for (int gch = 0; gch < 4; ++gch) {
          const uint4 v = row_ok ? __ldg(qrow + 64 + 4 * h + gch) : make_uint4(0, 0, 0, 0);
          const __nv_bfloat162* a = reinterpret_cast<const __nv_bfloat162*>(&v);
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(a[e]);
            __nv_bfloat162 o2 = __halves2bfloat162(__float2bfloat16_rn(div_by(f.x, sq, rsq)),
                                                   __float2bfloat16_rn(div_by(f.y, sq, rsq)));
            w[e] = *reinterpret_cast<uint32_t*>(&o2);
          }
          const int c = 4 * h + gch;
          sts_u4(sbase + kOffQr + r * 128 + ((c ^ (r & 7)) << 4), w[0], w[1], w[2], w[3]);
        }
        fence_proxy_async_smem();
        mbar_arrive(&bars.q_full);
      }

      const int L = __ldg(p.seq_lens + u.b);
      for (int j = u.k0; j < u.k1; ++j, ++n) {
        const uint32_t st = n % kSlots;
        mbar_wait(&bars.s_full[st], (n / kSlots) & 1, 7, n);
        tc_fence_after();
        if (threadIdx.x == 32 * kWarpSoftmax) TRACE(TR_SM_IN, n);
        float tt[32];
        tmem_ld_16x32bx2_x32<32>(tmem_S + lane_base + 64 * st, *reinterpret_cast<uint32_t(*)[32]>(tt));
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(&bars.s_empty[st]);
        if (threadIdx.x == 32 * kWarpSoftmax) TRACE(TR_S1, n);

        // sigma_K of my 32 tokens (from the TMA'd slot), kept in registers
        const uint32_t sk = sbase + kOffKv + st * kStage + 5 * kBoxBytes + 128 * h;
        const int nvalid = L - (j * kBc + 32 * h);   // tokens of my half inside the sequence
#pragma unroll
        for (int i = 0; i < 32; i += 4) {                              // Alg.1 step 3 (descale)
          const float4 s4 = lds_f4(sk + 4 * i);
          const float2 a = __fmul2_rn(make_float2(tt[i], tt[i + 1]), make_float2(s4.x, s4.y));
          const float2 b = __fmul2_rn(make_float2(tt[i + 2], tt[i + 3]), make_float2(s4.z, s4.w));
          tt[i] = a.x;
          tt[i + 1] = a.y;
          tt[i + 2] = b.x;
          tt[i + 3] = b.y;
        }
        if (nvalid < 32) {                                             // ragged tail block: mask (R19)
#pragma unroll
          for (int i = 0; i < 32; ++i) tt[i] = i < nvalid ? tt[i] : -INFINITY;
        }
        float mx0 = fmaxf(tt[0], tt[1]), mx1 = fmaxf(tt[2], tt[3]);
#pragma unroll
        for (int i = 4; i < 32; i += 4) {
          mx0 = fmaxf(mx0, fmaxf(tt[i], tt[i + 1]));
          mx1 = fmaxf(mx1, fmaxf(tt[i + 2], tt[i + 3]));
        }
        float mx = fmaxf(mx0, mx1);
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));          // block max of t (local m)
        if (threadIdx.x == 32 * kWarpSoftmax) TRACE(TR_S2, n);
        const float mc = mx * c_row;
        float ls[4] = {0.f, 0.f, 0.f, 0.f};
        float mb0 = 0.f, mb1 = 0.f;
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 s4 = lds_f4(sk + 4 * i);                        // sigma_K (re-read, LDS broadcast)
          const float2 e0 = __ffma2_rn(make_float2(tt[i], tt[i + 1]), make_float2(c_row, c_row), make_float2(-mc, -mc));
          const float2 e1 = __ffma2_rn(make_float2(tt[i + 2], tt[i + 3]), make_float2(c_row, c_row), make_float2(-mc, -mc));
          const float2 p0 = make_float2(ex2_approx(e0.x), ex2_approx(e0.y));   // step 5 (block reference)
          const float2 p1 = make_float2(ex2_approx(e1.x), ex2_approx(e1.y));
          const float2 w0 = __fmul2_rn(p0, make_float2(s4.x, s4.y));           // step 6: p * sigma_K
          const float2 w1 = __fmul2_rn(p1, make_float2(s4.z, s4.w));
          ls[0] += p0.x;
          ls[1] += p0.y;
          ls[2] += p1.x;
          ls[3] += p1.y;
          tt[i] = w0.x;
          tt[i + 1] = w0.y;
          tt[i + 2] = w1.x;
          tt[i + 3] = w1.y;
          mb0 = fmaxf(mb0, fmaxf(w0.x, w0.y));
          mb1 = fmaxf(mb1, fmaxf(w1.x, w1.y));
        }
        float lsum = (ls[0] + ls[1]) + (ls[2] + ls[3]);
        float mb = fmaxf(mb0, mb1);
        mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 16));
        lsum += __shfl_xor_sync(0xffffffffu, lsum, 16);
        if (threadIdx.x == 32 * kWarpSoftmax) TRACE(TR_S3, n);
        // step 7: sigma_p = max/448, P' = E4M3(w * 448/max); a zero-max block gives
        // P' = 0 and is skipped by the recurrence (R11)
        const float inv = mb > 0.f ? __fdividef(448.0f, mb) : 0.f;
        uint32_t pw[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          pw[i] = cvt4_e4m3(tt[4 * i] * inv, tt[4 * i + 1] * inv, tt[4 * i + 2] * inv, tt[4 * i + 3] * inv);
        if (threadIdx.x == 32 * kWarpSoftmax) TRACE(TR_S4, n);
        // P' slot free once PV_L and PV_R of block n - kSlots completed
        mbar_wait(&bars.p_empty[st], ((n / kSlots) & 1) ^ 1, 8, n);
        if (threadIdx.x == 32 * kWarpSoftmax) TRACE(TR_S5, n);
        // K-major core matrices: byte(row, tok) = (tok/16)*1024 + row*16 + tok%16
        const uint32_t pdst = sbase + kOffP + st * 4096 + r * 16;
        sts_u4(pdst + (2 * h) * 1024, pw[0], pw[1], pw[2], pw[3]);
        sts_u4(pdst + (2 * h + 1) * 1024, pw[4], pw[5], pw[6], pw[7]);
        if (h == 0) {
          sts_f32(smem_u32(&bars.stat[st][0][r]), mb > 0.f ? mc : -INFINITY);
          sts_f32(smem_u32(&bars.stat[st][1][r]), __fdiv_rn(mb, 448.0f));
          sts_f32(smem_u32(&bars.stat[st][2][r]), lsum);
        }
        fence_proxy_async_smem();
        mbar_arrive(&bars.p_full[st]);
        if (threadIdx.x == 32 * kWarpSoftmax) TRACE(TR_SM_OUT, n);
      }
    }
  } else {
    regs_inc<kRegsAcc>();
    // ========= accumulators: Alg.1 recurrence per row, O <- gamma O + T in registers =========
    const int half = warp >> 2;              // 0: O cols 0-255 (T_L), 1: cols 256-511 (T_R)
    const int k = warp & 3;
    const int t = lane & 15, hh = lane >> 4;
    const int r = 16 * k + t;
    const int head = ht * kHeadTile + r;
    const bool row_ok = head < p.num_heads;
    const uint32_t taddr = tmem_T + ((uint32_t)(32 * k) << 16) + 256 * half;
    uint32_t n = 0;
    while (it.next(u)) {
      const uint32_t n0 = n;
      // O holds sum_b (sig_b 2^{m_b - m_O}) P'_b V in units of sig_O 2^{m_O} (log2 units);
      // l_run = sum_b l_b 2^{m_b - m_ref}.  This thread: row r, cols 256 half + 128 hh + [0, 128).
      float o[128];
      float m_ref = -INFINITY, m_O = 0.f, sig_O = 1.f, l_run = 0.f;
      for (int j = u.k0; j < u.k1; ++j, ++n) {
        const uint32_t st = n % kSlots;
        mbar_wait(&bars.p_full[st], (n / kSlots) & 1, 9, n);
        if (threadIdx.x == 0) TRACE(TR_C0, n);
        const float mb = lds_f32(smem_u32(&bars.stat[st][0][r]));
        const float sb = lds_f32(smem_u32(&bars.stat[st][1][r]));
        const float lb = lds_f32(smem_u32(&bars.stat[st][2][r]));
        const float m_new = fmaxf(m_ref, mb);                          // step 4 (running max)
        // a block whose contributions are < 2^-64 of the running total is dropped
        // (Alg.1 loses it to fp32 underflow of exp(s - m)); so is a zero-max block
        const bool first = n == n0;
        const bool skip = !first && ((mb == -INFINITY) || (mb < m_new - 64.f));
        float gamma = 1.f;
        if (first) {
          m_O = mb;
          sig_O = sb;
          l_run = lb;
          m_ref = mb;
        } else if (!skip) {
          gamma = ex2_approx(m_O - mb) * __fdiv_rn(sig_O, sb);         // steps 9-10
          l_run = l_run * ex2_approx(m_ref - m_new) + lb * ex2_approx(mb - m_new);
          m_ref = m_new;
          m_O = mb;
          sig_O = sb;
        }
        mbar_wait(&bars.t_full[half], n & 1, 10, n);                   // T(n) = P'(n) V complete
        tc_fence_after();
        if (threadIdx.x == 0) TRACE(TR_C1, n);
        const float2 g2 = make_float2(gamma, gamma);
        // software-pipelined T reads (8 chunks of 16 columns): chunk c+1 is in
        // flight while chunk c is FMA'd
        uint32_t tv[2][16];
        tmem_ld_16x32bx2_x16<128>(taddr, tv[0]);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          tmem_wait_ld();
          if (c < 7) tmem_ld_16x32bx2_x16<128>(taddr + 16 * (c + 1), tv[(c + 1) & 1]);
          else {
            tc_fence_before();
            mbar_arrive(&bars.t_free[half]);                           // PV(n+1) may overwrite T
          }
          const uint32_t* cur = tv[c & 1];
          if (first) {
#pragma unroll
            for (int i = 0; i < 16; ++i) o[16 * c + i] = __uint_as_float(cur[i]);
          } else if (!skip) {
#pragma unroll
            for (int i = 0; i < 16; i += 2) {
              const float2 a = __ffma2_rn(make_float2(o[16 * c + i], o[16 * c + i + 1]), g2,
                                          make_float2(__uint_as_float(cur[i]), __uint_as_float(cur[i + 1])));
              o[16 * c + i] = a.x;
              o[16 * c + i + 1] = a.y;
            }
          }
        }
        if (threadIdx.x == 0) TRACE(TR_C_L, n);
      }
      // ---------------- epilogue (a9): o = sig_O 2^{m_O - m_ref} O / l ; L = (m_ref + log2 l) ln 2
      const float f = sig_O * ex2_approx(m_O - m_ref) / l_run;
      const int64_t prow = ((int64_t)u.slot * p.n_ht + ht) * kHeadTile + r;
      if (row_ok) {
        float* dst = p.o_part + prow * kDc + 256 * half + 128 * hh;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          // chunk c of this thread = TMEM cols [32c, 32c+32) (+128 for threads 16-31)
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4*>(dst + 32 * c + i) =
                make_float4(o[32 * c + i] * f, o[32 * c + i + 1] * f, o[32 * c + i + 2] * f, o[32 * c + i + 3] * f);
        }
        if (half == 0 && hh == 0) p.lse_part[prow] = (m_ref + log2f(l_run)) * 0.69314718055994531f;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kWarpQk) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
  if (p.trace != nullptr && threadIdx.x == 0) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(gt));
    p.trace[TR_NEV * kTraceN + 2 * blockIdx.x + 1] = gt;
  }
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

static unsigned long long* g_trace = nullptr;

int device_num_sms() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return n;
}

}  // namespace snapmla

using namespace snapmla;

// Debug only (include/snapmla_debug.h): subsequent decodes record a CTA-0 event timeline.
extern "C" void mla_debug_set_trace(unsigned long long* dev_buf) { g_trace = dev_buf; }

extern "C" size_t mla_decode_workspace_bytes(int batch, int num_heads, int num_sms) {
  if (batch < 0 || num_heads <= 0) return 0;
  if (num_sms <= 0) num_sms = device_num_sms();
  if (num_sms <= 0) num_sms = 148;
  return ws_layout(batch, num_heads, num_sms).total;
}

extern "C" mla_status mla_decode_fp8(const void* q, const uint8_t* kv_fp8, const void* kv_rope,
                                     const float* kv_scale, const int32_t* block_table, const int32_t* seq_lens,
                                     int batch, int num_heads, int kv_lora_rank, int rope_dim, int page_size,
                                     int max_pages_per_seq, int64_t num_pages, float softmax_scale,
                                     void* workspace, size_t workspace_bytes, mla_stream_t stream) {
  if (batch < 0 || num_heads <= 0 || max_pages_per_seq < 0 || num_pages < 0) return MLA_ERR_SHAPE;
  if (kv_lora_rank != kDc || rope_dim != kDr || page_size != kPage) return MLA_ERR_UNSUPPORTED;
  if (num_heads > 2 * kHeadTile) return MLA_ERR_UNSUPPORTED;
  if (num_pages * kPage >= (int64_t)INT32_MAX) return MLA_ERR_UNSUPPORTED;   // TMA row coordinate is int32
  if (!workspace) return MLA_ERR_WORKSPACE;
  if (batch == 0) return MLA_OK;
  if (!q || !kv_fp8 || !kv_rope || !kv_scale || !block_table || !seq_lens) return MLA_ERR_NULL;
  if (!aligned(q, 16) || !aligned(kv_fp8, 128) || !aligned(kv_rope, 128) || !aligned(kv_scale, 16) ||
      !aligned(workspace, 256))
    return MLA_ERR_ALIGN;
  const int sms = device_num_sms();
  if (sms <= 0) return MLA_ERR_CUDA;
  const WsLayout wl = ws_layout(batch, num_heads, sms);
  if (workspace_bytes < wl.total) return MLA_ERR_WORKSPACE;
  const int n_ht = (num_heads + kHeadTile - 1) / kHeadTile;
  const int groups = sms / n_ht;

  CUtensorMap tm_kv, tm_rope;
  const uint64_t rows = (uint64_t)num_pages * kPage;
  if (num_pages == 0) return MLA_ERR_SHAPE;
  if (!encode_2d(&tm_kv, CU_TENSOR_MAP_DATA_TYPE_UINT8, kv_fp8, kDc, rows, kDc, 128, 64)) return MLA_ERR_CUDA;
  if (!encode_2d(&tm_rope, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, kv_rope, kDr, rows, kDr * 2, 64, 64))
    return MLA_ERR_CUDA;

  char* ws = static_cast<char*>(workspace);
  int32_t* hdr = reinterpret_cast<int32_t*>(ws);
  int32_t* cum = reinterpret_cast<int32_t*>(ws + wl.cum);
  int32_t* first = reinterpret_cast<int32_t*>(ws + wl.first);
  cudaStream_t st = (cudaStream_t)stream;
  plan_kernel<<<1, 1024, 0, st>>>(seq_lens, batch, num_heads, groups, hdr, cum, first);
  if (cudaGetLastError() != cudaSuccess) return MLA_ERR_CUDA;

  if (cudaFuncSetAttribute(mla_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes) !=
      cudaSuccess)
    return MLA_ERR_CUDA;
  DecodeParams prm;
  prm.q = (const __nv_bfloat16*)q;
  prm.kv_scale = kv_scale;
  prm.block_table = block_table;
  prm.seq_lens = seq_lens;
  prm.ws_hdr = hdr;
  prm.cum = cum;
  prm.first_req = first;
  prm.lse_part = reinterpret_cast<float*>(ws + wl.lse);
  prm.o_part = reinterpret_cast<float*>(ws + wl.o);
  prm.batch = batch;
  prm.num_heads = num_heads;
  prm.n_ht = n_ht;
  prm.max_pages = max_pages_per_seq;
  prm.scale_log2 = softmax_scale * 1.4426950408889634f;
  prm.trace = g_trace;
  // programmatic dependent launch: the decode CTAs start (barrier init, TMEM
  // alloc, descriptor prefetch) while the plan kernel runs; griddepcontrol.wait
  // in the kernel orders every read of the plan / cache after it.
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(groups * n_ht);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, mla_decode_kernel, tm_kv, tm_rope, prm) != cudaSuccess) return MLA_ERR_CUDA;
  return cudaGetLastError() == cudaSuccess ? MLA_OK : MLA_ERR_CUDA;
}
