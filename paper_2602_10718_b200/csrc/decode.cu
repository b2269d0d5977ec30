// a2-a9: absorbed-MLA FP8 decode with the reconstructed PV pipeline, sm_100a.
//
// Method (PAPER.md, arXiv 2602.10718): Eq.5 absorbed score, Eq.6
// pre-scaled RoPE alignment, scale fusion + block-wise dynamic P
// quantization + implicit dequantization, Algorithm 1
// with Appendix C's strictly monotonic accumulation order.
//
// B200 design: one persistent CTA per SM, one 64-row query-head
// tile per CTA (UMMA M = 64), split-KV over 64-token key blocks planned on the
// device, a 4-slot ring of 64-token KV blocks in SMEM.  Warp roles (13 warps):
//   warp 0       TMA producer: per block 4 x 8 KB FP8 boxes + 8 KB BF16 RoPE box
//                (SWIZZLE_128B, row coordinate from the block table) + 256 B scales
//   warps 1, 2   QK issuers for even / odd blocks (warp 1 also owns TMEM):
//                16 x kind::f8f6f4 (K=32) + 4 x kind::f16 (K=16) into ONE fp32
//                accumulator S (Eq.6 makes the two domains agree)
//   warps 3, 4   PV_L / PV_R issuers: P' (SMEM, K-major) x V (the SAME FP8 tile
//                read MN-major: no transpose) into O_L / O_R
//   warps 5-8    Q-quant prologue (Fused-Q-Quant), online softmax, scale fusion,
//                block P quantization; thread = (head row, 32-token half)
//   warps 9-12   correction O_L / O_R <- gamma O in TMEM, epilogue (fp32 partials)
// Issue warps run converged and elect one lane per tcgen05 op.  Measured on
// B200 (scripts/mma_bench.cu): a tcgen05.commit stalls the issuing warp's next
// MMA until completion, so every MMA stream that commits gets its own warp and
// the streams overlap in the tensor pipe.
// TMEM (512 cols): O in the lower half-subpartitions (lanes 0-15 of each 32),
// four S buffers (64 cols each) in the upper half-subpartitions (lanes 16-31).
#include "snapmla_internal.h"

namespace snapmla {

constexpr int kThreads = 416;   // 13 warps
constexpr int kSlots = 4;       // KV / S / P' ring depth (blocks)
constexpr uint32_t kBoxBytes = 8192;                        // 64 rows x 128 B
constexpr uint32_t kKvTx = kBc * (kDc + 2 * kDr + 4);       // 41216 B per block
constexpr uint32_t kStage = 41984;                          // kKvTx rounded up to 1024
constexpr uint32_t kOffQc = 0;                              // 4 x [64 rows x 128 B] SW128
constexpr uint32_t kOffQr = 32768;                          // [64 rows x 128 B] SW128
constexpr uint32_t kOffP = 40960;                           // 4 slots x 4096 B, K-major core matrices
constexpr uint32_t kOffKv = 57344;                          // 4 slots: 4 content boxes | RoPE box | scales
constexpr uint32_t kOffBar = kOffKv + kSlots * kStage;
constexpr uint32_t kSmemBytes = kOffBar + 3072 + 1024;      // barriers/gamma/stats + alignment slack
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
enum TraceEv { TR_TMA = 0, TR_QK, TR_PVL, TR_PVR, TR_SM_IN, TR_SM_OUT, TR_C_L, TR_C_R, TR_NEV };
#define TRACE(ev, n)                                                                          \
  do {                                                                                        \
    if (p.trace != nullptr && blockIdx.x == 0 && (n) < (uint32_t)kTraceN)                     \
      p.trace[(ev) * kTraceN + (n)] = clock64();                                              \
  } while (0)

struct Bars {
  uint64_t kv_full[kSlots], kv_empty[kSlots];   // TMA -> QK / PV_L + PV_R -> TMA
  uint64_t s_full[kSlots], s_empty[kSlots];     // QK -> softmax / softmax -> QK
  uint64_t p_full[kSlots], p_empty[kSlots];     // P', gamma: softmax -> PV + correction / PV_L + PV_R -> softmax
  uint64_t oL_ready, oR_ready, oL_done, oR_done;   // correction <-> PV halves
  uint64_t q_full;                    // Q-quant prologue -> QK
  uint64_t st_full[2], st_empty[2];   // per-unit epilogue factors softmax -> correction
  uint32_t tmem_base;
  float gamma[kSlots][64];
  float stat[2][64][2];
};
static_assert(sizeof(Bars) <= 3072, "barrier region");

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
// O <- gamma O on 16 lanes x 256 columns (threads 0-15 [c, c+32), 16-31 [c+128, c+160))
__device__ __forceinline__ void rescale_half(uint32_t taddr, float gamma) {
  const float2 g2 = make_float2(gamma, gamma);
#pragma unroll
  for (int c = 0; c < 128; c += 64) {
    uint32_t v0[32], v1[32];
    tmem_ld_16x32bx2_x32<128>(taddr + c, v0);
    tmem_ld_16x32bx2_x32<128>(taddr + c + 32, v1);
    tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      float2 a = __fmul2_rn(make_float2(__uint_as_float(v0[i]), __uint_as_float(v0[i + 1])), g2);
      v0[i] = __float_as_uint(a.x);
      v0[i + 1] = __float_as_uint(a.y);
      a = __fmul2_rn(make_float2(__uint_as_float(v1[i]), __uint_as_float(v1[i + 1])), g2);
      v1[i] = __float_as_uint(a.x);
      v1[i + 1] = __float_as_uint(a.y);
    }
    tmem_st_16x32bx2_x32<128>(taddr + c, v0);
    tmem_st_16x32bx2_x32<128>(taddr + c + 32, v1);
  }
  tmem_wait_st();
}

// x / s for a row-constant s: rcp + one Newton/FMA correction of the quotient
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
      mbar_init(&bars.st_full[i], 128);
      mbar_init(&bars.st_empty[i], 128);
    }
    mbar_init(&bars.oL_ready, 128);
    mbar_init(&bars.oR_ready, 128);
    mbar_init(&bars.oL_done, 1);
    mbar_init(&bars.oR_done, 1);
    mbar_init(&bars.q_full, 128);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_kv);
    tma_prefetch_desc(&tm_rope);
  }
  if (warp == 1) tmem_alloc(&bars.tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars.tmem_base;
  const uint32_t tmem_O = tmem;                       // lanes 0-15 (+32k): O_L cols 0-255, O_R 256-511
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

  if (warp == 0) {
    // ============================ TMA producer ============================
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
      uint32_t n = 0;
      while (it.next(u)) {
        const int32_t* bt = p.block_table + (int64_t)u.b * p.max_pages;
        for (int j = u.k0; j < u.k1; ++j, ++n) {
          const uint32_t st = n % kSlots;
          mbar_wait(&bars.kv_empty[st], ((n / kSlots) & 1) ^ 1);
          TRACE(TR_TMA, n);
          const int row = __ldg(bt + j) * kPage;
          const uint32_t dst = sbase + kOffKv + st * kStage;
          mbar_arrive_expect_tx(&bars.kv_full[st], kKvTx);
#pragma unroll
          for (int c = 0; c < 4; ++c) tma_load_2d(dst + c * kBoxBytes, &tm_kv, &bars.kv_full[st], c * 128, row, pol);
          tma_load_2d(dst + 4 * kBoxBytes, &tm_rope, &bars.kv_full[st], 0, row, pol);
          bulk_load(dst + 5 * kBoxBytes, p.kv_scale + (int64_t)row, 256, &bars.kv_full[st], pol);
        }
      }
    }
  } else if (warp <= 2) {
    // =================== QK issuers (warp 1: even blocks, warp 2: odd) ===================
    const uint32_t parity = warp - 1;
    uint32_t n = 0, unit = 0;
    while (it.next(u)) {
      mbar_wait(&bars.q_full, unit & 1);
      for (int j = u.k0; j < u.k1; ++j, ++n) {
        if ((n & 1) != parity) continue;
        const uint32_t st = n % kSlots;
        mbar_wait(&bars.kv_full[st], (n / kSlots) & 1);
        mbar_wait(&bars.s_empty[st], ((n / kSlots) & 1) ^ 1);
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
  } else if (warp <= 4) {
    // ========================= PV_L (warp 3) / PV_R (warp 4) =========================
    const uint32_t half = warp - 3;
    uint64_t* ready = half == 0 ? &bars.oL_ready : &bars.oR_ready;
    uint64_t* done = half == 0 ? &bars.oL_done : &bars.oR_done;
    uint32_t n = 0;
    while (it.next(u)) {
      const uint32_t n0 = n;
      for (int j = u.k0; j < u.k1; ++j, ++n) {
        const uint32_t st = n % kSlots;
        mbar_wait(&bars.p_full[st], (n / kSlots) & 1);    // P'(n) in SMEM
        mbar_wait(ready, n & 1);                          // O half rescaled by gamma(n)
        tc_fence_after();
        if (lane == 0) TRACE(half == 0 ? TR_PVL : TR_PVR, n);
        const uint32_t pA = sbase + kOffP + st * 4096;
        const uint32_t vb = sbase + kOffKv + st * kStage + (2 * half) * kBoxBytes;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const uint64_t a = make_smem_desc(pA + ks * 2048, 1024, 128, LAYOUT_NONE);
          const uint64_t b = make_smem_desc(vb + ks * 4096, kBoxBytes, 1024, LAYOUT_SW128);
          mma_f8_ws(tmem_O + 256 * half, a, b, kIdescPv, (n == n0 && ks == 0) ? 0u : 1u);
        }
        mma_commit_ws(done);
        mma_commit_ws(&bars.p_empty[st]);
        mma_commit_ws(&bars.kv_empty[st]);
      }
    }
  } else if (warp <= 8) {
    // ====== softmax / scale fusion / P quantization (warps 5-8): thread = (row, token half) ======
    const int k = warp & 3;                  // TMEM subpartition of this warp
    const int t = lane & 15, h = lane >> 4;  // row-in-quarter, 32-token half
    const int r = 16 * k + t;                // query-head row inside the tile
    const int head = ht * kHeadTile + r;
    const bool row_ok = head < p.num_heads;
    const uint32_t lane_base = (uint32_t)(32 * k) << 16;
    uint32_t n = 0, unit = 0;
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
        uint8_t* qc = smem + kOffQc;
#pragma unroll 4
        for (int gch = 0; gch < 16; ++gch) {   // 16-byte chunk of codes (re-read: L1 hit)
          uint4 v[2];
          v[0] = row_ok ? __ldg(qrow + 32 * h + 2 * gch) : make_uint4(0, 0, 0, 0);
          v[1] = row_ok ? __ldg(qrow + 32 * h + 2 * gch + 1) : make_uint4(0, 0, 0, 0);
          const __nv_bfloat162* a = reinterpret_cast<const __nv_bfloat162*>(v);
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f0 = __bfloat1622float2(a[2 * e]), f1 = __bfloat1622float2(a[2 * e + 1]);
            w[e] = cvt4_e4m3(div_by(f0.x, sq, rsq), div_by(f0.y, sq, rsq), div_by(f1.x, sq, rsq),
                             div_by(f1.y, sq, rsq));
          }
          const int byte = 256 * h + 16 * gch;          // byte offset inside the 512-B row
          const int sub = byte >> 7, c = (byte >> 4) & 7;
          *reinterpret_cast<uint4*>(qc + sub * 8192 + r * 128 + ((c ^ (r & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        uint8_t* qr = smem + kOffQr;
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
          *reinterpret_cast<uint4*>(qr + r * 128 + ((c ^ (r & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        fence_proxy_async_smem();
        mbar_arrive(&bars.q_full);
      }

      const int L = __ldg(p.seq_lens + u.b);
      float m_run = -INFINITY;   // running max of t = S * sigma_K (Alg.1 m)
      float l_part = 0.f;        // this thread's partial of l = sum_j 2^{(t_j - m) c}
      float sigma_p = 1.0f;      // Alg.1 line 1
      for (int j = u.k0; j < u.k1; ++j, ++n) {
        const uint32_t st = n % kSlots;
        mbar_wait(&bars.s_full[st], (n / kSlots) & 1);
        tc_fence_after();
        if (threadIdx.x == 160) TRACE(TR_SM_IN, n);
        float tt[32];
        tmem_ld_16x32bx2_x32<32>(tmem_S + lane_base + 64 * st, *reinterpret_cast<uint32_t(*)[32]>(tt));
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(&bars.s_empty[st]);

        // sigma_K of my 32 tokens (from the TMA'd slot)
        const float* sk = reinterpret_cast<const float*>(smem + kOffKv + st * kStage + 5 * kBoxBytes) + 32 * h;
        const int nvalid = min(32, L - (j * kBc + 32 * h));
        float mx = -INFINITY;
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 s4 = *reinterpret_cast<const float4*>(sk + i);
          tt[i + 0] = (i + 0 < nvalid) ? tt[i + 0] * s4.x : -INFINITY;   // Alg.1 step 3
          tt[i + 1] = (i + 1 < nvalid) ? tt[i + 1] * s4.y : -INFINITY;
          tt[i + 2] = (i + 2 < nvalid) ? tt[i + 2] * s4.z : -INFINITY;
          tt[i + 3] = (i + 3 < nvalid) ? tt[i + 3] * s4.w : -INFINITY;
          mx = fmaxf(mx, fmaxf(fmaxf(tt[i], tt[i + 1]), fmaxf(tt[i + 2], tt[i + 3])));
        }
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
        const float m_new = fmaxf(m_run, mx);                          // step 4
        const float mc = m_new * c_row;
        float lsum = 0.f, mb = 0.f;
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 s4 = *reinterpret_cast<const float4*>(sk + i);
          const float sv[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float pe = ex2_approx(fmaf(tt[i + e], c_row, -mc));   // step 5
            lsum += pe;
            tt[i + e] = pe * sv[e];                                      // step 6: p * sigma_K
            mb = fmaxf(mb, tt[i + e]);
          }
        }
        mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 16));
        const float alpha = ex2_approx((m_run - m_new) * c_row);       // 0 on the first block
        l_part = l_part * alpha + lsum;
        // step 7: sigma_p = max/448, P' = E4M3(w * 448/max); zero-max block -> P' = 0 (R11)
        const float inv = mb > 0.f ? __fdiv_rn(448.0f, mb) : 0.f;
        const float sp_new = mb > 0.f ? __fdiv_rn(mb, 448.0f) : sigma_p;
        const float gamma = alpha * __fdiv_rn(sigma_p, sp_new);        // step 9
        uint32_t pw[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          pw[i] = cvt4_e4m3(tt[4 * i] * inv, tt[4 * i + 1] * inv, tt[4 * i + 2] * inv, tt[4 * i + 3] * inv);
        // P' slot free once PV_L and PV_R of block n - kSlots completed
        mbar_wait(&bars.p_empty[st], ((n / kSlots) & 1) ^ 1);
        // K-major core matrices: byte(row, tok) = (tok/16)*1024 + row*16 + tok%16
        uint8_t* pdst = smem + kOffP + st * 4096 + r * 16;
        *reinterpret_cast<uint4*>(pdst + (2 * h) * 1024) = make_uint4(pw[0], pw[1], pw[2], pw[3]);
        *reinterpret_cast<uint4*>(pdst + (2 * h + 1) * 1024) = make_uint4(pw[4], pw[5], pw[6], pw[7]);
        if (h == 0) bars.gamma[st][r] = gamma;
        fence_proxy_async_smem();
        mbar_arrive(&bars.p_full[st]);
        if (threadIdx.x == 160) TRACE(TR_SM_OUT, n);
        m_run = m_new;
        sigma_p = sp_new;
      }
      // per-row epilogue factors (a9): o = sigma_p * O / l ; L = (m c + log2 l) ln 2
      const float l_tot = l_part + __shfl_xor_sync(0xffffffffu, l_part, 16);
      const uint32_t sb = unit & 1;
      mbar_wait(&bars.st_empty[sb], ((unit >> 1) & 1) ^ 1);
      if (h == 0) {
        bars.stat[sb][r][0] = sigma_p / l_tot;
        bars.stat[sb][r][1] = (m_run * c_row + log2f(l_tot)) * 0.69314718055994531f;
      }
      mbar_arrive(&bars.st_full[sb]);
      ++unit;
    }
  } else {
    // ============ correction + epilogue (warps 9-12): O <- gamma O ============
    const int k = warp & 3;
    const int t = lane & 15, h = lane >> 4;
    const int r = 16 * k + t;
    const int head = ht * kHeadTile + r;
    const bool row_ok = head < p.num_heads;
    const uint32_t lane_base = (uint32_t)(32 * k) << 16;
    uint32_t n = 0, unit = 0;
    while (it.next(u)) {
      const uint32_t n0 = n;
      for (int j = u.k0; j < u.k1; ++j, ++n) {
        if (n != n0) {
          const uint32_t st = n % kSlots;
          mbar_wait(&bars.p_full[st], (n / kSlots) & 1);
          const float gamma = bars.gamma[st][r];
          mbar_wait(&bars.oL_done, (n - 1) & 1);
          tc_fence_after();
          rescale_half(tmem_O + lane_base, gamma);
          tc_fence_before();
          mbar_arrive(&bars.oL_ready);
          if (threadIdx.x == 288) TRACE(TR_C_L, n);
          mbar_wait(&bars.oR_done, (n - 1) & 1);
          tc_fence_after();
          rescale_half(tmem_O + lane_base + 256, gamma);
          tc_fence_before();
          mbar_arrive(&bars.oR_ready);
          if (threadIdx.x == 288) TRACE(TR_C_R, n);
        } else {
          mbar_arrive(&bars.oL_ready);     // first block of the unit: PV starts a fresh accumulator
          mbar_arrive(&bars.oR_ready);
        }
      }
      // ---------------- epilogue: fp32 partial o and LSE of this split
      mbar_wait(&bars.oL_done, (n - 1) & 1);
      mbar_wait(&bars.oR_done, (n - 1) & 1);
      tc_fence_after();
      const uint32_t sb = unit & 1;
      mbar_wait(&bars.st_full[sb], (unit >> 1) & 1);
      const float f = bars.stat[sb][r][0];
      const float lse = bars.stat[sb][r][1];
      mbar_arrive(&bars.st_empty[sb]);
      const int64_t prow = ((int64_t)u.slot * p.n_ht + ht) * kHeadTile + r;
#pragma unroll 1
      for (int c = 0; c < 512; c += 64) {
        // threads 0-15: cols [c, c+32); threads 16-31: cols [c+32, c+64)
        uint32_t ov[32];
        tmem_ld_16x32bx2_x32<32>(tmem_O + lane_base + c, ov);
        tmem_wait_ld();
        if (row_ok) {
          float4* dst = reinterpret_cast<float4*>(p.o_part + prow * kDc + c + 32 * h);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            dst[i] = make_float4(__uint_as_float(ov[4 * i]) * f, __uint_as_float(ov[4 * i + 1]) * f,
                                 __uint_as_float(ov[4 * i + 2]) * f, __uint_as_float(ov[4 * i + 3]) * f);
        }
      }
      if (row_ok && h == 0) p.lse_part[prow] = lse;
      tc_fence_before();
      ++unit;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
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
