// Declarations shared by the decode kernels (decode.cu: plan, single-CTA, block-pair; decode_mx.cu:
// the MX-scaled variant).  Product code only.
#pragma once
#include <atomic>
#include "snapmla_internal.h"

namespace snapmla {

constexpr int kThreads = 512;     // 16 warps (single-CTA and block-pair kernels)
constexpr uint32_t kBoxBytes = 8192;                        // 64 rows x 128 B TMA box

struct DecodeParams {
  const __nv_bfloat16* q;
  const uint8_t* kv_fp8;         // pools (L2 prefetch addresses; the loads go through the tensor maps)
  const __nv_bfloat16* kv_rope;
  const float* kv_scale;
  const int32_t* block_table;
  const int32_t* seq_lens;
  const int32_t* ws_hdr;
  const int32_t* cum;
  const int32_t* first_req;
  float* lse_part;
  float* o_part;
  const uint8_t* qc;             // Fused-Q-Quant results (written by the plan kernel): E4M3 codes [row][512],
  const __nv_bfloat16* qr;       //   q_r / sigma_q in BF16 [row][64] (Eq.6), sigma_q [row]; row = b * num_heads + h
  const float* sq;
  int batch, num_heads, n_ht, max_pages;   // num_heads = rows per request = q_len x heads
  int q_len, heads;                         // MTP: row = t * heads + h for query token t
  float scale_log2;   // softmax_scale * log2(e)
  unsigned long long* trace;   // debug timeline (CTA 0), only in SNAPMLA_TRACE builds
};

// debug timeline (SNAPMLA_TRACE builds only): trace[ev * kTraceN + n] = clock64() of event ev at block n (CTA 0)
constexpr int kTraceN = 256;
enum TraceEv { TR_TMA = 0, TR_QK, TR_PVL, TR_PVR, TR_SM_IN, TR_SM_OUT, TR_C_L, TR_C_R, TR_S1, TR_S2, TR_S3, TR_S4, TR_S5, TR_C0, TR_C1, TR_C2, TR_NEV };
#ifdef SNAPMLA_TRACE
#define TRACE(ev, n)                                                                          \
  do {                                                                                        \
    if (p.trace != nullptr && blockIdx.x == 0 && (n) < (uint32_t)kTraceN)                     \
      p.trace[(ev) * kTraceN + (n)] = clock64();                                              \
  } while (0)
#else
#define TRACE(ev, n) \
  do {               \
  } while (0)
#endif

// Warp-level arrive on a barrier that publishes (or releases) this warp's SMEM writes (reads):
// by default lane 0 arrives after __syncwarp (one arrival per warp); a SNAPMLA_LANE_ARRIVE build
// (compute-sanitizer racecheck runs, scripts/sanitize_all.sh) makes every lane arrive, which the
// tool models as synchronisation; counts scale by kArriveMul.
#ifdef SNAPMLA_LANE_ARRIVE
constexpr uint32_t kArriveMul = 32;
__device__ __forceinline__ void warp_arrive(uint32_t bar, int) { mbar_arrive(bar); }
#else
constexpr uint32_t kArriveMul = 1;
__device__ __forceinline__ void warp_arrive(uint32_t bar, int lane) {
  __syncwarp();
  if (lane == 0) mbar_arrive(bar);
}
#endif

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


// The TMA producer's page-id loads are a dependent chain (each TMA needs its block-table entry);
// at a unit start they would cost one DRAM round trip per block (~2K cycles, CTA-0 timeline),
// so the unit's block-table segment is requested up front, one L1 prefetch per 128-byte line.
__device__ __forceinline__ void prefetch_block_table(const int32_t* bt, int k0, int k1) {
  for (int j = k0 & ~31; j < k1; j += 32) asm volatile("prefetch.global.L1 [%0];" ::"l"(bt + j));
}

// Wait with a hardware suspend hint, for warps off the critical path (accumulators and MMA / TMA
// issuers waiting for work): spinning, they take issue slots -- and power under the board's cap --
// from the softmax warps on the same SMSPs; the thread is woken when the phase completes.
#ifndef SNAPMLA_SLEEP_NS
#define SNAPMLA_SLEEP_NS 20000
#endif
__device__ __forceinline__ void mbar_wait_sleep(uint32_t a, uint32_t parity) {
#ifdef SNAPMLA_NO_SLEEP
  mbar_wait(a, parity);
#else
  while (!mbar_try_wait_ns(a, parity, SNAPMLA_SLEEP_NS)) {
  }
#endif
}

// x / s for a row-constant s: rcp + one FMA correction of the quotient
// (Markstein); q codes are not bit-gated (the oracle re-quantizes q itself).
__device__ __forceinline__ float div_by(float x, float s, float rs) {
  const float q = x * rs;
  return fmaf(fmaf(-q, s, x), rs, q);
}
// the same on a pair, packed f32x2 (bit-identical to two div_by calls: fma(q, -s, x) == fma(-q, s, x))
__device__ __forceinline__ float2 div_by2(float2 x, float s, float rs) {
  const float2 rs2 = make_float2(rs, rs), ns2 = make_float2(-s, -s);
  const float2 q = __fmul2_rn(x, rs2);
  return __ffma2_rn(__ffma2_rn(q, ns2, x), rs2, q);
}

// Plan (a3) launch shared by the decode entry points: a programmatic dependent of the append,
// writes hdr / cum / first_req for `groups` CTA groups.
mla_status launch_plan(const int32_t* seq_lens, int batch, int num_heads, int groups, int32_t* hdr, int32_t* cum,
                       int32_t* first_req, int num_sms, cudaStream_t st, const __nv_bfloat16* q = nullptr,
                       uint8_t* qc = nullptr, __nv_bfloat16* qr = nullptr, float* sq = nullptr);
// the encoded TMA map of a pool (cached per device; kind 0 FP8 content, 1 BF16 content, 2 RoPE)
bool cached_tmap(int dev, const void* base, uint64_t rows, int kind, CUtensorMap* out);
int current_device();
// the swapped-operand kernel for rows <= 32 (decode_sw.cu); the plan has been launched
mla_status launch_decode_sw(const CUtensorMap& tm_kv, const CUtensorMap& tm_rope, const DecodeParams& prm, int dev,
                            int sms, cudaStream_t st);
extern std::atomic<unsigned long long*> g_trace;

}  // namespace snapmla
