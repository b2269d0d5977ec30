// Internal constants and helpers shared by the CUDA translation units.
#pragma once
#include <cstddef>
#include <cstdint>

#include <cuda.h>

#include "../../include/snapmla.h"
#include "ptx.cuh"

namespace snapmla {

constexpr int kDc = 512;      // kv_lora_rank (north_star)
constexpr int kDr = 64;       // rope dim
constexpr int kDqk = kDc + kDr;
constexpr int kPage = 64;     // tokens per page
constexpr int kBc = 64;       // key / P-quant block
constexpr int kHeadTile = 64; // query rows per CTA (UMMA M = 64)
constexpr int kMaxRows = 4 * kHeadTile;   // rows per request (q_len x heads) the decode supports
constexpr float kSigmaMin = 0x1p-24f;   // reading R2

inline bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

// ---- workspace layout (shared by decode and combine) ---------------------
// int32 header[kHdr] | int32 cum[batch+1] | int32 first_req[groups] |
// float lse_part[slots*n_ht*64] | float o_part[slots*n_ht*64*512] |
// u8 q_c[batch*rows*512] | bf16 q_r'[batch*rows*64] | float sigma_q[batch*rows]   (Fused-Q-Quant, by the plan)
// slot of (request b, group g) = b + g; slots = batch + groups.
constexpr int kHdr = 16;
enum HdrField { H_TOTAL = 0, H_PER = 1, H_GROUPS = 2, H_NHT = 3, H_BATCH = 4, H_HEADS = 5, H_SMS = 6 };

struct WsLayout {
  size_t cum, first, lse, o, qc, qr, sq, total;
};
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
inline WsLayout ws_layout(int batch, int num_heads, int num_sms) {
  const int n_ht = (num_heads + kHeadTile - 1) / kHeadTile;
  const int groups = num_sms / (n_ht > 0 ? n_ht : 1);
  const size_t slots = (size_t)batch + (size_t)groups;
  WsLayout w;
  w.cum = kHdr * 4;
  w.first = align_up(w.cum + ((size_t)batch + 1) * 4, 16);
  w.lse = align_up(w.first + (size_t)(groups + 1) * 4, 256);
  w.o = align_up(w.lse + slots * n_ht * kHeadTile * 4, 256);
  const size_t rows = (size_t)batch * (size_t)num_heads;
  w.qc = align_up(w.o + slots * n_ht * kHeadTile * (size_t)kDc * 4, 256);
  w.qr = align_up(w.qc + rows * kDc, 256);
  w.sq = align_up(w.qr + rows * kDr * 2, 256);
  w.total = align_up(w.sq + rows * 4, 256);
  return w;
}

int device_num_sms();

}  // namespace snapmla
