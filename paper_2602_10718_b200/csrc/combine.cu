// a10: split-KV combine (Algorithm 1 returns o and the logsumexp L).
//   L = log sum_s e^{L_s};   o = sum_s e^{L_s - L} o_s
// One warp per (request, head, quarter of the 512 columns); lane l owns 4 columns; the split LSEs and
// weights are handled lane-parallel, eight splits' partial rows are in flight at a time.
// The split list of request b is the contiguous slot range b + g for the
// groups g that the decode plan assigned to b's key blocks.
#include "snapmla_internal.h"

namespace snapmla {

// NEXT-4(c): the TP all-gather fused into the combine epilogue.  Each rank combines its
// head slice and stores the BF16 rows straight into EVERY rank's gathered output
// [batch, world * num_heads, 512] (heads rank-major) through peer-mapped pointers
// (NVLink P2P stores; on one GPU the "peers" are local buffers).
constexpr int kMaxPeers = 8;
struct Peers {
  void* out[kMaxPeers];
  int world, rank;
};

// kQ warps per (request, head) row, each owning 512 / kQ columns (kQ = 4 when requests have many
// splits -- small batches -- so more partial loads are in flight; kQ = 1 otherwise).
template <bool kF32Out, bool kGather = false, int kQ = 1>
__global__ void __launch_bounds__(128) combine_kernel(const char* __restrict__ ws, size_t off_cum, size_t off_lse,
                                                      size_t off_o, int batch, int num_heads, int num_sms,
                                                      void* __restrict__ out, float* __restrict__ lse_out,
                                                      const Peers peers = Peers{}) {
  pdl_wait();   // launched as a programmatic dependent of the decode: its partials are complete here
  const int lane = threadIdx.x & 31;
  const int widx = blockIdx.x * 4 + (threadIdx.x >> 5);
  const int idx = widx / kQ, qc = widx % kQ;   // row (request, head) and its share of the 512 columns
  if (idx >= batch * num_heads) return;
  const int b = idx / num_heads, h = idx % num_heads;
  const int32_t* hdr = reinterpret_cast<const int32_t*>(ws);
  // The workspace must come from a decode of the same shape on a device with the same SM
  // count (the partial offsets depend on them, snapmla.h): a mismatch -- e.g. heads passed
  // instead of q_len x heads for MTP, another batch, another device -- traps loudly instead
  // of reading out of bounds.
  if (hdr[H_BATCH] != batch || hdr[H_HEADS] != num_heads || hdr[H_SMS] != num_sms) __trap();
  const int32_t* cum = reinterpret_cast<const int32_t*>(ws + off_cum);
  const float* lse_p = reinterpret_cast<const float*>(ws + off_lse);
  const float* o_p = reinterpret_cast<const float*>(ws + off_o);
  const int per = hdr[H_PER], n_ht = hdr[H_NHT];
  const int c0 = cum[b], c1 = cum[b + 1];
  const int ht = h / kHeadTile, row = h % kHeadTile;
  constexpr int kV = 4 / kQ;              // float4 per lane per split
  constexpr int kIn = 8 / kV;              // splits' partial rows in flight
  const int col = (512 / kQ) * qc + 4 * kV * lane;   // this lane's 4 kV output columns

  float4 acc[kV];
#pragma unroll
  for (int e = 0; e < kV; ++e) acc[e] = make_float4(0.f, 0.f, 0.f, 0.f);
  float lse = -INFINITY;
  if (c1 > c0) {
    const int g0 = c0 / per, g1 = (c1 - 1) / per;
    int ns = g1 - g0 + 1;   // splits of request b
    const int64_t sstride = (int64_t)n_ht * kHeadTile;   // rows between consecutive splits' partials
    const float* lse_row = lse_p + ((int64_t)(b + g0) * n_ht + ht) * kHeadTile + row;
    // the split LSEs are read lane-parallel (a serial loop over many splits -- small batches split
    // over all CTA groups -- is a chain of dependent memory latencies)
    float mx = -INFINITY;
    for (int s = lane; s < ns; s += 32) mx = fmaxf(mx, lse_row[s * sstride]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (mx == -INFINITY) ns = 0;   // the row saw no key at all (MTP token beyond a short cache)
    float wsum = 0.f;
    const float* src0 = o_p + (((int64_t)(b + g0) * n_ht + ht) * kHeadTile + row) * kDc + col;
    for (int s0 = 0; s0 < ns; s0 += 32) {
      const float wl = s0 + lane < ns ? expf(lse_row[(s0 + lane) * sstride] - mx) : 0.f;
      wsum += wl;
      const int cnt = min(32, ns - s0);
      const float* src = src0 + (int64_t)s0 * sstride * kDc;
      int i = 0;
      for (; i + kIn <= cnt; i += kIn) {   // kIn splits' partial rows in flight, accumulated in split order
        float4 v[kIn][kV];
#pragma unroll
        for (int k = 0; k < kIn; ++k)
#pragma unroll
          for (int e = 0; e < kV; ++e)
            v[k][e] = reinterpret_cast<const float4*>(src + (int64_t)(i + k) * sstride * kDc)[e];
#pragma unroll
        for (int k = 0; k < kIn; ++k) {
          const float w = __shfl_sync(0xffffffffu, wl, i + k);
#pragma unroll
          for (int e = 0; e < kV; ++e)
            acc[e] = make_float4(fmaf(w, v[k][e].x, acc[e].x), fmaf(w, v[k][e].y, acc[e].y), fmaf(w, v[k][e].z, acc[e].z),
                                 fmaf(w, v[k][e].w, acc[e].w));
        }
      }
      for (; i < cnt; ++i) {
        const float w = __shfl_sync(0xffffffffu, wl, i);
#pragma unroll
        for (int e = 0; e < kV; ++e) {
          const float4 v = reinterpret_cast<const float4*>(src + (int64_t)i * sstride * kDc)[e];
          acc[e] = make_float4(fmaf(w, v.x, acc[e].x), fmaf(w, v.y, acc[e].y), fmaf(w, v.z, acc[e].z), fmaf(w, v.w, acc[e].w));
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
    if (wsum > 0.f) {
      const float inv = 1.0f / wsum;
#pragma unroll
      for (int e = 0; e < kV; ++e) acc[e] = make_float4(acc[e].x * inv, acc[e].y * inv, acc[e].z * inv, acc[e].w * inv);
      lse = mx + logf(wsum);
    }
  }
  const int64_t orow = (int64_t)idx * kDc + col;
  if constexpr (kF32Out) {
#pragma unroll
    for (int e = 0; e < kV; ++e) reinterpret_cast<float4*>(static_cast<float*>(out) + orow)[e] = acc[e];
  } else {
    uint2 wv[kV];
#pragma unroll
    for (int e = 0; e < kV; ++e) {
      __nv_bfloat162 v0 = __floats2bfloat162_rn(acc[e].x, acc[e].y), v1 = __floats2bfloat162_rn(acc[e].z, acc[e].w);
      wv[e] = make_uint2(*reinterpret_cast<uint32_t*>(&v0), *reinterpret_cast<uint32_t*>(&v1));
    }
    if constexpr (kGather) {
      // row (b, rank * num_heads + h) of the [batch, world * num_heads, 512] output of every rank
      const int64_t grow = ((int64_t)b * peers.world * num_heads + (int64_t)peers.rank * num_heads + h) * kDc + col;
      for (int r = 0; r < peers.world; ++r)
#pragma unroll
        for (int e = 0; e < kV; ++e) reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(peers.out[r]) + grow)[e] = wv[e];
    } else {
#pragma unroll
      for (int e = 0; e < kV; ++e) reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(out) + orow)[e] = wv[e];
    }
  }
  if (lse_out && lane == 0 && qc == 0) lse_out[idx] = lse;
}

// programmatic dependent launch (the kernel's griddepcontrol.wait orders it after the decode)
template <typename... KArgs, typename... Args>
static mla_status launch_pdl(void (*kernel)(KArgs...), int grid, mla_stream_t stream, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...) == cudaSuccess ? MLA_OK : MLA_ERR_CUDA;
}

template <bool kF32>
static mla_status launch_combine(const void* workspace, int batch, int num_heads, int kv_lora_rank, void* out,
                                 float* lse, mla_stream_t stream) {
  if (batch < 0 || num_heads <= 0) return MLA_ERR_SHAPE;
  if (kv_lora_rank != kDc) return MLA_ERR_UNSUPPORTED;
  if (num_heads > kMaxRows) return MLA_ERR_UNSUPPORTED;
  if (batch == 0) return MLA_OK;
  if (!workspace) return MLA_ERR_WORKSPACE;
  if (!out) return MLA_ERR_NULL;
  if (!aligned(out, 16) || !aligned(workspace, 256)) return MLA_ERR_ALIGN;
  const int sms = device_num_sms();
  if (sms <= 0) return MLA_ERR_CUDA;
  const WsLayout wl = ws_layout(batch, num_heads, sms);
  const int n = batch * num_heads;   // rows
  const int groups = sms / ((num_heads + kHeadTile - 1) / kHeadTile);
  if (2 * batch < groups)   // several splits per request: 4 warps per row (4 warps per CTA)
    return launch_pdl(combine_kernel<kF32, false, 4>, n, stream, static_cast<const char*>(workspace), wl.cum, wl.lse,
                      wl.o, batch, num_heads, sms, out, lse, Peers{});
  return launch_pdl(combine_kernel<kF32, false, 1>, (n + 3) / 4, stream, static_cast<const char*>(workspace), wl.cum,
                    wl.lse, wl.o, batch, num_heads, sms, out, lse, Peers{});
}

}  // namespace snapmla

using namespace snapmla;

extern "C" mla_status mla_combine_gather(const void* workspace, int batch, int num_heads, int kv_lora_rank,
                                         void* const* out_peers, int world, int rank, float* lse,
                                         mla_stream_t stream) {
  if (batch < 0 || num_heads <= 0) return MLA_ERR_SHAPE;
  if (kv_lora_rank != kDc) return MLA_ERR_UNSUPPORTED;
  if (num_heads > kMaxRows || world < 1 || world > kMaxPeers) return MLA_ERR_UNSUPPORTED;
  if (rank < 0 || rank >= world) return MLA_ERR_SHAPE;
  if (batch == 0) return MLA_OK;
  if (!workspace) return MLA_ERR_WORKSPACE;
  if (!out_peers) return MLA_ERR_NULL;
  Peers peers = {};
  peers.world = world;
  peers.rank = rank;
  for (int r = 0; r < world; ++r) {
    if (!out_peers[r]) return MLA_ERR_NULL;
    if (!aligned(out_peers[r], 16)) return MLA_ERR_ALIGN;
    peers.out[r] = out_peers[r];
  }
  if (!aligned(workspace, 256)) return MLA_ERR_ALIGN;
  const int sms = device_num_sms();
  if (sms <= 0) return MLA_ERR_CUDA;
  const WsLayout wl = ws_layout(batch, num_heads, sms);
  const int n = batch * num_heads;
  return launch_pdl(combine_kernel<false, true, 1>, (n + 3) / 4, stream, static_cast<const char*>(workspace), wl.cum,
                    wl.lse, wl.o, batch, num_heads, sms, static_cast<void*>(nullptr), lse, peers);
}

extern "C" mla_status mla_combine(const void* workspace, int batch, int num_heads, int kv_lora_rank, void* out,
                                  float* lse, mla_stream_t stream) {
  return launch_combine<false>(workspace, batch, num_heads, kv_lora_rank, out, lse, stream);
}

extern "C" mla_status mla_combine_f32(const void* workspace, int batch, int num_heads, int kv_lora_rank,
                                      float* out, float* lse, mla_stream_t stream) {
  return launch_combine<true>(workspace, batch, num_heads, kv_lora_rank, out, lse, stream);
}

extern "C" const char* mla_status_str(mla_status s) {
  switch (s) {
    case MLA_OK: return "MLA_OK";
    case MLA_ERR_NULL: return "MLA_ERR_NULL";
    case MLA_ERR_SHAPE: return "MLA_ERR_SHAPE";
    case MLA_ERR_UNSUPPORTED: return "MLA_ERR_UNSUPPORTED";
    case MLA_ERR_ALIGN: return "MLA_ERR_ALIGN";
    case MLA_ERR_WORKSPACE: return "MLA_ERR_WORKSPACE";
    case MLA_ERR_CUDA: return "MLA_ERR_CUDA";
  }
  return "MLA_ERR_UNKNOWN";
}

extern "C" int mla_abi_version(void) { return 1; }
