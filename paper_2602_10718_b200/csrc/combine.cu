// a10: split-KV combine (Algorithm 1 returns o and the logsumexp L).
//   L = log sum_s e^{L_s};   o = sum_s e^{L_s - L} o_s
// One warp per (request, head); lane l owns output columns [16l, 16l+16).
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

template <bool kF32Out, bool kGather = false>
__global__ void __launch_bounds__(128) combine_kernel(const char* __restrict__ ws, size_t off_cum, size_t off_lse,
                                                      size_t off_o, int batch, int num_heads, int num_sms,
                                                      void* __restrict__ out, float* __restrict__ lse_out,
                                                      const Peers peers = Peers{}) {
  pdl_wait();   // launched as a programmatic dependent of the decode: its partials are complete here
  const int lane = threadIdx.x & 31;
  const int idx = blockIdx.x * 4 + (threadIdx.x >> 5);
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

  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0.f;
  float lse = -INFINITY;
  if (c1 > c0) {
    int g0 = c0 / per, g1 = (c1 - 1) / per;
    float mx = -INFINITY;
    for (int g = g0; g <= g1; ++g) mx = fmaxf(mx, lse_p[((int64_t)(b + g) * n_ht + ht) * kHeadTile + row]);
    if (mx == -INFINITY) g1 = g0 - 1;   // the row saw no key at all (MTP token beyond a short cache)
    float wsum = 0.f;
    for (int g = g0; g <= g1; ++g) {
      const int64_t pr = ((int64_t)(b + g) * n_ht + ht) * kHeadTile + row;
      const float w = expf(lse_p[pr] - mx);
      wsum += w;
      const float4* src = reinterpret_cast<const float4*>(o_p + pr * kDc + lane * 16);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4 v = src[i];
        acc[4 * i + 0] = fmaf(w, v.x, acc[4 * i + 0]);
        acc[4 * i + 1] = fmaf(w, v.y, acc[4 * i + 1]);
        acc[4 * i + 2] = fmaf(w, v.z, acc[4 * i + 2]);
        acc[4 * i + 3] = fmaf(w, v.w, acc[4 * i + 3]);
      }
    }
    if (wsum > 0.f) {
      const float inv = 1.0f / wsum;
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] *= inv;
      lse = mx + logf(wsum);
    }
  }
  const int64_t orow = (int64_t)idx * kDc + lane * 16;
  if constexpr (kF32Out) {
    float4* dst = reinterpret_cast<float4*>(static_cast<float*>(out) + orow);
#pragma unroll
    for (int i = 0; i < 4; ++i) dst[i] = make_float4(acc[4 * i], acc[4 * i + 1], acc[4 * i + 2], acc[4 * i + 3]);
  } else {
    uint32_t wv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      __nv_bfloat162 v = __floats2bfloat162_rn(acc[2 * i], acc[2 * i + 1]);
      wv[i] = *reinterpret_cast<uint32_t*>(&v);
    }
    if constexpr (kGather) {
      // row (b, rank * num_heads + h) of the [batch, world * num_heads, 512] output of every rank
      const int64_t grow = ((int64_t)b * peers.world * num_heads + (int64_t)peers.rank * num_heads + h) * kDc + lane * 16;
      for (int r = 0; r < peers.world; ++r) {
        uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(peers.out[r]) + grow);
        dst[0] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        dst[1] = make_uint4(wv[4], wv[5], wv[6], wv[7]);
      }
    } else {
      uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(out) + orow);
      dst[0] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
      dst[1] = make_uint4(wv[4], wv[5], wv[6], wv[7]);
    }
  }
  if (lse_out && lane == 0) lse_out[idx] = lse;
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
  const int n = batch * num_heads;
  return launch_pdl(combine_kernel<kF32>, (n + 3) / 4, stream, static_cast<const char*>(workspace), wl.cum, wl.lse,
                    wl.o, batch, num_heads, sms, out, lse, Peers{});
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
  return launch_pdl(combine_kernel<false, true>, (n + 3) / 4, stream, static_cast<const char*>(workspace), wl.cum,
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
