"""B200-native (sm_100a) SnapMLA FP8 MLA decode hot path (arXiv 2602.10718).

  synth   seeded synthetic inputs (no method arithmetic)
  ops     ctypes binding of libsnapmla.so: mla_kv_append_quant, mla_decode_fp8,
          mla_combine (+ workspace query, fp32 combine), PagedMLACache
  build   in-tree nvcc build of libsnapmla.so

The library is loaded lazily on first use; there is no CPU fallback.
"""
