/*
 * snapmla_debug.h -- diagnostics of libsnapmla.so (not part of the hot path).
 */
#ifndef SNAPMLA_DEBUG_H_
#define SNAPMLA_DEBUG_H_
#ifdef __cplusplus
extern "C" {
#endif
/* When dev_buf != NULL, every later mla_decode_fp8 on this process records a
 * clock64() timeline of CTA 0 into dev_buf (device memory, >= 8 * 256 uint64):
 * dev_buf[ev * 256 + n] for events ev = {TMA issue, QK issue, PV_L issue,
 * PV_R issue, softmax start, softmax done, O_L rescaled, O_R rescaled} of the
 * CTA's n-th key block.  NULL disables it (default). */
void mla_debug_set_trace(unsigned long long* dev_buf);
/* Kernel for decodes with 64 < rows <= 128 (e.g. 128 heads): v = 0 the single-CTA
 * kernel (two independent M = 64 CTAs per key range; the default),
 * v = 2 the 2-SM kernel (cta_group::2 QK and PV with token / dims halves per CTA of
 * a cluster pair; §7.8), v = 1 the CTA-pair kernel (cta_group::2 QK over two key
 * blocks, per-CTA PV; §7.6).  v = 1, 2 are experimental.  Process-global. */
void mla_debug_set_pair(int v);
/* Cap the number of CTA pairs the pair kernel launches (0 = as many as fit);
 * returns the cudaOccupancyMaxActiveClusters limit seen on the last pair launch
 * (-1 before the first).  For measurements only. */
int mla_debug_set_pair_groups(int v);
#ifdef __cplusplus
}
#endif
#endif
