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
#ifdef __cplusplus
}
#endif
#endif
