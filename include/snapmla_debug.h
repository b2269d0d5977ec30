/*
 * snapmla_debug.h -- diagnostics of libsnapmla.so (not part of the hot path).
 */
#ifndef SNAPMLA_DEBUG_H_
#define SNAPMLA_DEBUG_H_
#include <stddef.h>
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
 * kernel (two independent M = 64 CTAs per key range), v = 2 the 2-SM
 * kernel (cta_group::2 QK and PV with token / dims halves per CTA of a cluster pair;
 * §7.8), v = 3 the block-pair 2-SM kernel (§7.9).  Process-global. */
void mla_debug_set_pair(int v);
/* Kernel for decodes with rows <= 32 (e.g. 16 heads per TP8 rank): v = 1 the swapped-operand
 * kernel (heads on the MMA N dimension), v = 0 the single-CTA kernel (heads
 * padded to M = 64; §7.3), v = -1 (default) the swapped kernel for rows <= 16 and the
 * single-CTA kernel above.  Process-global. */
void mla_debug_set_small(int v);
/* Measurement only (bench.py's roofline denominator): a read-only stream over
 * [buf, buf + bytes) (device memory, 16-B aligned, bytes % 16 == 0), one XOR
 * fold per CTA into sink[0 .. min(sink_len, 4 x SMs)) (device memory, zeroed by
 * the caller).  Enqueued on `stream`; returns an mla_status. */
int mla_measure_read_stream(const void* buf, size_t bytes, unsigned long long* sink, int sink_len,
                            void* stream);
/* Test only: out[i] (device, count bytes, 4-byte aligned, count % 4 == 0) = the E4M3 code the
 * kernels' encoder (cvt.rn.satfinite.e4m3x2.f32, 4 values per call as the kernels pack them)
 * gives the fp32 whose bit pattern is first_bits + i.  Used for the exhaustive sweep of all
 * finite fp32 against oracle.codec.encode_e4m3 (scripts/cvt_sweep.py). */
int mla_debug_cvt_e4m3(unsigned int first_bits, unsigned int count, unsigned char* out, void* stream);
#ifdef __cplusplus
}
#endif
#endif
