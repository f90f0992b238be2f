/*
 * uot_b200_bench.h -- measurement hooks used by bench.py (not part of the
 * reference-facing boundary in uot_b200.h).
 */
#ifndef UOT_B200_BENCH_H
#define UOT_B200_BENCH_H

#include <stddef.h>
#include "uot_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Runs the descriptor once, then times `reps` launches of the g-direction and
 * f-direction log-sum-exp kernels (CUDA events on `stream`): ms_out[0..1]. */
int uot_sinkhorn_time_main(const uot_sinkhorn_desc* desc, void* workspace, size_t workspace_bytes,
                           void* stream, int reps, float* ms_out);

/* MUFU ex2.approx.ftz.f32 throughput probe: independent ex2 chains on every
 * SM; returns ex2 results per second (measured with CUDA events). */
int uot_probe_mufu_ex2(void* stream, double* ex2_per_s);

/* One-tile tcgen05 check: D[128x128] = A[128xK] * B[128xK]^T (kind::tf32,
 * A from TMEM, B from shared memory); device pointers, row-major. */
int uot_tc_selftest(const float* A, const float* B, int K, float* D, void* stream);

/* CTA-pair check: D[256x128] = A[256xK] * B[128xK]^T with
 * tcgen05.mma.cta_group::2 on a cluster of two CTAs (A rows and B rows split
 * between the pair's TMEM / shared memory). */
int uot_tc_selftest2(const float* A, const float* B, int K, float* D, void* stream);

/* tcgen05 issue-rate probe: each of `ctas` CTAs issues `reps` back-to-back
 * 128 x n x 8 kind::tf32 MMAs (A from TMEM if ss == 0, else shared memory)
 * and adds its clock64 cycle count to *out_dev (device pointer). */
int uot_probe_tc_rate(int ctas, int reps, int n, int ss, unsigned long long* out_dev,
                      void* stream);

/* FP64 DFMA throughput probe (DFMA per second). */
int uot_probe_dfma(void* stream, double* dfma_per_s);

#ifdef __cplusplus
}
#endif

#endif
