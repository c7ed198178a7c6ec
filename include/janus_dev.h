/*
 * janus_dev.h — kernel-level test hooks of libjanus (not part of the step ABI in janus.h).
 * The GPU unit tests use them to check single kernels against the oracle's numerics.
 * All pointers are device pointers; calls are asynchronous on `stream`; return 0 or a
 * cudaError_t code.
 */
#ifndef JANUS_DEV_H
#define JANUS_DEV_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* C[M,N] (fp32, row pitch ldc) (+)= A . B^T (+ bias_col[n]) (+ bias_row[m]), bf16 operands.
 * a_mn = 0: A is [M][lda] (K contiguous); 1: A is [K][lda] (M contiguous). Same for B with N. */
int32_t janus_dev_gemm_bf16(int32_t M, int32_t N, int32_t K, const void *A, int32_t lda,
                            int32_t a_mn, const void *B, int32_t ldb, int32_t b_mn, float *C,
                            int32_t ldc, const float *bias_col, const float *bias_row,
                            int32_t accumulate, void *stream);

#ifdef __cplusplus
}
#endif
#endif
