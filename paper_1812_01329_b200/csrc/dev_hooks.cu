// dev_hooks.cu — kernel-level test entry points (include/janus_dev.h). Not part of the step path;
// the GPU unit tests call them to check one kernel at a time against the oracle's numerics.
#include "../../include/janus_dev.h"
#include "common.cuh"
#include "gemm_tc.h"
#include <stdlib.h>

extern "C" int32_t janus_dev_gemm_bf16(int32_t M, int32_t N, int32_t K, const void *A, int32_t lda,
                                       int32_t a_mn, const void *B, int32_t ldb, int32_t b_mn,
                                       float *C, int32_t ldc, const float *bias_col,
                                       const float *bias_row, int32_t accumulate, void *stream) {
  jk::GemmOp op;
  op.M = M; op.N = N; op.K = K;
  op.A = static_cast<const __nv_bfloat16 *>(A); op.lda = lda; op.a_mn = a_mn;
  op.B = static_cast<const __nv_bfloat16 *>(B); op.ldb = ldb; op.b_mn = b_mn;
  op.ep.C = C; op.ep.ldc = ldc; op.ep.bias_col = bias_col; op.ep.bias_row = bias_row;
  op.ep.accumulate = accumulate;
  cudaError_t e = jk::gemm_bf16(op, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? 0 : (int32_t)e;
}

extern "C" int32_t janus_dev_gemm_bf16_splitk(int32_t M, int32_t N, int32_t K, const void *A,
                                              int32_t lda, int32_t a_mn, const void *B, int32_t ldb,
                                              int32_t b_mn, float *C, int32_t ldc,
                                              const float *bias_col, const float *bias_row,
                                              int32_t accumulate, int32_t splits, void *stream) {
  static unsigned *flags = nullptr;
  static float *partials = nullptr;
  static size_t nflags = 0, npart = 0;
  const size_t need = jk::gemm_flags_count(M, N);
  const size_t need_p = need * 8 * 128 * 256;  // up to 8 splits of 128 x 256 tiles
  if (need > nflags) {
    if (flags) cudaFree(flags);
    if (cudaMalloc(&flags, need * sizeof(unsigned)) != cudaSuccess) return (int32_t)cudaErrorMemoryAllocation;
    cudaMemset(flags, 0, need * sizeof(unsigned));
    nflags = need;
  }
  if (need_p > npart) {
    if (partials) cudaFree(partials);
    if (cudaMalloc(&partials, need_p * sizeof(float)) != cudaSuccess) return (int32_t)cudaErrorMemoryAllocation;
    npart = need_p;
  }
  jk::GemmOp op;
  op.M = M; op.N = N; op.K = K;
  op.A = static_cast<const __nv_bfloat16 *>(A); op.lda = lda; op.a_mn = a_mn;
  op.B = static_cast<const __nv_bfloat16 *>(B); op.ldb = ldb; op.b_mn = b_mn;
  op.ep.C = C; op.ep.ldc = ldc; op.ep.bias_col = bias_col; op.ep.bias_row = bias_row;
  op.ep.accumulate = accumulate;
  op.flags = flags;
  op.partials = partials;
  op.partials_cap = npart;
  op.splits = splits;
  // dev knob: the two-way reduce-add split (GemmOp::split_add; C must be zero on entry)
  op.split_add = getenv("JANUS_GEMM_SPLIT_ADD") && getenv("JANUS_GEMM_SPLIT_ADD")[0] == '1';
  cudaError_t e = jk::gemm_bf16(op, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? 0 : (int32_t)e;
}
