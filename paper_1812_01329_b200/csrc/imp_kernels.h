// imp_kernels.h — per-op kernels of the imperative executor (janus_run_imperative): one launch
// per op instance, SIMT fp32 with the bf16 operand-rounding points applied on load in bf16 mode.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace jk {
namespace imp {

// GEMMs: with both operands rounded to bf16 (the graph's R1/R2/R3 rounding points) and enough
// work, the operands are cast into the scratch set here and the product runs on the tcgen05 GEMM
// (gemm_tc.cu, fp32 accumulate); otherwise a SIMT kernel rounds on load. set_scratch: device bytes
// for the two bf16 operand copies (stream-ordered reuse, one GEMM at a time); take_extra_launches:
// launches issued beyond one per call since the last query (the casts).
void set_scratch(void *p, size_t bytes);
uint64_t take_extra_launches();
// Y[n][N] (+)= X[n][K] . W[N][K]^T          (rx / rw: round the operand to bf16 on load)
cudaError_t gemm_nt(float *Y, const float *X, const float *W, int n, int N, int K, int ldx, int ldw,
                    int ldy, bool acc, bool rx, bool rw, cudaStream_t s);
// Y[n][K] (+)= D[n][N] . W[N][K]
cudaError_t gemm_nn(float *Y, const float *D, const float *W, int n, int N, int K, int ldd, int ldw,
                    int ldy, bool acc, bool rd, bool rw, cudaStream_t s);
// G[N][K] (+)= D[n][N]^T . X[n][K]
cudaError_t gemm_tn(float *G, const float *D, const float *X, int n, int N, int K, int ldd, int ldx,
                    int ldg, bool acc, bool rd, bool rx, cudaStream_t s);
// y[r][c] += b[c]
cudaError_t add_bias(float *Y, const float *b, int n, int N, int ldy, cudaStream_t s);
// g[c] (+)= sum_r rd(D[r][c])
cudaError_t colsum(float *g, const float *D, int n, int N, int ldd, bool acc, bool rd, cudaStream_t s);
cudaError_t fill(float *p, float v, int64_t n, cudaStream_t s);
cudaError_t fill_i(int *p, int v, int64_t n, cudaStream_t s);
cudaError_t err_to_float(float *y, const int *err, cudaStream_t s);  // y[0] = err[0] != 0 ? 1 : 0
cudaError_t axpy(float *y, const float *x, float a, int64_t n, cudaStream_t s);        // y += a x
cudaError_t copy(float *y, const float *x, int64_t n, cudaStream_t s);
cudaError_t round_copy(float *y, const float *x, int64_t n, bool r, cudaStream_t s);   // y = rb(x)
cudaError_t copy_i(int *y, const int *x, int64_t n, cudaStream_t s);
cudaError_t i64_to_i32(int *y, const long long *x, int64_t n, cudaStream_t s);
// rows of E (optionally rounded); out-of-range ids set *err and read row 0
cudaError_t embedding(float *X, const float *E, const int *ids, int n, int V, int Ed, bool r, int *err,
                      cudaStream_t s);
// dE[ids[r]] += dX[r], rows in ascending r (deterministic: one thread per column)
cudaError_t embedding_bwd(float *dE, const float *dX, const int *ids, int n, int V, int Ed,
                          cudaStream_t s);
cudaError_t column(int *out, const int *M, int rows, int W, int t, int *err, cudaStream_t s);
cudaError_t element_i(int *out, const int *v, int n, int i, int *err, cudaStream_t s);
cudaError_t element_f(float *out, const float *v, int n, int i, int *err, cudaStream_t s);
cudaError_t less_iv(int *out, int a, const int *v, int n, cudaStream_t s);   // out[i] = a < v[i]
cudaError_t less_vi(int *out, const int *v, int a, int n, cudaStream_t s);   // out[i] = v[i] < a
cudaError_t cmp_scalar(int *out, const int *x, int a, int op, cudaStream_t s); // op 0: x<a, 1: a<x, 2: x==a
cudaError_t max_reduce(int *out, const int *v, int n, cudaStream_t s);
cudaError_t sum_all(float *out, const float *x, int64_t n, cudaStream_t s);
cudaError_t seq_mask(int *out, const int *lens, int B, int T, cudaStream_t s);
cudaError_t time_major(int *out, const int *M, int B, int W, int T, int *err, cudaStream_t s);
cudaError_t add_f(float *out, const float *a, const float *b, int64_t n, int64_t nb, cudaStream_t s);
// LSTM cell on the pre-activation Z [B][4H] (blocks i,f,g,o): writes gates (activations), c, h;
// rows with valid[b]==0 keep (h, c)
cudaError_t lstm_fwd(float *gates, float *c2, float *h2, const float *Z, const float *c, const float *h,
                     const int *valid, int B, int H, cudaStream_t s);
// dz (masked rows 0), dh_pass (valid ? 0 : dh2), dc_prev
cudaError_t lstm_bwd(float *dz, float *dh_pass, float *dc_prev, const float *dh2, const float *dc2,
                     const float *gates, const float *c, const float *c2, const int *valid, int B, int H,
                     cudaStream_t s);
cudaError_t tree_leaf_fwd(float *gates, float *c, float *h, const float *Z, const float *b, int n, int H,
                          cudaStream_t s);
cudaError_t tree_leaf_bwd(float *dz, const float *dh, const float *dcin, const float *gates,
                          const float *c, int n, int H, cudaStream_t s);
cudaError_t tree_cell_fwd(float *gates, float *c, float *h, const float *Z, const float *b,
                          const float *cl, const float *cr, int n, int H, cudaStream_t s);
cudaError_t tree_cell_bwd(float *dz, float *dcl, float *dcr, const float *dh, const float *dcin,
                          const float *gates, const float *c, const float *cl, const float *cr, int n,
                          int H, cudaStream_t s);
// leaf bias [b_i; b_o; b_u] and cell bias [b_i; b_f; b_f; b_o; b_u] gathered from b (i,f,o,u)
cudaError_t tree_bias(float *out, const float *b, int H, int cell, cudaStream_t s);
// db (i,f,o,u) += bias-vector gradient of a leaf (3H) or a cell (5H)
cudaError_t tree_bias_bwd(float *db, const float *g, int H, int cell, cudaStream_t s);
// mean masked xent: loss (device scalar), dy = mask (softmax - onehot) / n_valid
cudaError_t xent(float *loss, float *dy, const float *logits, const int *tgt, const int *mask, int n,
                 int C, int *err, cudaStream_t s);
cudaError_t sgd(float *W, const float *g, float lr, int64_t n, cudaStream_t s);
// TreeRNN cell activation: y = tanh(y); its backward dz = dh (1 - h^2)
cudaError_t tanh_inplace(float *y, int64_t n, cudaStream_t s);
cudaError_t tanh_bwd(float *dz, const float *dh, const float *h, int64_t n, cudaStream_t s);

}  // namespace imp
}  // namespace jk
