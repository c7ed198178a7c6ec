// imp_kernels.cu — per-op kernels of the imperative executor (TF-Eager analogue, P:53, P:160,
// Table 3 column "Imp."). Plain SIMT fp32; in bf16 mode the GEMM operands are rounded to bf16 on
// load at the same points as the graph path (reading R).
#include "common.cuh"
#include "imp_kernels.h"
#include "gemm_tc.h"

namespace jk {
namespace imp {

static constexpr int NSM = 148;
JN_DEV float rnd(float x, bool r) { return r ? bf16_round(x) : x; }
static int blocks_for(int64_t n, int per = 256) {
  int64_t b = (n + per - 1) / per;
  return (int)(b < 8 * NSM ? (b > 0 ? b : 1) : 8 * NSM);
}

// ------------------------------------------------------------------------------ tcgen05 path
static thread_local uint8_t *g_scr = nullptr;
static thread_local size_t g_scr_bytes = 0;
static thread_local uint64_t g_extra = 0;
void set_scratch(void *p, size_t bytes) {
  g_scr = static_cast<uint8_t *>(p);
  g_scr_bytes = p ? bytes : 0;
}
uint64_t take_extra_launches() {
  const uint64_t e = g_extra;
  g_extra = 0;
  return e;
}
static int r8i(int x) { return (x + 7) & ~7; }
// dst[r][0..ldd) = rb(src[r][0..cols)), zero beyond cols
__global__ void cast_pad_k(__nv_bfloat16 *dst, int ldd, const float *src, int lds, int rows, int cols) {
  const int64_t n = (int64_t)rows * ldd;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / ldd), c = (int)(e - (int64_t)r * ldd);
    dst[e] = __float2bfloat16_rn(c < cols ? src[(size_t)r * lds + c] : 0.f);
  }
}
// C[M][N] (+)= A . B^T with A stored [a_rows][a_cols] (pitch lda, a_mn: [K][M]) and B likewise;
// false when this call stays on the SIMT kernel (f32 mode, too little work, scratch too small)
static bool tc_gemm(float *C, int ldc, bool acc, const float *A, int a_rows, int a_cols, int lda, bool a_mn,
                    const float *B, int b_rows, int b_cols, int ldb, bool b_mn, int M, int N, int K,
                    bool rx, bool rw, cudaStream_t s, cudaError_t *err) {
  if (!rx || !rw || (long long)M * N * K < (1ll << 21) || M <= 0 || N <= 0 || K <= 0) return false;
  const size_t abytes = (((size_t)a_rows * r8i(a_cols) * 2) + 255) & ~size_t(255);
  const size_t bbytes = (size_t)b_rows * r8i(b_cols) * 2;
  if (!g_scr || abytes + bbytes > g_scr_bytes) return false;
  __nv_bfloat16 *Ab = reinterpret_cast<__nv_bfloat16 *>(g_scr), *Bb = reinterpret_cast<__nv_bfloat16 *>(g_scr + abytes);
  cast_pad_k<<<blocks_for((int64_t)a_rows * r8i(a_cols)), 256, 0, s>>>(Ab, r8i(a_cols), A, lda, a_rows, a_cols);
  cast_pad_k<<<blocks_for((int64_t)b_rows * r8i(b_cols)), 256, 0, s>>>(Bb, r8i(b_cols), B, ldb, b_rows, b_cols);
  g_extra += 2;
  GemmOp op;
  op.M = M; op.N = N; op.K = K;
  op.A = Ab; op.lda = r8i(a_cols); op.a_mn = a_mn;
  op.B = Bb; op.ldb = r8i(b_cols); op.b_mn = b_mn;
  op.ep.C = C; op.ep.ldc = ldc; op.ep.accumulate = acc;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = gemm_bf16(op, s);
  *err = e;
  return true;
}

// ------------------------------------------------------------------------------ GEMMs (16x16 tiles)
constexpr int TS = 16;
__global__ void gemm_nt_k(float *Y, const float *X, const float *W, int n, int N, int K, int ldx, int ldw,
                          int ldy, bool acc, bool rx, bool rw) {
  __shared__ float sx[TS][TS + 1], sw[TS][TS + 1];
  const int r = blockIdx.y * TS + threadIdx.y, c = blockIdx.x * TS + threadIdx.x;
  float a = 0.f;
  for (int k0 = 0; k0 < K; k0 += TS) {
    const int kx = k0 + threadIdx.x;
    sx[threadIdx.y][threadIdx.x] = (r < n && kx < K) ? rnd(X[(size_t)r * ldx + kx], rx) : 0.f;
    const int wr = blockIdx.x * TS + threadIdx.y;
    sw[threadIdx.y][threadIdx.x] = (wr < N && kx < K) ? rnd(W[(size_t)wr * ldw + kx], rw) : 0.f;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < TS; ++k) a += sx[threadIdx.y][k] * sw[threadIdx.x][k];
    __syncthreads();
  }
  if (r < n && c < N) Y[(size_t)r * ldy + c] = acc ? Y[(size_t)r * ldy + c] + a : a;
}
cudaError_t gemm_nt(float *Y, const float *X, const float *W, int n, int N, int K, int ldx, int ldw,
                    int ldy, bool acc, bool rx, bool rw, cudaStream_t s) {
  cudaError_t te;
  if (tc_gemm(Y, ldy, acc, X, n, K, ldx, false, W, N, K, ldw, false, n, N, K, rx, rw, s, &te)) return te;
  dim3 g((N + TS - 1) / TS, (n + TS - 1) / TS);
  gemm_nt_k<<<g, dim3(TS, TS), 0, s>>>(Y, X, W, n, N, K, ldx, ldw, ldy, acc, rx, rw);
  return cudaGetLastError();
}
__global__ void gemm_nn_k(float *Y, const float *D, const float *W, int n, int N, int K, int ldd, int ldw,
                          int ldy, bool acc, bool rd, bool rw) {
  __shared__ float sd[TS][TS + 1], sw[TS][TS + 1];
  const int r = blockIdx.y * TS + threadIdx.y, c = blockIdx.x * TS + threadIdx.x;  // c in [0, K)
  float a = 0.f;
  for (int j0 = 0; j0 < N; j0 += TS) {
    const int jd = j0 + threadIdx.x;
    sd[threadIdx.y][threadIdx.x] = (r < n && jd < N) ? rnd(D[(size_t)r * ldd + jd], rd) : 0.f;
    const int jw = j0 + threadIdx.y;
    sw[threadIdx.y][threadIdx.x] = (jw < N && c < K) ? rnd(W[(size_t)jw * ldw + c], rw) : 0.f;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < TS; ++j) a += sd[threadIdx.y][j] * sw[j][threadIdx.x];
    __syncthreads();
  }
  if (r < n && c < K) Y[(size_t)r * ldy + c] = acc ? Y[(size_t)r * ldy + c] + a : a;
}
cudaError_t gemm_nn(float *Y, const float *D, const float *W, int n, int N, int K, int ldd, int ldw,
                    int ldy, bool acc, bool rd, bool rw, cudaStream_t s) {
  // Y[n][K] = D[n][N] . W[N][K]: reduction over N; W is the MN-major ([K_red][N_out]) operand
  cudaError_t te;
  if (tc_gemm(Y, ldy, acc, D, n, N, ldd, false, W, N, K, ldw, true, n, K, N, rd, rw, s, &te)) return te;
  dim3 g((K + TS - 1) / TS, (n + TS - 1) / TS);
  gemm_nn_k<<<g, dim3(TS, TS), 0, s>>>(Y, D, W, n, N, K, ldd, ldw, ldy, acc, rd, rw);
  return cudaGetLastError();
}
__global__ void gemm_tn_k(float *G, const float *D, const float *X, int n, int N, int K, int ldd, int ldx,
                          int ldg, bool acc, bool rd, bool rx) {
  __shared__ float sd[TS][TS + 1], sx[TS][TS + 1];
  const int row = blockIdx.y * TS + threadIdx.y;  // in [0, N)
  const int col = blockIdx.x * TS + threadIdx.x;  // in [0, K)
  float a = 0.f;
  for (int r0 = 0; r0 < n; r0 += TS) {
    const int rr = r0 + threadIdx.x;
    const int dc = blockIdx.y * TS + threadIdx.y;
    sd[threadIdx.y][threadIdx.x] = (rr < n && dc < N) ? rnd(D[(size_t)rr * ldd + dc], rd) : 0.f;
    const int rx2 = r0 + threadIdx.y;
    sx[threadIdx.y][threadIdx.x] = (rx2 < n && col < K) ? rnd(X[(size_t)rx2 * ldx + col], rx) : 0.f;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < TS; ++j) a += sd[threadIdx.y][j] * sx[j][threadIdx.x];
    __syncthreads();
  }
  if (row < N && col < K) G[(size_t)row * ldg + col] = acc ? G[(size_t)row * ldg + col] + a : a;
}
cudaError_t gemm_tn(float *G, const float *D, const float *X, int n, int N, int K, int ldd, int ldx,
                    int ldg, bool acc, bool rd, bool rx, cudaStream_t s) {
  // G[N][K] = D[n][N]^T . X[n][K]: reduction over n; both operands MN-major
  cudaError_t te;
  if (tc_gemm(G, ldg, acc, D, n, N, ldd, true, X, n, K, ldx, true, N, K, n, rd, rx, s, &te)) return te;
  dim3 g((K + TS - 1) / TS, (N + TS - 1) / TS);
  gemm_tn_k<<<g, dim3(TS, TS), 0, s>>>(G, D, X, n, N, K, ldd, ldx, ldg, acc, rd, rx);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------ element-wise
__global__ void add_bias_k(float *Y, const float *b, int n, int N, int ldy) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)n * N; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / N), c = (int)(e % N);
    Y[(size_t)r * ldy + c] += b[c];
  }
}
cudaError_t add_bias(float *Y, const float *b, int n, int N, int ldy, cudaStream_t s) {
  add_bias_k<<<blocks_for((int64_t)n * N), 256, 0, s>>>(Y, b, n, N, ldy);
  return cudaGetLastError();
}
__global__ void colsum_k(float *g, const float *D, int n, int N, int ldd, bool acc, bool rd) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < N; c += gridDim.x * blockDim.x) {
    float a = 0.f;
    for (int r = 0; r < n; ++r) a += rnd(D[(size_t)r * ldd + c], rd);
    g[c] = acc ? g[c] + a : a;
  }
}
cudaError_t colsum(float *g, const float *D, int n, int N, int ldd, bool acc, bool rd, cudaStream_t s) {
  colsum_k<<<blocks_for(N), 256, 0, s>>>(g, D, n, N, ldd, acc, rd);
  return cudaGetLastError();
}
__global__ void fill_k(float *p, float v, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) p[e] = v;
}
cudaError_t fill(float *p, float v, int64_t n, cudaStream_t s) {
  fill_k<<<blocks_for(n), 256, 0, s>>>(p, v, n);
  return cudaGetLastError();
}
__global__ void fill_i_k(int *p, int v, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) p[e] = v;
}
cudaError_t fill_i(int *p, int v, int64_t n, cudaStream_t s) {
  fill_i_k<<<blocks_for(n), 256, 0, s>>>(p, v, n);
  return cudaGetLastError();
}
__global__ void tanh_inplace_k(float *y, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    y[e] = tanhf(y[e]);
}
cudaError_t tanh_inplace(float *y, int64_t n, cudaStream_t s) {
  tanh_inplace_k<<<blocks_for(n), 256, 0, s>>>(y, n);
  return cudaGetLastError();
}
__global__ void tanh_bwd_k(float *dz, const float *dh, const float *h, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    dz[e] = dh[e] * (1.f - h[e] * h[e]);
}
cudaError_t tanh_bwd(float *dz, const float *dh, const float *h, int64_t n, cudaStream_t s) {
  tanh_bwd_k<<<blocks_for(n), 256, 0, s>>>(dz, dh, h, n);
  return cudaGetLastError();
}
__global__ void err_to_float_k(float *y, const int *err) { y[0] = err[0] != 0 ? 1.f : 0.f; }
cudaError_t err_to_float(float *y, const int *err, cudaStream_t s) {
  err_to_float_k<<<1, 1, 0, s>>>(y, err);
  return cudaGetLastError();
}
__global__ void axpy_k(float *y, const float *x, float a, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) y[e] += a * x[e];
}
cudaError_t axpy(float *y, const float *x, float a, int64_t n, cudaStream_t s) {
  axpy_k<<<blocks_for(n), 256, 0, s>>>(y, x, a, n);
  return cudaGetLastError();
}
__global__ void copy_k(float *y, const float *x, int64_t n, bool r) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) y[e] = rnd(x[e], r);
}
cudaError_t copy(float *y, const float *x, int64_t n, cudaStream_t s) {
  copy_k<<<blocks_for(n), 256, 0, s>>>(y, x, n, false);
  return cudaGetLastError();
}
cudaError_t round_copy(float *y, const float *x, int64_t n, bool r, cudaStream_t s) {
  copy_k<<<blocks_for(n), 256, 0, s>>>(y, x, n, r);
  return cudaGetLastError();
}
__global__ void copy_i_k(int *y, const int *x, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) y[e] = x[e];
}
cudaError_t copy_i(int *y, const int *x, int64_t n, cudaStream_t s) {
  copy_i_k<<<blocks_for(n), 256, 0, s>>>(y, x, n);
  return cudaGetLastError();
}
__global__ void i64_to_i32_k(int *y, const long long *x, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const long long v = x[e];
    y[e] = (v > 2147483647LL || v < -2147483647LL) ? -1 : (int)v;  // out of range -> invalid id
  }
}
cudaError_t i64_to_i32(int *y, const long long *x, int64_t n, cudaStream_t s) {
  i64_to_i32_k<<<blocks_for(n), 256, 0, s>>>(y, x, n);
  return cudaGetLastError();
}
__global__ void embedding_k(float *X, const float *E, const int *ids, int n, int V, int Ed, bool r, int *err) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)n * Ed; e += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(e / Ed), k = (int)(e % Ed);
    int id = ids[row];
    if (id < 0 || id >= V) { if (k == 0) atomicOr(err, 1); id = 0; }
    X[e] = rnd(E[(size_t)id * Ed + k], r);
  }
}
cudaError_t embedding(float *X, const float *E, const int *ids, int n, int V, int Ed, bool r, int *err,
                      cudaStream_t s) {
  embedding_k<<<blocks_for((int64_t)n * Ed), 256, 0, s>>>(X, E, ids, n, V, Ed, r, err);
  return cudaGetLastError();
}
__global__ void embedding_bwd_k(float *dE, const float *dX, const int *ids, int n, int V, int Ed) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < Ed; k += gridDim.x * blockDim.x)
    for (int r = 0; r < n; ++r) {
      const int id = ids[r];
      if (id >= 0 && id < V) dE[(size_t)id * Ed + k] += dX[(size_t)r * Ed + k];
    }
}
cudaError_t embedding_bwd(float *dE, const float *dX, const int *ids, int n, int V, int Ed, cudaStream_t s) {
  embedding_bwd_k<<<blocks_for(Ed, 128), 128, 0, s>>>(dE, dX, ids, n, V, Ed);
  return cudaGetLastError();
}
__global__ void column_k(int *out, const int *M, int rows, int W, int t, int *err) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < rows) {
    if (t < 0 || t >= W) { if (r == 0) atomicOr(err, 4); out[r] = 0; }
    else out[r] = M[(size_t)r * W + t];
  }
}
cudaError_t column(int *out, const int *M, int rows, int W, int t, int *err, cudaStream_t s) {
  column_k<<<(rows + 255) / 256, 256, 0, s>>>(out, M, rows, W, t, err);
  return cudaGetLastError();
}
__global__ void element_i_k(int *out, const int *v, int n, int i, int *err) {
  if (i < 0 || i >= n) { atomicOr(err, 8); *out = 0; } else *out = v[i];
}
cudaError_t element_i(int *out, const int *v, int n, int i, int *err, cudaStream_t s) {
  element_i_k<<<1, 1, 0, s>>>(out, v, n, i, err);
  return cudaGetLastError();
}
__global__ void element_f_k(float *out, const float *v, int n, int i, int *err) {
  if (i < 0 || i >= n) { atomicOr(err, 8); *out = 0.f; } else *out = v[i];
}
cudaError_t element_f(float *out, const float *v, int n, int i, int *err, cudaStream_t s) {
  element_f_k<<<1, 1, 0, s>>>(out, v, n, i, err);
  return cudaGetLastError();
}
__global__ void less_iv_k(int *out, int a, const int *v, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = a < v[i];
}
cudaError_t less_iv(int *out, int a, const int *v, int n, cudaStream_t s) {
  less_iv_k<<<(n + 255) / 256, 256, 0, s>>>(out, a, v, n);
  return cudaGetLastError();
}
__global__ void less_vi_k(int *out, const int *v, int a, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = v[i] < a;
}
cudaError_t less_vi(int *out, const int *v, int a, int n, cudaStream_t s) {
  less_vi_k<<<(n + 255) / 256, 256, 0, s>>>(out, v, a, n);
  return cudaGetLastError();
}
__global__ void cmp_scalar_k(int *out, const int *x, int a, int op) {
  const int v = *x;
  *out = op == 0 ? (v < a) : op == 1 ? (a < v) : (v == a);
}
cudaError_t cmp_scalar(int *out, const int *x, int a, int op, cudaStream_t s) {
  cmp_scalar_k<<<1, 1, 0, s>>>(out, x, a, op);
  return cudaGetLastError();
}
__global__ void max_reduce_k(int *out, const int *v, int n) {
  __shared__ int m;
  if (threadIdx.x == 0) m = -2147483647 - 1;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) atomicMax(&m, v[i]);
  __syncthreads();
  if (threadIdx.x == 0) *out = m;
}
cudaError_t max_reduce(int *out, const int *v, int n, cudaStream_t s) {
  max_reduce_k<<<1, 256, 0, s>>>(out, v, n);
  return cudaGetLastError();
}
__global__ void sum_all_k(float *out, const float *x, int64_t n) {
  if (threadIdx.x == 0) {
    float a = 0.f;
    for (int64_t i = 0; i < n; ++i) a += x[i];
    *out = a;
  }
}
cudaError_t sum_all(float *out, const float *x, int64_t n, cudaStream_t s) {
  sum_all_k<<<1, 32, 0, s>>>(out, x, n);
  return cudaGetLastError();
}
__global__ void seq_mask_k(int *out, const int *lens, int B, int T) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < B * T) out[i] = (i / B) < lens[i % B];
}
cudaError_t seq_mask(int *out, const int *lens, int B, int T, cudaStream_t s) {
  seq_mask_k<<<(B * T + 255) / 256, 256, 0, s>>>(out, lens, B, T);
  return cudaGetLastError();
}
__global__ void time_major_k(int *out, const int *M, int B, int W, int T, int *err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < B * T) {
    const int t = i / B, b = i % B;
    if (t >= W) { atomicOr(err, 4); out[i] = 0; } else out[i] = M[(size_t)b * W + t];
  }
}
cudaError_t time_major(int *out, const int *M, int B, int W, int T, int *err, cudaStream_t s) {
  time_major_k<<<(B * T + 255) / 256, 256, 0, s>>>(out, M, B, W, T, err);
  return cudaGetLastError();
}
__global__ void add_f_k(float *out, const float *a, const float *b, int64_t n, int64_t nb) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = a[e] + b[nb == 1 ? 0 : e];
}
cudaError_t add_f(float *out, const float *a, const float *b, int64_t n, int64_t nb, cudaStream_t s) {
  add_f_k<<<blocks_for(n), 256, 0, s>>>(out, a, b, n, nb);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------ cells
__global__ void lstm_fwd_k(float *gates, float *c2, float *h2, const float *Z, const float *c, const float *h,
                           const int *valid, int B, int H) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < B * H; e += gridDim.x * blockDim.x) {
    const int b = e / H, u = e % H;
    const float *z = Z + (size_t)b * 4 * H;
    const float ig = sigmoidf_(z[u]), fg = sigmoidf_(z[H + u]), gg = tanhf(z[2 * H + u]), og = sigmoidf_(z[3 * H + u]);
    float *g = gates + (size_t)b * 4 * H;
    g[u] = ig; g[H + u] = fg; g[2 * H + u] = gg; g[3 * H + u] = og;
    const float cc = fg * c[e] + ig * gg;
    const bool v = valid[b] != 0;
    c2[e] = v ? cc : c[e];
    h2[e] = v ? og * tanhf(cc) : h[e];
  }
}
cudaError_t lstm_fwd(float *gates, float *c2, float *h2, const float *Z, const float *c, const float *h,
                     const int *valid, int B, int H, cudaStream_t s) {
  lstm_fwd_k<<<blocks_for(B * H), 256, 0, s>>>(gates, c2, h2, Z, c, h, valid, B, H);
  return cudaGetLastError();
}
__global__ void lstm_bwd_k(float *dz, float *dh_pass, float *dc_prev, const float *dh2, const float *dc2,
                           const float *gates, const float *c, const float *c2, const int *valid, int B, int H) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < B * H; e += gridDim.x * blockDim.x) {
    const int b = e / H, u = e % H;
    const float *g = gates + (size_t)b * 4 * H;
    float *d = dz + (size_t)b * 4 * H;
    const float ig = g[u], fg = g[H + u], gg = g[2 * H + u], og = g[3 * H + u];
    if (valid[b] != 0) {
      const float tc = tanhf(c2[e]);
      const float dout = dh2[e] * tc;
      const float dc = dc2[e] + dh2[e] * og * (1.f - tc * tc);
      d[u] = dc * gg * ig * (1.f - ig);
      d[H + u] = dc * c[e] * fg * (1.f - fg);
      d[2 * H + u] = dc * ig * (1.f - gg * gg);
      d[3 * H + u] = dout * og * (1.f - og);
      dc_prev[e] = dc * fg;
      dh_pass[e] = 0.f;
    } else {
      d[u] = d[H + u] = d[2 * H + u] = d[3 * H + u] = 0.f;
      dc_prev[e] = dc2[e];
      dh_pass[e] = dh2[e];
    }
  }
}
cudaError_t lstm_bwd(float *dz, float *dh_pass, float *dc_prev, const float *dh2, const float *dc2,
                     const float *gates, const float *c, const float *c2, const int *valid, int B, int H,
                     cudaStream_t s) {
  lstm_bwd_k<<<blocks_for(B * H), 256, 0, s>>>(dz, dh_pass, dc_prev, dh2, dc2, gates, c, c2, valid, B, H);
  return cudaGetLastError();
}
__global__ void tree_leaf_fwd_k(float *gates, float *c, float *h, const float *Z, const float *b, int n, int H) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * H; e += gridDim.x * blockDim.x) {
    const int r = e / H, u = e % H;
    const float *z = Z + (size_t)r * 3 * H;
    const float ig = sigmoidf_(z[u] + b[u]), og = sigmoidf_(z[H + u] + b[H + u]), ug = tanhf(z[2 * H + u] + b[2 * H + u]);
    float *g = gates + (size_t)r * 3 * H;
    g[u] = ig; g[H + u] = og; g[2 * H + u] = ug;
    c[e] = ig * ug;
    h[e] = og * tanhf(ig * ug);
  }
}
cudaError_t tree_leaf_fwd(float *gates, float *c, float *h, const float *Z, const float *b, int n, int H,
                          cudaStream_t s) {
  tree_leaf_fwd_k<<<blocks_for(n * H), 256, 0, s>>>(gates, c, h, Z, b, n, H);
  return cudaGetLastError();
}
__global__ void tree_leaf_bwd_k(float *dz, const float *dh, const float *dcin, const float *gates,
                                const float *c, int n, int H) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * H; e += gridDim.x * blockDim.x) {
    const int r = e / H, u = e % H;
    const float *g = gates + (size_t)r * 3 * H;
    const float ig = g[u], og = g[H + u], ug = g[2 * H + u];
    const float tc = tanhf(c[e]);
    const float dc = dcin[e] + dh[e] * og * (1.f - tc * tc);
    float *d = dz + (size_t)r * 3 * H;
    d[u] = dc * ug * ig * (1.f - ig);
    d[H + u] = dh[e] * tc * og * (1.f - og);
    d[2 * H + u] = dc * ig * (1.f - ug * ug);
  }
}
cudaError_t tree_leaf_bwd(float *dz, const float *dh, const float *dcin, const float *gates,
                          const float *c, int n, int H, cudaStream_t s) {
  tree_leaf_bwd_k<<<blocks_for(n * H), 256, 0, s>>>(dz, dh, dcin, gates, c, n, H);
  return cudaGetLastError();
}
__global__ void tree_cell_fwd_k(float *gates, float *c, float *h, const float *Z, const float *b,
                                const float *cl, const float *cr, int n, int H) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * H; e += gridDim.x * blockDim.x) {
    const int r = e / H, u = e % H;
    const float *z = Z + (size_t)r * 5 * H;
    const float ig = sigmoidf_(z[u] + b[u]), fl = sigmoidf_(z[H + u] + b[H + u]);
    const float fr = sigmoidf_(z[2 * H + u] + b[2 * H + u]), og = sigmoidf_(z[3 * H + u] + b[3 * H + u]);
    const float ug = tanhf(z[4 * H + u] + b[4 * H + u]);
    float *g = gates + (size_t)r * 5 * H;
    g[u] = ig; g[H + u] = fl; g[2 * H + u] = fr; g[3 * H + u] = og; g[4 * H + u] = ug;
    const float cc = ig * ug + fl * cl[e] + fr * cr[e];
    c[e] = cc;
    h[e] = og * tanhf(cc);
  }
}
cudaError_t tree_cell_fwd(float *gates, float *c, float *h, const float *Z, const float *b,
                          const float *cl, const float *cr, int n, int H, cudaStream_t s) {
  tree_cell_fwd_k<<<blocks_for(n * H), 256, 0, s>>>(gates, c, h, Z, b, cl, cr, n, H);
  return cudaGetLastError();
}
__global__ void tree_cell_bwd_k(float *dz, float *dcl, float *dcr, const float *dh, const float *dcin,
                                const float *gates, const float *c, const float *cl, const float *cr, int n, int H) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * H; e += gridDim.x * blockDim.x) {
    const int r = e / H, u = e % H;
    const float *g = gates + (size_t)r * 5 * H;
    const float ig = g[u], fl = g[H + u], fr = g[2 * H + u], og = g[3 * H + u], ug = g[4 * H + u];
    const float tc = tanhf(c[e]);
    const float dc = dcin[e] + dh[e] * og * (1.f - tc * tc);
    float *d = dz + (size_t)r * 5 * H;
    d[u] = dc * ug * ig * (1.f - ig);
    d[H + u] = dc * cl[e] * fl * (1.f - fl);
    d[2 * H + u] = dc * cr[e] * fr * (1.f - fr);
    d[3 * H + u] = dh[e] * tc * og * (1.f - og);
    d[4 * H + u] = dc * ig * (1.f - ug * ug);
    dcl[e] = dc * fl;
    dcr[e] = dc * fr;
  }
}
cudaError_t tree_cell_bwd(float *dz, float *dcl, float *dcr, const float *dh, const float *dcin,
                          const float *gates, const float *c, const float *cl, const float *cr, int n,
                          int H, cudaStream_t s) {
  tree_cell_bwd_k<<<blocks_for(n * H), 256, 0, s>>>(dz, dcl, dcr, dh, dcin, gates, c, cl, cr, n, H);
  return cudaGetLastError();
}
__global__ void tree_bias_k(float *out, const float *b, int H, int cell) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < H; u += gridDim.x * blockDim.x) {
    if (cell) {
      out[u] = b[u]; out[H + u] = b[H + u]; out[2 * H + u] = b[H + u];
      out[3 * H + u] = b[2 * H + u]; out[4 * H + u] = b[3 * H + u];
    } else {
      out[u] = b[u]; out[H + u] = b[2 * H + u]; out[2 * H + u] = b[3 * H + u];
    }
  }
}
cudaError_t tree_bias(float *out, const float *b, int H, int cell, cudaStream_t s) {
  tree_bias_k<<<(H + 255) / 256, 256, 0, s>>>(out, b, H, cell);
  return cudaGetLastError();
}
__global__ void tree_bias_bwd_k(float *db, const float *g, int H, int cell) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < H; u += gridDim.x * blockDim.x) {
    if (cell) {
      db[u] += g[u]; db[H + u] += g[H + u] + g[2 * H + u]; db[2 * H + u] += g[3 * H + u]; db[3 * H + u] += g[4 * H + u];
    } else {
      db[u] += g[u]; db[2 * H + u] += g[H + u]; db[3 * H + u] += g[2 * H + u];
    }
  }
}
cudaError_t tree_bias_bwd(float *db, const float *g, int H, int cell, cudaStream_t s) {
  tree_bias_bwd_k<<<(H + 255) / 256, 256, 0, s>>>(db, g, H, cell);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------ xent
__global__ void xent_k(float *loss, float *dy, const float *logits, const int *tgt, const int *mask, int n,
                       int C, int *err) {
  __shared__ float s_n;
  __shared__ float part[1024];
  if (threadIdx.x == 0) {
    int k = 0;
    for (int r = 0; r < n; ++r) k += mask[r] != 0;
    s_n = (float)(k > 0 ? k : 1);
  }
  __syncthreads();
  float acc = 0.f;
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    const float *y = logits + (size_t)r * C;
    float *d = dy + (size_t)r * C;
    if (mask[r] == 0) {
      for (int c = 0; c < C; ++c) d[c] = 0.f;
      continue;
    }
    int t = tgt[r];
    if (t < 0 || t >= C) { atomicOr(err, 2); t = 0; }
    float m = -INFINITY;
    for (int c = 0; c < C; ++c) m = fmaxf(m, y[c]);
    float sm = 0.f;
    for (int c = 0; c < C; ++c) sm += expf(y[c] - m);
    const float lse = m + logf(sm);
    for (int c = 0; c < C; ++c) d[c] = (expf(y[c] - lse) - (c == t ? 1.f : 0.f)) / s_n;
    acc += (lse - y[t]) / s_n;
  }
  part[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float a = 0.f;
    for (int i = 0; i < (int)blockDim.x; ++i) a += part[i];
    *loss = a;
  }
}
// Row-parallel form (one block per row; the single-block kernel above took 39 ms of a 67 ms
// imperative C2 step): valid-row count, per-row loss and dy, then the loss summed in row order
// (deterministic). Same arithmetic per element as xent_k.
__global__ void count_valid_k(float *n_valid, const int *mask, int n) {
  __shared__ int part[256];
  int k = 0;
  for (int r = threadIdx.x; r < n; r += blockDim.x) k += mask[r] != 0;
  part[threadIdx.x] = k;
  __syncthreads();
  if (threadIdx.x == 0) {
    int a = 0;
    for (int i = 0; i < (int)blockDim.x; ++i) a += part[i];
    *n_valid = (float)(a > 0 ? a : 1);
  }
}
__device__ float block_sum_max(float v, float *sh, bool is_max) {
  for (int o = 16; o > 0; o >>= 1) {
    const float x = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmaxf(v, x) : v + x;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    float a = sh[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) a = is_max ? fmaxf(a, sh[i]) : a + sh[i];
    sh[32] = a;
  }
  __syncthreads();
  const float r = sh[32];
  __syncthreads();
  return r;
}
__global__ void xent_rows_k(float *rowloss, float *dy, const float *logits, const int *tgt, const int *mask,
                            const float *n_valid, int C, int *err) {
  __shared__ float sh[33];
  const int r = blockIdx.x;
  const float *y = logits + (size_t)r * C;
  float *d = dy + (size_t)r * C;
  if (mask[r] == 0) {
    for (int c = threadIdx.x; c < C; c += blockDim.x) d[c] = 0.f;
    if (threadIdx.x == 0) rowloss[r] = 0.f;
    return;
  }
  int t = tgt[r];
  if (t < 0 || t >= C) {
    if (threadIdx.x == 0) atomicOr(err, 2);
    t = 0;
  }
  const float sn = *n_valid;
  float m = -INFINITY;
  for (int c = threadIdx.x; c < C; c += blockDim.x) m = fmaxf(m, y[c]);
  m = block_sum_max(m, sh, true);
  float sm = 0.f;
  for (int c = threadIdx.x; c < C; c += blockDim.x) sm += expf(y[c] - m);
  sm = block_sum_max(sm, sh, false);
  const float lse = m + logf(sm);
  for (int c = threadIdx.x; c < C; c += blockDim.x) d[c] = (expf(y[c] - lse) - (c == t ? 1.f : 0.f)) / sn;
  if (threadIdx.x == 0) rowloss[r] = (lse - y[t]) / sn;
}
__global__ void sum_rows_k(float *loss, const float *rowloss, int n) {  // in row order
  if (threadIdx.x == 0) {
    float a = 0.f;
    for (int r = 0; r < n; ++r) a += rowloss[r];
    *loss = a;
  }
}
cudaError_t xent(float *loss, float *dy, const float *logits, const int *tgt, const int *mask, int n,
                 int C, int *err, cudaStream_t s) {
  if (g_scr && g_scr_bytes >= (size_t)(n + 1) * 4 && n > 0) {
    float *nv = reinterpret_cast<float *>(g_scr), *rowloss = nv + 1;
    count_valid_k<<<1, 256, 0, s>>>(nv, mask, n);
    xent_rows_k<<<n, 256, 0, s>>>(rowloss, dy, logits, tgt, mask, nv, C, err);
    sum_rows_k<<<1, 32, 0, s>>>(loss, rowloss, n);
    g_extra += 2;
    return cudaGetLastError();
  }
  xent_k<<<1, 1024, 0, s>>>(loss, dy, logits, tgt, mask, n, C, err);
  return cudaGetLastError();
}
__global__ void sgd_k(float *W, const float *g, float lr, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) W[e] -= lr * g[e];
}
cudaError_t sgd(float *W, const float *g, float lr, int64_t n, cudaStream_t s) {
  sgd_k<<<blocks_for(n), 256, 0, s>>>(W, g, lr, n);
  return cudaGetLastError();
}

}  // namespace imp
}  // namespace jk
