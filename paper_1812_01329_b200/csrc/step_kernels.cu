// step_kernels.cu — SIMT phases of the speculative training step (see step_kernels.h).
// HBM-bound work: 128-bit / coalesced access, grids sized in multiples of the SM count.
#include <algorithm>

#include "common.cuh"
#include "philox.cuh"
#include "step_kernels.h"

namespace jk {

static constexpr int NSM = 148;

// ------------------------------------------------------------------------------ init / guards
__global__ void step_init_kernel(DevStatus *st, unsigned int *bar, int nbar, int stride) {
  pdl_enter();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) {
    st->key = KEY_PASS;
    st->observed = 0;
    st->runtime_err = 0;
    st->status = 0;
    st->loss = 0.f;
    st->trip = 0;
    st->flags = 0;
  }
  for (int k = i; k * stride < nbar; k += gridDim.x * blockDim.x) bar[(size_t)k * stride] = 0;
}

cudaError_t launch_step_init(DevStatus *st, unsigned int *barriers, int nbar, cudaStream_t s, int stride) {
  const int n = (nbar + stride - 1) / stride;
  {
    const cudaError_t pe_ = launch_pdl(step_init_kernel, dim3(std::max(1, std::min((n + 255) / 256, 8))), dim3(256), 0, s, st, barriers, nbar, stride);
    if (pe_ != cudaSuccess) return pe_;
  }
  return cudaGetLastError();
}

// One block per assumption; each failing element proposes (id << 40 | index) to an atomicMin,
// so the reported failure is the minimum id and, within it, the first element (reading Q9).
JN_DEV void guard_eval(const GuardDesc &g, DevStatus *st, int tid, int nthr) {
  const unsigned long long mask = (1ull << IDX_BITS) - 1;
  if (g.kind == G_TREE) return;  // evaluated by tree_guard_kernel
  if (g.kind == G_FORCED) {
    if (tid == 0) atomicMin(&st->key, ((unsigned long long)g.id << IDX_BITS) | mask);
    return;
  }
  const long long n = (g.kind == G_FIRST_EQ || g.kind == G_FIRST_TRUTH) ? 1 : g.n;
  for (long long i = tid; i < n; i += nthr) {
    const long long v = g.data[i];
    bool bad = false;
    if (g.kind == G_ALL_EQ || g.kind == G_FIRST_EQ) bad = v != g.value;
    else if (g.kind == G_FIRST_TRUTH) bad = (v != 0) != (g.value != 0);
    else if (g.kind == G_RANGE) bad = v < g.lo || v > g.hi;
    if (bad) atomicMin(&st->key, ((unsigned long long)g.id << IDX_BITS) | (unsigned long long)i);
  }
}
__global__ void guards_kernel(GuardList gl, DevStatus *st) {
  pdl_enter();
  guard_eval(gl.g[blockIdx.x], st, threadIdx.x, blockDim.x);
}

// The step's first launch when nothing runs between the init and the guards: one block zeroes
// the status word and the step flags, then evaluates every runtime guard (one launch instead of
// two; bar.sync orders thread 0's key reset before the block's atomicMin proposals).
__global__ void __launch_bounds__(512) step_init_guards_kernel(DevStatus *st, unsigned int *bar, int nbar,
                                                              int stride, GuardList gl) {
  pdl_enter();
  if (threadIdx.x == 0) {
    st->key = KEY_PASS;
    st->observed = 0;
    st->runtime_err = 0;
    st->status = 0;
    st->loss = 0.f;
    st->trip = 0;
    st->flags = 0;
  }
  for (int k = threadIdx.x; k * stride < nbar; k += blockDim.x) bar[(size_t)k * stride] = 0;
  __syncthreads();
  for (int j = 0; j < gl.n; ++j) guard_eval(gl.g[j], st, threadIdx.x, blockDim.x);
}
cudaError_t launch_step_init_guards(DevStatus *st, unsigned int *barriers, int nbar, int stride,
                                    const GuardList &gl, cudaStream_t s) {
  {
    const cudaError_t pe_ = launch_pdl(step_init_guards_kernel, dim3(1), dim3(512), 0, s, st, barriers, nbar, stride, gl);
    if (pe_ != cudaSuccess) return pe_;
  }
  return cudaGetLastError();
}

cudaError_t launch_guards(const GuardList &gl, DevStatus *st, cudaStream_t s) {
  if (gl.n <= 0) return cudaSuccess;
  {
    const cudaError_t pe_ = launch_pdl(guards_kernel, dim3(gl.n), dim3(128), 0, s, gl, st);
    if (pe_ != cudaSuccess) return pe_;
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------ gather
// one warp per row; X[t*B+b][k] = rb(E[id][k]); ones column at k = Edim.
// blk / nblk: this block among the nblk blocks doing the gather
JN_DEV void gather_body(const float *__restrict__ E, int V, int Edim, const int *__restrict__ tok, int B, int W,
                        int T, const int *T_dev, __nv_bfloat16 *X, int ldx, DevStatus *st, int blk, int nblk) {
  const int warp = (blk * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int rows = T * B;
  const int Tb = T_dev ? *T_dev : T;
  for (int r = warp; r < rows; r += (nblk * blockDim.x) >> 5) {
    const int t = r / B, b = r - t * B;
    int id = tok[(size_t)b * W + t];
    if (id < 0 || id >= V) {
      if (lane == 0 && t < Tb) atomicOr(reinterpret_cast<unsigned int *>(&st->runtime_err), 1u);
      id = 0;
    }
    const float *src = E + (size_t)id * Edim;
    __nv_bfloat16 *dst = X + (size_t)r * ldx;
    if ((Edim & 3) == 0) {
      for (int k = lane * 4; k < Edim; k += 128) {
        const float4 v = *reinterpret_cast<const float4 *>(src + k);
        __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), c = __floats2bfloat162_rn(v.z, v.w);
        *reinterpret_cast<__nv_bfloat162 *>(dst + k) = a;
        *reinterpret_cast<__nv_bfloat162 *>(dst + k + 2) = c;
      }
    } else if ((Edim & 1) == 0) {  // e.g. E = 650: 8-B loads, 4-B stores, all issued before use
#pragma unroll 4
      for (int k = lane * 2; k < Edim; k += 64) {
        const float2 v = *reinterpret_cast<const float2 *>(src + k);
        *reinterpret_cast<__nv_bfloat162 *>(dst + k) = __floats2bfloat162_rn(v.x, v.y);
      }
    } else {
      for (int k = lane; k < Edim; k += 32) dst[k] = __float2bfloat16_rn(src[k]);
    }
    for (int k = Edim + lane; k < ldx; k += 32) dst[k] = __float2bfloat16_rn(k == Edim ? 1.f : 0.f);
  }
}
__global__ void gather_kernel(const float *__restrict__ E, int V, int Edim, const int *__restrict__ tok,
                              int B, int W, int T, const int *T_dev, __nv_bfloat16 *X, int ldx,
                              DevStatus *st) {
  pdl_enter();
  gather_body(E, V, Edim, tok, B, W, T, T_dev, X, ldx, st, blockIdx.x, gridDim.x);
}

cudaError_t launch_gather(const float *E, int V, int Edim, const int *tok, int B, int W, int T,
                          const int *T_dev, __nv_bfloat16 *X, int ldx, DevStatus *st,
                          cudaStream_t s) {
  const int rows = T * B;
  int blocks = (rows * 32 + 255) / 256;
  blocks = blocks < 4 * NSM ? blocks : 4 * NSM;
  {
    const cudaError_t pe_ = launch_pdl(gather_kernel, dim3(blocks), dim3(256), 0, s, E, V, Edim, tok, B, W, T, T_dev, X, ldx, st);
    if (pe_ != cudaSuccess) return pe_;
  }
  return cudaGetLastError();
}

__global__ void trip_kernel(const int *lens, int B, int W, DevStatus *st) {
  pdl_enter();
  if (threadIdx.x == 0) {
    int T = 0;
    for (int b = 0; b < B; ++b) T = max(T, lens[b]);
    st->trip = min(max(T, 0), W);
  }
}
cudaError_t launch_trip(const int *lens, int B, int W, DevStatus *st, cudaStream_t s) {
  {
    const cudaError_t pe_ = launch_pdl(trip_kernel, dim3(1), dim3(32), 0, s, lens, B, W, st);
    if (pe_ != cudaSuccess) return pe_;
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------ casts
// Block: 4 destination rows at a time, each thread 2 columns per row per 512-column chunk, all
// four rows' loads issued before the stores (memory-level parallelism for an HBM-bound copy).
constexpr int CR_ROWS = 4;
__global__ void __launch_bounds__(256) cast_rows_kernel(const float *__restrict__ src, int R, int Cc,
                                                        int ld_src, __nv_bfloat16 *__restrict__ dst,
                                                        int ld_dst, int H) {
  const bool pairs = ((ld_src | Cc) & 1) == 0 && (reinterpret_cast<uintptr_t>(src) & 7) == 0;
  for (int r0 = blockIdx.x * CR_ROWS; r0 < R; r0 += gridDim.x * CR_ROWS) {
    for (int k0 = 0; k0 < ld_dst; k0 += 512) {
      const int k = k0 + 2 * threadIdx.x;
      float2 v[CR_ROWS];
#pragma unroll
      for (int q = 0; q < CR_ROWS; ++q) {
        const int r = r0 + q;
        v[q] = make_float2(0.f, 0.f);
        if (r < R && k < Cc) {
          const int rs = H > 0 ? (r & 3) * H + (r >> 2) : r;  // interleaved row 4u+g <- g*H+u
          const float *sr = src + (size_t)rs * ld_src;
          if (pairs) v[q] = *reinterpret_cast<const float2 *>(sr + k);
          else { v[q].x = sr[k]; if (k + 1 < Cc) v[q].y = sr[k + 1]; }
        }
      }
#pragma unroll
      for (int q = 0; q < CR_ROWS; ++q)
        if (r0 + q < R && k < ld_dst)  // ld_dst is even
          reinterpret_cast<__nv_bfloat162 *>(dst + (size_t)(r0 + q) * ld_dst)[k >> 1] =
              __floats2bfloat162_rn(v[q].x, v[q].y);
    }
  }
}

cudaError_t launch_cast_rows(const float *src, int R, int Cc, int ld_src, __nv_bfloat16 *dst,
                             int ld_dst, int interleave_H, cudaStream_t s) {
  if (ld_dst & 1) return cudaErrorInvalidValue;
  const int blocks = std::min((R + CR_ROWS - 1) / CR_ROWS, 16 * NSM);
  cast_rows_kernel<<<blocks, 256, 0, s>>>(src, R, Cc, ld_src, dst, ld_dst, interleave_H);
  return cudaGetLastError();
}

// WT[u][ri] = rb(W[rc][u]),  ri = 4u'+g <-> rc = g*H+u'.  32x32 smem tiles.
__global__ void cast_transpose_il_kernel(const float *__restrict__ W, int H, __nv_bfloat16 *WT,
                                         int ldwt) {
  __shared__ float tile[32][33];
  const int ri0 = blockIdx.x * 32, u0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int i = ty; i < 32; i += 8) {
    const int ri = ri0 + i, u = u0 + tx;
    float v = 0.f;
    if (ri < 4 * H && u < H) v = W[(size_t)((ri & 3) * H + (ri >> 2)) * H + u];
    tile[i][tx] = v;
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int u = u0 + i, ri = ri0 + tx;
    if (u < H && ri < 4 * H) WT[(size_t)u * ldwt + ri] = __float2bfloat16_rn(tile[tx][i]);
  }
}

cudaError_t launch_cast_transpose_interleaved(const float *W, int H, __nv_bfloat16 *WT, int ldwt,
                                              cudaStream_t s) {
  dim3 grid((4 * H + 31) / 32, (H + 31) / 32);
  cast_transpose_il_kernel<<<grid, dim3(32, 8), 0, s>>>(W, H, WT, ldwt);
  return cudaGetLastError();
}

__global__ void bias_il_kernel(const float *b, int H, float *out) {
  for (int ri = blockIdx.x * blockDim.x + threadIdx.x; ri < 4 * H; ri += gridDim.x * blockDim.x)
    out[ri] = b[(ri & 3) * H + (ri >> 2)];
}
cudaError_t launch_bias_interleave(const float *b, int H, float *out, cudaStream_t s) {
  bias_il_kernel<<<(4 * H + 255) / 256, 256, 0, s>>>(b, H, out);
  return cudaGetLastError();
}

// X[r][col] = v, X[r][col+1 .. zero_to) = 0: one thread per element.
__global__ void fill_col_kernel(__nv_bfloat16 *X, int rows, int ld, int col, float v, int zero_to) {
  const int w = zero_to > col ? zero_to - col : 1;
  const long long n = (long long)rows * w;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(e / w), k = (int)(e - (long long)r * w);
    X[(size_t)r * ld + col + k] = __float2bfloat16_rn(k == 0 ? v : 0.f);
  }
}
cudaError_t launch_fill_col(__nv_bfloat16 *X, int rows, int ld, int col, float v, int zero_to,
                            cudaStream_t s) {
  const long long n = (long long)rows * (zero_to > col ? zero_to - col : 1);
  const int blocks = (int)std::min<long long>((n + 255) / 256, 8 * NSM);
  fill_col_kernel<<<blocks, 256, 0, s>>>(X, rows, ld, col, v, zero_to);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------ fused prep
// Every per-step operand copy of the LM step in ONE launch: row casts (optionally
// gate-interleaving), the interleaved transpose of W_hh, bias interleave, ones-column fill. Each
// segment owns a block range of the 1-D grid sized to its work (launch_prep) and strides its work
// units over that range (bx of gx blocks).
JN_DEV int seg_of_block(const int *blk, int n, int *bx, int *gx) {
  int k = 0;
  while (k + 1 < n && (int)blockIdx.x >= blk[k + 1]) ++k;
  *bx = (int)blockIdx.x - blk[k];
  *gx = blk[k + 1] - blk[k];
  return k;
}
JN_DEV void prep_body(const PrepList &pl) {
  int bx, gx;
  const PrepSeg sg = pl.s[seg_of_block(pl.blk, pl.n, &bx, &gx)];
  switch (sg.kind) {
    case P_CAST_ROWS: {
      // HBM-bound copy: every load of PR rows x (<= 2) 512-column chunks is issued before any
      // store (up to 128 B in flight per thread; the Little's-law depth an SM needs at ~1 us of
      // DRAM latency); wider rows fall back to one chunk at a time
      constexpr int PR = 8;
      const bool pairs = ((sg.ld_src | sg.cols) & 1) == 0 && (reinterpret_cast<uintptr_t>(sg.src) & 7) == 0;
      const int nkc = (sg.ld_dst + 511) / 512;
      for (int r0 = bx * PR; r0 < sg.rows; r0 += gx * PR) {
        for (int kc0 = 0; kc0 < nkc; kc0 += 2) {
          float2 v[PR][2];
#pragma unroll
          for (int q = 0; q < PR; ++q)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              const int r = r0 + q, k = (kc0 + c) * 512 + 2 * threadIdx.x;
              v[q][c] = make_float2(0.f, 0.f);
              if (r < sg.rows && k < sg.cols) {
                const int rs = sg.H > 0 ? (r & 3) * sg.H + (r >> 2) : r;
                const float *sr = sg.src + (size_t)rs * sg.ld_src;
                if (pairs) v[q][c] = __ldcs(reinterpret_cast<const float2 *>(sr + k));
                else { v[q][c].x = sr[k]; if (k + 1 < sg.cols) v[q][c].y = sr[k + 1]; }
              }
            }
#pragma unroll
          for (int q = 0; q < PR; ++q)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              const int k = (kc0 + c) * 512 + 2 * threadIdx.x;
              if (r0 + q < sg.rows && k < sg.ld_dst)  // ld_dst is even
                reinterpret_cast<__nv_bfloat162 *>(sg.dst + (size_t)(r0 + q) * sg.ld_dst)[k >> 1] =
                    __floats2bfloat162_rn(v[q][c].x, v[q][c].y);
            }
        }
      }
    } break;
    case P_CAST_T_IL: {  // WT[u][ri] = rb(W[rc][u]): panels of 32 ri x 128 u, threads as 32 x 8
      __shared__ float tile[32][129];
      const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
      const int H = sg.H, nti = (4 * H + 31) / 32, ntp = (H + 127) / 128;
      for (int tb = bx; tb < nti * ntp; tb += gx) {
        const int ri0 = (tb % nti) * 32, u0 = (tb / nti) * 128;
        float v[4][4];  // all 16 loads of the panel in flight before the shared-memory stores
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int ri = ri0 + ty + 8 * a, u = u0 + 32 * c + tx;
            v[a][c] = (ri < 4 * H && u < H) ? __ldcs(sg.src + (size_t)((ri & 3) * H + (ri >> 2)) * H + u) : 0.f;
          }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c) tile[ty + 8 * a][32 * c + tx] = v[a][c];
        __syncthreads();
        for (int i = ty; i < 128; i += 8) {
          const int u = u0 + i, ri = ri0 + tx;
          if (u < H && ri < 4 * H) sg.dst[(size_t)u * sg.ld_dst + ri] = __float2bfloat16_rn(tile[tx][i]);
        }
        __syncthreads();
      }
    } break;
    case P_BIAS_IL:
      for (int ri = bx * blockDim.x + threadIdx.x; ri < 4 * sg.H; ri += gx * blockDim.x)
        sg.fdst[ri] = sg.src[(ri & 3) * sg.H + (ri >> 2)];
      break;
    case P_FILL_COL: {  // dst[r][col] = 1, dst[r][col+1 .. ld_dst) = 0
      const int w = max(1, sg.ld_dst - sg.cols);
      const long long n = (long long)sg.rows * w;
      for (long long e = bx * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gx * blockDim.x) {
        const int r = (int)(e / w), k = (int)(e - (long long)r * w);
        sg.dst[(size_t)r * sg.ld_dst + sg.cols + k] = __float2bfloat16_rn(k == 0 ? 1.f : 0.f);
      }
    } break;
  }
}

// blocks of a segment: half its grid-stride work units (two per block), at least 1, at most 4 / SM
// blocks of a segment: one per two of its grid-stride work units, at least 1, at most 4 per SM
// (measured at C2 against one unit per block and against 4 / SM for every segment: the prep
// and commit phases 25.9 / 38.7 us vs 27.9 / 40.6 and 30.1 / 44.1 us)
__global__ void __launch_bounds__(256, 5) prep_kernel(PrepList pl) {
  pdl_enter();
  prep_body(pl);
}
// operand prep and the embedding gather in one launch: blocks [0, prep) run the prep segments,
// the rest the gather (independent work; one launch boundary fewer)
__global__ void __launch_bounds__(256, 5) prep_gather_kernel(PrepList pl, const float *__restrict__ E, int V,
                                                           int Edim, const int *__restrict__ tok, int B, int W,
                                                           int T, const int *T_dev, __nv_bfloat16 *X, int ldx,
                                                           DevStatus *st) {
  pdl_enter();
  const int np = pl.blk[pl.n];
  if ((int)blockIdx.x < np) {
    prep_body(pl);
    return;
  }
  gather_body(E, V, Edim, tok, B, W, T, T_dev, X, ldx, st, blockIdx.x - np, gridDim.x - np);
}

static int seg_blocks(long long units) { return (int)std::max(1LL, std::min<long long>(4 * NSM, (units + 1) / 2)); }
cudaError_t launch_prep(const PrepList &pl0, cudaStream_t s) {
  if (pl0.n <= 0) return cudaSuccess;
  PrepList pl = pl0;
  pl.blk[0] = 0;
  for (int k = 0; k < pl.n; ++k) {
    const PrepSeg &g = pl.s[k];
    long long u = 1;
    if (g.kind == P_CAST_ROWS) u = (g.rows + 7) / 8;
    else if (g.kind == P_CAST_T_IL) u = (long long)((4 * g.H + 31) / 32) * ((g.H + 127) / 128);
    else if (g.kind == P_BIAS_IL) u = (4LL * g.H + 255) / 256;
    else if (g.kind == P_FILL_COL) u = ((long long)g.rows * std::max(1, g.ld_dst - g.cols) + 255) / 256;
    pl.blk[k + 1] = pl.blk[k] + seg_blocks(u);
  }
  {
    const cudaError_t pe_ = launch_pdl(prep_kernel, dim3(pl.blk[pl.n]), dim3(256), 0, s, pl);
    if (pe_ != cudaSuccess) return pe_;
  }
  return cudaGetLastError();
}
cudaError_t launch_prep_gather(const PrepList &pl0, const float *E, int V, int Edim, const int *tok, int B, int W,
                              int T, const int *T_dev, __nv_bfloat16 *X, int ldx, DevStatus *st, cudaStream_t s) {
  PrepList pl = pl0;
  pl.blk[0] = 0;
  for (int k = 0; k < pl.n; ++k) {
    const PrepSeg &g = pl.s[k];
    long long u = 1;
    if (g.kind == P_CAST_ROWS) u = (g.rows + 7) / 8;
    else if (g.kind == P_CAST_T_IL) u = (long long)((4 * g.H + 31) / 32) * ((g.H + 127) / 128);
    else if (g.kind == P_BIAS_IL) u = (4LL * g.H + 255) / 256;
    else if (g.kind == P_FILL_COL) u = ((long long)g.rows * std::max(1, g.ld_dst - g.cols) + 255) / 256;
    pl.blk[k + 1] = pl.blk[k] + seg_blocks(u);
  }
  {
    int gblocks = (T * B * 32 + 255) / 256;
    gblocks = gblocks < 4 * NSM ? gblocks : 4 * NSM;
    const cudaError_t pe_ = launch_pdl(prep_gather_kernel, dim3(pl.blk[pl.n] + gblocks), dim3(256), 0, s, pl, E, V,
                                       Edim, tok, B, W, T, T_dev, X, ldx, st);
    if (pe_ != cudaSuccess) return pe_;
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------ xent
template <int NT>
__device__ float block_reduce(float v, float *sh, bool is_max) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float x = __shfl_xor_sync(0xffffffff, v, o);
    v = is_max ? fmaxf(v, x) : v + x;
  }
  if (lane == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    v = lane < NT / 32 ? sh[lane] : (is_max ? -INFINITY : 0.f);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float x = __shfl_xor_sync(0xffffffff, v, o);
      v = is_max ? fmaxf(v, x) : v + x;
    }
    if (lane == 0) sh[32] = v;
  }
  __syncthreads();
  const float r = sh[32];
  __syncthreads();
  return r;
}

template <int NT>
__global__ void __launch_bounds__(NT) xent_kernel(const float *__restrict__ logits, int V, int ldl, int rows,
                                                  const int *__restrict__ tgt, int B, int W,
                                                  const int *lens, const int *T_dev, float n_valid,
                                                  __nv_bfloat16 *dy, int lddy, float *rowloss,
                                                  DevStatus *st, float4 *zero, long long zero_n4) {
  pdl_enter();
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < zero_n4; e += (long long)gridDim.x * blockDim.x)
    zero[e] = make_float4(0.f, 0.f, 0.f, 0.f);
  __shared__ float sh[33];
  __shared__ float s_nv;
  const int Tb = T_dev ? *T_dev : rows / B;
  if (lens && threadIdx.x == 0) {
    int acc = 0;
    for (int b = 0; b < B; ++b) acc += min(lens[b], Tb);
    s_nv = (float)max(acc, 1);
  }
  __syncthreads();
  const float nv = lens ? s_nv : n_valid;
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    const int t = r / B, b = r - t * B;
    const bool valid = t < Tb && (!lens || t < lens[b]);
    const float *y = logits + (size_t)r * ldl;
    __nv_bfloat16 *d = dy + (size_t)r * lddy;
    if (!valid) {
      for (int k = threadIdx.x; k < V; k += NT) d[k] = __float2bfloat16_rn(0.f);
      if (threadIdx.x == 0) rowloss[r] = 0.f;
      continue;
    }
    int tg = tgt[(size_t)b * W + t];
    if (tg < 0 || tg >= V) {
      if (threadIdx.x == 0) atomicOr(reinterpret_cast<unsigned int *>(&st->runtime_err), 2u);
      tg = 0;
    }
    float m = -INFINITY;
    for (int k = threadIdx.x; k < V; k += NT) m = fmaxf(m, y[k]);
    m = block_reduce<NT>(m, sh, true);
    float sum = 0.f;
    for (int k = threadIdx.x; k < V; k += NT) sum += expf(y[k] - m);
    sum = block_reduce<NT>(sum, sh, false);
    const float lse = m + logf(sum);
    const float inv = 1.f / nv;
    for (int k = threadIdx.x; k < V; k += NT) {
      const float p = expf(y[k] - lse) - (k == tg ? 1.f : 0.f);
      d[k] = __float2bfloat16_rn(p * inv);
    }
    if (threadIdx.x == 0) rowloss[r] = (lse - y[tg]) * inv;
  }
}

// Single-read variant: the row lives in registers (NV4 float4 per thread), so logits are read from
// HBM once and dy is written with 8-B stores. Same arithmetic as xent_kernel (max, sum of exp,
// lse, dy = rb((softmax - onehot) / n_valid)); used when V <= NT * 4 * NV4 and rows are 16-B aligned.
template <int NT, int NV4>
__global__ void __launch_bounds__(NT) xent_reg_kernel(const float *__restrict__ logits, int V, int ldl, int rows,
                                                      const int *__restrict__ tgt, int B, int W,
                                                      const int *lens, const int *T_dev, float n_valid,
                                                      __nv_bfloat16 *dy, int lddy, float *rowloss,
                                                      DevStatus *st, float4 *zero, long long zero_n4) {
  pdl_enter();
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < zero_n4; e += (long long)gridDim.x * blockDim.x)
    zero[e] = make_float4(0.f, 0.f, 0.f, 0.f);
  __shared__ float sh[33];
  __shared__ float s_nv;
  const int Tb = T_dev ? *T_dev : rows / B;
  if (lens && threadIdx.x == 0) {
    int acc = 0;
    for (int b = 0; b < B; ++b) acc += min(lens[b], Tb);
    s_nv = (float)max(acc, 1);
  }
  __syncthreads();
  const float nv = lens ? s_nv : n_valid;
  const float inv = 1.f / nv;
  const int V4 = (V + 3) >> 2;
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    const int t = r / B, b = r - t * B;
    const bool valid = t < Tb && (!lens || t < lens[b]);
    const float4 *y4 = reinterpret_cast<const float4 *>(logits + (size_t)r * ldl);
    uint2 *d2 = reinterpret_cast<uint2 *>(dy + (size_t)r * lddy);
    if (!valid) {
      for (int k = threadIdx.x; k < V4; k += NT) d2[k] = make_uint2(0u, 0u);
      if (threadIdx.x == 0) rowloss[r] = 0.f;
      continue;
    }
    int tg = tgt[(size_t)b * W + t];
    if (tg < 0 || tg >= V) {
      if (threadIdx.x == 0) atomicOr(reinterpret_cast<unsigned int *>(&st->runtime_err), 2u);
      tg = 0;
    }
    float4 v[NV4];
    float m = -INFINITY;
#pragma unroll
    for (int i = 0; i < NV4; ++i) {
      const int k4 = threadIdx.x + i * NT;
      v[i] = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      if (k4 < V4) {
        v[i] = __ldcs(y4 + k4);  // streamed: read once
        const int k = 4 * k4;
        if (k + 1 >= V) v[i].y = -INFINITY;
        if (k + 2 >= V) v[i].z = -INFINITY;
        if (k + 3 >= V) v[i].w = -INFINITY;
      }
      m = fmaxf(m, fmaxf(fmaxf(v[i].x, v[i].y), fmaxf(v[i].z, v[i].w)));
    }
    m = block_reduce<NT>(m, sh, true);
    float sum = 0.f;
#pragma unroll
    for (int i = 0; i < NV4; ++i) {  // e = exp(y - m), kept in registers (one exp per logit)
      v[i].x = __expf(v[i].x - m); v[i].y = __expf(v[i].y - m);
      v[i].z = __expf(v[i].z - m); v[i].w = __expf(v[i].w - m);
      sum += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    }
    sum = block_reduce<NT>(sum, sh, false);
    const float lse = m + logf(sum);
    const float sc = inv / sum;  // softmax / n_valid = e * sc
#pragma unroll
    for (int i = 0; i < NV4; ++i) {
      const int k4 = threadIdx.x + i * NT;
      if (k4 >= V4) continue;
      const int k = 4 * k4;
      const float p0 = v[i].x * sc - (k == tg ? inv : 0.f);
      const float p1 = v[i].y * sc - (k + 1 == tg ? inv : 0.f);
      const float p2 = v[i].z * sc - (k + 2 == tg ? inv : 0.f);
      const float p3 = v[i].w * sc - (k + 3 == tg ? inv : 0.f);
      __nv_bfloat162 lo = __floats2bfloat162_rn(p0, p1);
      __nv_bfloat162 hi = __floats2bfloat162_rn(p2, p3);
      if (k + 3 < V) {
        d2[k4] = make_uint2(*reinterpret_cast<unsigned *>(&lo), *reinterpret_cast<unsigned *>(&hi));
      } else {  // ragged tail of the row
        __nv_bfloat16 *d = dy + (size_t)r * lddy + k;
        d[0] = lo.x;
        if (k + 1 < V) d[1] = lo.y;
        if (k + 2 < V) d[2] = hi.x;
      }
    }
    if (threadIdx.x == 0) rowloss[r] = (lse - logits[(size_t)r * ldl + tg]) * inv;
  }
}

// Streaming variant: persistent blocks (two per SM) each own rows r = blockIdx.x + i * gridDim.x;
// row i + 1 is fetched into the other of two shared-memory buffers by one bulk copy while row i
// is reduced, so the HBM stream never waits for a reduction (the register variant above has only
// its own row in flight). Same arithmetic: max, sum of exp(y - m), lse, dy = rb(e * inv / sum -
// onehot * inv), the exponentials recomputed in the second pass rather than stored.
constexpr int XT_NT = 256;
__global__ void __launch_bounds__(XT_NT) xent_tma_kernel(const float *__restrict__ logits, int V, int ldl, int rows,
                                                         const int *__restrict__ tgt, int B, int W,
                                                         const int *lens, const int *T_dev, float n_valid,
                                                         __nv_bfloat16 *dy, int lddy, float *rowloss,
                                                         DevStatus *st, float4 *zero, long long zero_n4) {
  extern __shared__ __align__(16) uint8_t xs_raw[];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ float sh[33];
  __shared__ float s_nv;
  pdl_enter();
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < zero_n4; e += (long long)gridDim.x * blockDim.x)
    zero[e] = make_float4(0.f, 0.f, 0.f, 0.f);
  float *buf = reinterpret_cast<float *>(xs_raw);
  const size_t rb = ((size_t)V * 4 + 15) & ~size_t(15);  // bytes per buffer
  const int Tb = T_dev ? *T_dev : rows / B;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
    int acc = 0;
    if (lens)
      for (int b = 0; b < B; ++b) acc += min(lens[b], Tb);
    s_nv = (float)max(acc, 1);
  }
  __syncthreads();
  const float nv = lens ? s_nv : n_valid;
  const float inv = 1.f / nv;
  const int V4 = V >> 2;  // V % 4 == 0 on this path
  auto valid_row = [&](int r) {
    const int t = r / B, b = r - t * B;
    return t < Tb && (!lens || t < lens[b]);
  };
  auto issue = [&](int r, int k) {  // thread 0: row r into buffer k
    mbar_expect_tx(&bar[k], (uint32_t)V * 4);
    bulk_load(reinterpret_cast<uint8_t *>(buf) + k * rb, logits + (size_t)r * ldl, (uint32_t)V * 4, &bar[k]);
  };
  unsigned ph[2] = {0u, 0u};  // completed loads per buffer (uniform over the block)
  const int r0 = blockIdx.x;
  if (threadIdx.x == 0 && r0 < rows && valid_row(r0)) issue(r0, 0);
  for (int i = 0, r = r0; r < rows; ++i, r += gridDim.x) {
    const int k = i & 1;
    const int rn = r + gridDim.x;
    if (threadIdx.x == 0 && rn < rows && valid_row(rn)) issue(rn, k ^ 1);
    const int t = r / B, b = r - t * B;
    uint2 *d2 = reinterpret_cast<uint2 *>(dy + (size_t)r * lddy);
    if (!valid_row(r)) {
      for (int q = threadIdx.x; q < V4; q += XT_NT) d2[q] = make_uint2(0u, 0u);
      if (threadIdx.x == 0) rowloss[r] = 0.f;
      continue;  // nothing was loaded into buffer k for this row
    }
    int tg = tgt[(size_t)b * W + t];
    if (tg < 0 || tg >= V) {
      if (threadIdx.x == 0) atomicOr(reinterpret_cast<unsigned int *>(&st->runtime_err), 2u);
      tg = 0;
    }
    mbar_wait(&bar[k], ph[k] & 1);
    ++ph[k];
    const float4 *y4 = reinterpret_cast<const float4 *>(reinterpret_cast<uint8_t *>(buf) + k * rb);
    float m = -INFINITY;
    for (int q = threadIdx.x; q < V4; q += XT_NT) {
      const float4 v = y4[q];
      m = fmaxf(m, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
    }
    // the target logit (for the loss) before the buffer is overwritten with the exponentials: read
    // ahead of the reduction's barrier
    const float ytg = threadIdx.x == 0 ? reinterpret_cast<const float *>(y4)[tg] : 0.f;
    m = block_reduce<XT_NT>(m, sh, true);
    float sum = 0.f;
    float4 *e4 = const_cast<float4 *>(y4);
    for (int q = threadIdx.x; q < V4; q += XT_NT) {  // exp once: kept in place for the dy pass
      const float4 v = y4[q];
      const float4 e = make_float4(__expf(v.x - m), __expf(v.y - m), __expf(v.z - m), __expf(v.w - m));
      e4[q] = e;
      sum += (e.x + e.y) + (e.z + e.w);
    }
    sum = block_reduce<XT_NT>(sum, sh, false);
    const float lse = m + logf(sum);
    const float sc = inv / sum;
    for (int q = threadIdx.x; q < V4; q += XT_NT) {
      const float4 v = e4[q];  // this thread's own exponentials
      const int c = 4 * q;
      const float p0 = v.x * sc - (c == tg ? inv : 0.f);
      const float p1 = v.y * sc - (c + 1 == tg ? inv : 0.f);
      const float p2 = v.z * sc - (c + 2 == tg ? inv : 0.f);
      const float p3 = v.w * sc - (c + 3 == tg ? inv : 0.f);
      __nv_bfloat162 lo = __floats2bfloat162_rn(p0, p1);
      __nv_bfloat162 hi = __floats2bfloat162_rn(p2, p3);
      d2[q] = make_uint2(*reinterpret_cast<unsigned *>(&lo), *reinterpret_cast<unsigned *>(&hi));
    }
    if (threadIdx.x == 0) rowloss[r] = (lse - ytg) * inv;
    fence_proxy_async_shared();  // this thread's generic writes of buffer k precede the refill
    __syncthreads();  // every read of buffer k is done before it is refilled (iteration i + 2)
  }
}

cudaError_t launch_xent(const float *logits, int V, int ldl, int rows, const int *tgt, int B, int W,
                        const int *lens, const int *T_dev, float n_valid, __nv_bfloat16 *dy,
                        int lddy, float *rowloss, DevStatus *st, cudaStream_t s, float4 *zero,
                        long long zero_n4) {
  const int xt_smem = 2 * (int)(((size_t)V * 4 + 15) & ~size_t(15));
  if (V % 4 == 0 && (ldl % 4) == 0 && (lddy % 4) == 0 && (reinterpret_cast<uintptr_t>(logits) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(dy) & 7) == 0 && xt_smem <= 110 * 1024 && !getenv("JANUS_XENT_REG")) {
    cudaError_t e = set_smem_once((const void *)xent_tma_kernel, xt_smem);
    if (e != cudaSuccess) return e;
    const int blocks = rows < 2 * NSM ? rows : 2 * NSM;
    return launch_pdl(xent_tma_kernel, dim3(blocks), dim3(XT_NT), (size_t)xt_smem, s, logits, V, ldl, rows, tgt, B,
                      W, lens, T_dev, n_valid, dy, lddy, rowloss, st, zero, zero_n4);
  }
  int blocks = rows < 8 * NSM ? rows : 8 * NSM;
  constexpr int NT = 128, NV4 = 20;  // 4 rows in flight per SM (register-limited)
  const bool aligned = (ldl % 4) == 0 && (lddy % 4) == 0 && (reinterpret_cast<uintptr_t>(logits) & 15) == 0 &&
                       (reinterpret_cast<uintptr_t>(dy) & 7) == 0;
  if (aligned && V <= NT * 4 * NV4) {
    {
    const cudaError_t pe_ = launch_pdl(xent_reg_kernel<NT, NV4>, dim3(blocks), dim3(NT), 0, s, logits, V, ldl, rows, tgt, B, W, lens, T_dev, n_valid, dy,
                                                   lddy, rowloss, st, zero, zero_n4);
    if (pe_ != cudaSuccess) return pe_;
  }
  } else {
    {
    const cudaError_t pe_ = launch_pdl(xent_kernel<256>, dim3(blocks), dim3(256), 0, s, logits, V, ldl, rows, tgt, B, W, lens, T_dev, n_valid, dy,
                                            lddy, rowloss, st, zero, zero_n4);
    if (pe_ != cudaSuccess) return pe_;
  }
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------ dropout
uint32_t dropout_threshold(float p) {
  const double t = (double)p * 4294967296.0;
  return t >= 4294967295.0 ? 0xFFFFFFFFu : (uint32_t)t;
}

// one thread per (row, group of 4 columns): one Philox call gives the group's four words
__global__ void dropout_bf16_kernel(const __nv_bfloat16 *src, __nv_bfloat16 *dst, int rows, int cols, int ld,
                                    const int *key, int site, uint32_t thr, float scale) {
  pdl_enter();
  const uint2 k = make_uint2((uint32_t)key[0], (uint32_t)key[1]);
  const int gq = (ld + 3) >> 2;
  const long long n = (long long)rows * gq;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(e / gq), q = (int)(e - (long long)r * gq);
    const uint4 w = dropout_words(k, site, r, q);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int j = 4 * q + i;
      if (j >= ld) break;
      const size_t o = (size_t)r * ld + j;
      const float v = __bfloat162float(src[o]);
      dst[o] = j < cols ? __float2bfloat16_rn(ws[i] >= thr ? v * scale : 0.f) : src[o];
    }
  }
}
__global__ void dropout_f32_kernel(float *x, int rows, int cols, int ld, const int *key, int site, uint32_t thr,
                                   float scale, int row0) {
  pdl_enter();
  const uint2 k = make_uint2((uint32_t)key[0], (uint32_t)key[1]);
  const int gq = (cols + 3) >> 2;
  const long long n = (long long)rows * gq;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(e / gq), q = (int)(e - (long long)r * gq);
    const uint4 w = dropout_words(k, site, row0 + r, q);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int j = 4 * q + i;
      if (j >= cols) break;
      float *p = x + (size_t)r * ld + j;
      *p = ws[i] >= thr ? *p * scale : 0.f;
    }
  }
}
cudaError_t launch_dropout_bf16(const __nv_bfloat16 *src, __nv_bfloat16 *dst, int rows, int cols, int ld,
                                const int *key, int site, float p, cudaStream_t s) {
  const long long n = (long long)rows * ((ld + 3) / 4);
  const int blocks = (int)std::min<long long>((n + 255) / 256, 8 * NSM);
  return launch_pdl(dropout_bf16_kernel, dim3(blocks), dim3(256), 0, s, src, dst, rows, cols, ld, key, site,
                    dropout_threshold(p), 1.f / (1.f - p));
}
cudaError_t launch_dropout_f32(float *x, int rows, int cols, int ld, const int *key, int site, float p,
                               cudaStream_t s, int row0) {
  const long long n = (long long)rows * ((cols + 3) / 4);
  const int blocks = (int)std::min<long long>((n + 255) / 256, 8 * NSM);
  return launch_pdl(dropout_f32_kernel, dim3(blocks), dim3(256), 0, s, x, rows, cols, ld, key, site,
                    dropout_threshold(p), 1.f / (1.f - p), row0);
}

// ------------------------------------------------------------------------------ embedding grad
// dE[w] = sum of the dX rows r with tok(r) = w (the VJP of the embedding lookup):
//   1. bucket (one block): the first occurrence of each word in row order gets the next slot
//      (atomicMin of the row into owner[w], then a block scan of "is first") — the slot order is
//      deterministic; rows are counted per slot, offsets scanned, and every row appended to its
//      slot's list (append order arbitrary);
//   2. segsum (block per slot): the slot's rows are sorted ascending, warp j sums rows j,
//      j + EG_WARPS, ... over all columns, and the warps' partials are combined in warp order —
//      a fixed summation order, so every dE row is deterministic.
constexpr int EG_MAX = 8192;
constexpr int EG_WARPS = 8;  // 256-thread blocks: several blocks per SM
constexpr int EG_OWNER_SMEM = 24 * 1024;  // vocabularies whose owner table lives in shared memory (96 KB)
JN_DEV int tok_of(const int *tok, int B, int W, int r) {
  const int t = r / B, b = r - t * B;
  return tok[(size_t)b * W + t];
}

JN_DEV int block_excl_scan(int v, int *warp_sums, int *total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[w] = x;
  __syncthreads();
  if (w == 0) {
    int ws = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, ws, o);
      if (lane >= o) ws += y;
    }
    warp_sums[lane] = ws;
  }
  __syncthreads();
  const int r = x - v + (w > 0 ? warp_sums[w - 1] : 0);
  if (total) *total = warp_sums[(blockDim.x >> 5) - 1];
  __syncthreads();
  return r;
}

// owner: V ints preset to INT_MAX; seg_start: n + 1 ints; list: n ints
__global__ void __launch_bounds__(1024) embed_bucket_kernel(const int *tok, int B, int W, int T, const int *T_dev,
                                                            int *owner_g, int V, int owner_sm, int *seg_word,
                                                            int *seg_start, int *nseg, int *list) {
  pdl_enter();
  extern __shared__ int eb_smem[];
  int *s_word = eb_smem;             // [EG_MAX] word of row r, later its slot
  int *s_slot = eb_smem + EG_MAX;    // [EG_MAX] slot of a first-occurrence row
  int *s_cnt = eb_smem + 2 * EG_MAX; // [EG_MAX] rows per slot, then append cursors
  __shared__ int warp_sums[32];
  // first row of each word: in shared memory when the vocabulary fits (no global round trips),
  // else the caller's INT_MAX-preset global array
  int *owner = owner_sm ? eb_smem + 3 * EG_MAX : owner_g;
  if (owner_sm) {
    for (int w = threadIdx.x; w < V; w += blockDim.x) owner[w] = 0x7fffffff;
    __syncthreads();
  }
  const int n = (T_dev ? *T_dev : T) * B;
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    int w = tok_of(tok, B, W, r);
    w = (w >= 0 && w < V) ? w : 0;  // a bad id is reported by the gather (ERR_RUNTIME: no commit)
    s_word[r] = w;
    atomicMin(&owner[w], r);
    s_cnt[r] = 0;
  }
  __syncthreads();
  __threadfence_block();
  // slots in order of first occurrence: scan of is_first over the rows, chunk per thread
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int lo = min(n, (int)threadIdx.x * per), hi = min(n, lo + per);
  int nf = 0;
  for (int r = lo; r < hi; ++r) nf += owner[s_word[r]] == r;
  int total = 0;
  int slot = block_excl_scan(nf, warp_sums, &total);
  for (int r = lo; r < hi; ++r)
    if (owner[s_word[r]] == r) {
      s_slot[r] = slot;  // provisional: first rows know their slot
      seg_word[slot] = s_word[r];
      ++slot;
    }
  __syncthreads();
  // every row: slot of its word (through the first row), count per slot
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    const int sl = s_slot[owner[s_word[r]]];
    atomicAdd(&s_cnt[sl], 1);
    s_word[r] = sl;  // s_word now holds the row's slot
  }
  __syncthreads();
  // offsets
  const int per2 = (total + blockDim.x - 1) / blockDim.x;
  const int lo2 = min(total, (int)threadIdx.x * per2), hi2 = min(total, lo2 + per2);
  int c = 0;
  for (int k = lo2; k < hi2; ++k) c += s_cnt[k];
  int off = block_excl_scan(c, warp_sums, nullptr);
  for (int k = lo2; k < hi2; ++k) {
    const int ck = s_cnt[k];
    seg_start[k] = off;
    s_cnt[k] = off;  // append cursor
    off += ck;
  }
  if (threadIdx.x == 0) {
    *nseg = total;
    seg_start[total] = n;
  }
  __syncthreads();
  for (int r = threadIdx.x; r < n; r += blockDim.x) list[atomicAdd(&s_cnt[s_word[r]], 1)] = r;
}

// dynamic smem: rows[EG_MAX] ints, then part[EG_WARPS][NQ * 32] floats
template <int NQ>
__global__ void __launch_bounds__(EG_WARPS * 32, 2) embed_segsum_kernel(
    const int *seg_start, const int *list, const int *nseg, const float *__restrict__ dX, int ldx, int Edim,
    float *seg_grad, int ldg) {
  pdl_enter();
  extern __shared__ int eg_smem[];
  int *rows = eg_smem;
  float *part = reinterpret_cast<float *>(eg_smem + EG_MAX);  // [EG_WARPS][NQ * 32]
  const int ns = *nseg;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int sgi = blockIdx.x; sgi < ns; sgi += gridDim.x) {
    const int a = seg_start[sgi], cnt = seg_start[sgi + 1] - a;
    // the slot's rows, sorted ascending (bitonic over the next power of two; pads = INT_MAX)
    int np = 1;
    while (np < cnt) np <<= 1;
    for (int i = threadIdx.x; i < np; i += blockDim.x) rows[i] = i < cnt ? list[a + i] : 0x7fffffff;
    __syncthreads();
    for (int k = 2; k <= np; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = threadIdx.x; i < np; i += blockDim.x) {
          const int ixj = i ^ j;
          if (ixj > i) {
            const int x = rows[i], y = rows[ixj];
            if ((x > y) == ((i & k) == 0)) { rows[i] = y; rows[ixj] = x; }
          }
        }
        __syncthreads();
      }
    // warp w sums entries w, w + EG_WARPS, ... over ALL columns at once (lane: columns
    // lane + 32 q), two rows per iteration: up to 2 NQ independent loads in flight per lane
    float acc[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[q] = 0.f;
    int i = w;
    for (; i + 3 * EG_WARPS < cnt; i += 4 * EG_WARPS) {  // four rows in flight per iteration
      const float *rp[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) rp[u] = dX + (size_t)rows[i + u * EG_WARPS] * ldx;
      float x[4][NQ];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const int cc = lane + 32 * q;
          x[u][q] = cc < Edim ? rp[u][cc] : 0.f;
        }
#pragma unroll
      for (int q = 0; q < NQ; ++q) { acc[q] += x[0][q]; acc[q] += x[1][q]; acc[q] += x[2][q]; acc[q] += x[3][q]; }
    }
    for (; i < cnt; i += EG_WARPS) {
      const float *r0p = dX + (size_t)rows[i] * ldx;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int cc = lane + 32 * q;
        acc[q] += cc < Edim ? r0p[cc] : 0.f;
      }
    }
    // combine the warps' partial sums in warp order (deterministic)
#pragma unroll
    for (int q = 0; q < NQ; ++q) part[w * NQ * 32 + lane + 32 * q] = acc[q];
    __syncthreads();
    for (int cc = threadIdx.x; cc < Edim; cc += blockDim.x) {
      float sum = part[cc];
      for (int j = 1; j < EG_WARPS && j < cnt; ++j) sum += part[j * NQ * 32 + cc];
      seg_grad[(size_t)sgi * ldg + cc] = sum;
    }
    __syncthreads();
  }
}

cudaError_t launch_embed_grad(const int *tok, int B, int W, int T, const int *T_dev, int V,
                              const float *dX, int ldx, int Edim, int *seg_word, int *owner,
                              float *seg_grad, int ldg, int *nseg, cudaStream_t s, int part) {
  if (T * B > EG_MAX) return cudaErrorInvalidValue;
  const int owner_sm = V <= EG_OWNER_SMEM;
  cudaError_t e = cudaSuccess;
  if (!owner_sm && part != 2) {
    e = cudaMemsetAsync(owner, 0x7f, (size_t)V * sizeof(int), s);  // INT_MAX-ish
    if (e != cudaSuccess) return e;
  }
  int *seg_start = owner + V;                 // scratch: T*B + 1 ints
  int *list = seg_start + (size_t)T * B + 1;  // scratch: T*B ints
  const int bsmem = (3 * EG_MAX + (owner_sm ? V : 0)) * 4;
  e = set_smem_once((const void *)embed_bucket_kernel, (3 * EG_MAX + EG_OWNER_SMEM) * 4);
  if (e != cudaSuccess) return e;
  if (part != 2) {
    const cudaError_t pe_ = launch_pdl(embed_bucket_kernel, dim3(1), dim3(1024), bsmem, s, tok, B, W, T, T_dev, owner, V, owner_sm, seg_word, seg_start, nseg,
                                             list);
    if (pe_ != cudaSuccess) return pe_;
  }
  if (part == 1) return cudaGetLastError();
  auto go = [&](auto kern, int nq) {
    const int smem = EG_MAX * 4 + EG_WARPS * nq * 32 * 4;
    cudaError_t r = set_smem_once((const void *)kern, smem);
    if (r != cudaSuccess) return r;
    {
    const cudaError_t pe_ = launch_pdl(kern, dim3(8 * NSM), dim3(EG_WARPS * 32), smem, s, seg_start, list, nseg, dX, ldx, Edim, seg_grad, ldg);
    if (pe_ != cudaSuccess) return pe_;
  }
    return cudaGetLastError();
  };
  if (Edim <= 8 * 32) return go(embed_segsum_kernel<8>, 8);
  if (Edim <= 24 * 32) return go(embed_segsum_kernel<24>, 24);
  if (Edim <= 48 * 32) return go(embed_segsum_kernel<48>, 48);
  return cudaErrorInvalidValue;
}

// ------------------------------------------------------------------------------ finalize
JN_DEV void finalize_body(const float *rowloss, int rows, const GuardList &gl, DevStatus *st) {
  __shared__ float sh[1024];
  float acc = 0.f;
  for (int i = threadIdx.x; i < rows; i += blockDim.x) acc += rowloss[i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    st->loss = sh[0];
    const unsigned long long key = st->key;
    if (key != KEY_PASS) {
      st->status = 1;  // JANUS_ASSUMPTION_FAILED
      const unsigned id = (unsigned)(key >> IDX_BITS);
      const unsigned long long idx = key & ((1ull << IDX_BITS) - 1);
      long long obs = -1;
      if (idx != (1ull << IDX_BITS) - 1)
        for (int k = 0; k < gl.n; ++k)
          if (gl.g[k].id == id && gl.g[k].kind != G_FORCED)
            obs = (gl.g[k].kind == G_TREE && (long long)idx >= gl.g[k].n)
                      ? gl.g[k].data2[idx - gl.g[k].n] : gl.g[k].data[idx];
      st->observed = obs;
    } else if (st->runtime_err) {
      st->status = 4;  // JANUS_ERR_RUNTIME
    } else {
      st->status = 0;
    }
  }
}
__global__ void finalize_kernel(const float *rowloss, int rows, GuardList gl, DevStatus *st) {
  pdl_enter();
  finalize_body(rowloss, rows, gl, st);
}

cudaError_t launch_finalize(const float *rowloss, int rows, const GuardList &gl, DevStatus *st,
                            int world_size, cudaStream_t s) {
  (void)world_size;
  {
    const cudaError_t pe_ = launch_pdl(finalize_kernel, dim3(1), dim3(1024), 0, s, rowloss, rows, gl, st);
    if (pe_ != cudaSuccess) return pe_;
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------ data parallel
__global__ void dp_pack_kernel(const DevStatus *st, long long *sc, int rank) { dp_pack(*st, sc, rank); }
cudaError_t launch_dp_pack(const DevStatus *st, long long *scratch, int rank, cudaStream_t s) {
  dp_pack_kernel<<<1, 1, 0, s>>>(st, scratch, rank);
  return cudaGetLastError();
}
__global__ void dp_observed_kernel(const DevStatus *st, long long *sc) { dp_observed(*st, sc); }
cudaError_t launch_dp_observed(const DevStatus *st, long long *scratch, cudaStream_t s) {
  dp_observed_kernel<<<1, 1, 0, s>>>(st, scratch);
  return cudaGetLastError();
}
__global__ void dp_unpack_kernel(DevStatus *st, const long long *sc) { dp_unpack(*st, sc); }
cudaError_t launch_dp_unpack(DevStatus *st, const long long *scratch, cudaStream_t s) {
  dp_unpack_kernel<<<1, 1, 0, s>>>(st, scratch);
  return cudaGetLastError();
}
__global__ void set_failure_kernel(DevStatus *st, unsigned id, long long index, long long observed) {
  dp_set_failure(*st, id, index, observed);
}
cudaError_t launch_set_failure(DevStatus *st, unsigned id, long long index, long long observed,
                               cudaStream_t s) {
  set_failure_kernel<<<1, 1, 0, s>>>(st, id, index, observed);
  return cudaGetLastError();
}
__global__ void scatter_rows_kernel(const float *seg_grad, int ldg, const int *seg_word,
                                    const int *nseg, float *dense, int V, int cols) {
  const long long n = (long long)V * cols;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += stride) dense[e] = 0.f;
  // a grid-wide zero-then-scatter needs ordering: done by the second launch below
}
__global__ void scatter_rows2_kernel(const float *seg_grad, int ldg, const int *seg_word,
                                     const int *nseg, float *dense, int cols) {
  const int ns = *nseg;
  for (int k = blockIdx.x; k < ns; k += gridDim.x)
    for (int j = threadIdx.x; j < cols; j += blockDim.x)
      dense[(size_t)seg_word[k] * cols + j] = seg_grad[(size_t)k * ldg + j];
}
cudaError_t launch_scatter_rows(const float *seg_grad, int ldg, const int *seg_word, const int *nseg,
                                float *dense, int V, int cols, cudaStream_t s) {
  scatter_rows_kernel<<<4 * NSM, 256, 0, s>>>(seg_grad, ldg, seg_word, nseg, dense, V, cols);
  scatter_rows2_kernel<<<4 * NSM, 256, 0, s>>>(seg_grad, ldg, seg_word, nseg, dense, cols);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------ commit
// Predicated on the device status: with any failure nothing is written (all-or-nothing).
JN_DEV void commit_body(const CommitList &cl) {
  int bx, gx;
  const CommitSeg sg = cl.s[seg_of_block(cl.blk, cl.n, &bx, &gx)];
  if (sg.pred && *sg.pred == 0) return;
  const long long stride = (long long)gx * blockDim.x;
  const long long tid = bx * (long long)blockDim.x + threadIdx.x;
  switch (sg.kind) {
    case C_DENSE:  // 4 rows per block iteration, 2 columns per thread, loads before stores
    case C_DENSE_IL: {
      const int ng = sg.ng ? sg.ng : 4;
      const bool pairs = ((sg.cols | sg.ldg) & 1) == 0 &&
                         ((reinterpret_cast<uintptr_t>(sg.dst) | reinterpret_cast<uintptr_t>(sg.grad)) & 7) == 0;
      for (int r0 = bx * CR_ROWS; r0 < sg.rows; r0 += gx * CR_ROWS) {
        for (int k0 = 0; k0 < sg.cols; k0 += 512) {
          const int k = k0 + 2 * threadIdx.x;
          float2 dv[CR_ROWS], gv[CR_ROWS];
#pragma unroll
          for (int q = 0; q < CR_ROWS; ++q) {
            const int rc = r0 + q;
            dv[q] = gv[q] = make_float2(0.f, 0.f);
            if (rc < sg.rows && k < sg.cols) {
              const int ri = sg.kind == C_DENSE ? rc : ng * (rc % sg.H) + rc / sg.H;
              const float *d = sg.dst + (size_t)rc * sg.cols + k;
              const float *g = sg.grad + (size_t)ri * sg.ldg + k;
              if (pairs) { dv[q] = *reinterpret_cast<const float2 *>(d); gv[q] = *reinterpret_cast<const float2 *>(g); }
              else { dv[q].x = d[0]; gv[q].x = g[0]; if (k + 1 < sg.cols) { dv[q].y = d[1]; gv[q].y = g[1]; } }
            }
          }
#pragma unroll
          for (int q = 0; q < CR_ROWS; ++q) {
            const int rc = r0 + q;
            if (rc < sg.rows && k < sg.cols) {
              float *d = sg.dst + (size_t)rc * sg.cols + k;
              const float2 o = make_float2(dv[q].x - sg.lr * gv[q].x, dv[q].y - sg.lr * gv[q].y);
              if (pairs) *reinterpret_cast<float2 *>(d) = o;
              else { d[0] = o.x; if (k + 1 < sg.cols) d[1] = o.y; }
              if (sg.bcopy) {  // the next step's bf16 working copy of this master (R1)
                const int rb = sg.kind == C_DENSE ? rc : ng * (rc % sg.H) + rc / sg.H;
                __nv_bfloat16 *bc = sg.bcopy + (size_t)rb * sg.ldb + k;
                if (pairs) *reinterpret_cast<__nv_bfloat162 *>(bc) = __floats2bfloat162_rn(o.x, o.y);
                else { bc[0] = __float2bfloat16_rn(o.x); if (k + 1 < sg.cols) bc[1] = __float2bfloat16_rn(o.y); }
              }
            }
          }
        }
      }
    } break;
    case C_DENSE_IL_T: {
      // 32 interleaved rows x 64 columns per tile: update the master rows, write the row copy,
      // and through shared memory the transposed copy tcopy[k][ri] (coalesced along ri)
      __shared__ __nv_bfloat16 tt[32][72];
      const int ng = sg.ng ? sg.ng : 4;  // gates per unit (interleaved row ri = ng*u + g)
      const int R = ng * sg.H, nti = (R + 31) / 32, ntk = (sg.cols + 63) / 64;
      const int tr = threadIdx.x >> 3, tc = (threadIdx.x & 7) * 8;  // this thread: row tr, 8 columns
      for (int tb = bx; tb < nti * ntk; tb += gx) {
        const int ri0 = (tb % nti) * 32, k0 = (tb / nti) * 64;
        const int ri = ri0 + tr, rc = (ri % ng) * sg.H + ri / ng;
        float2 dv[4], gv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int k = k0 + tc + 2 * j;
          dv[j] = gv[j] = make_float2(0.f, 0.f);
          if (ri < R && k < sg.cols) {  // cols and pitches even: pairs stay inside a row
            dv[j] = *reinterpret_cast<const float2 *>(sg.dst + (size_t)rc * sg.cols + k);
            gv[j] = __ldcs(reinterpret_cast<const float2 *>(sg.grad + (size_t)ri * sg.ldg + k));
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int k = k0 + tc + 2 * j;
          const float2 o = make_float2(dv[j].x - sg.lr * gv[j].x, dv[j].y - sg.lr * gv[j].y);
          const __nv_bfloat162 ob = __floats2bfloat162_rn(o.x, o.y);
          if (ri < R && k < sg.cols) {
            *reinterpret_cast<float2 *>(sg.dst + (size_t)rc * sg.cols + k) = o;
            *reinterpret_cast<__nv_bfloat162 *>(sg.bcopy + (size_t)ri * sg.ldb + k) = ob;
          }
          *reinterpret_cast<__nv_bfloat162 *>(&tt[tr][tc + 2 * j]) = ob;
        }
        __syncthreads();
        {  // 64 k rows x 32 ri: thread -> k = k0 + t / 4, 8 consecutive ri
          const int kk = threadIdx.x >> 2, r8 = (threadIdx.x & 3) * 8;
          const int k = k0 + kk;
          if (k < sg.cols) {
            __nv_bfloat16 *td = sg.tcopy + (size_t)k * sg.ldt + ri0 + r8;
            if (ri0 + r8 + 8 <= R && ((reinterpret_cast<uintptr_t>(td) & 15) == 0)) {
              __align__(16) __nv_bfloat16 v8[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) v8[i] = tt[r8 + i][kk];
              *reinterpret_cast<uint4 *>(td) = *reinterpret_cast<const uint4 *>(v8);
            } else {
              for (int i = 0; i < 8 && ri0 + r8 + i < R; ++i) td[i] = tt[r8 + i][kk];
            }
          }
        }
        __syncthreads();
      }
    } break;
    case C_TREE_BIAS:  // b blocks (i, f, o, u): internal gates (i, f_l, f_r, o, u), leaf (i, o, u)
      for (long long e = tid; e < 4LL * sg.H; e += stride) {
        const int q = (int)(e / sg.H), u = (int)(e % sg.H);
        const float *gi = sg.grad + (size_t)5 * u * sg.ldg + sg.col;
        const float *gl = sg.grad2 + (size_t)3 * u * sg.ldg2 + sg.col2;
        float g = 0.f;
        if (q == 0) g = gi[0] + gl[0];
        else if (q == 1) g = gi[(size_t)sg.ldg] + gi[2 * (size_t)sg.ldg];
        else if (q == 2) g = gi[3 * (size_t)sg.ldg] + gl[(size_t)sg.ldg2];
        else g = gi[4 * (size_t)sg.ldg] + gl[2 * (size_t)sg.ldg2];
        sg.dst[e] -= sg.lr * g;
      }
      break;
    case C_BIAS_COL:
      for (long long e = tid; e < sg.rows; e += stride)
        sg.dst[e] -= sg.lr * sg.grad[(size_t)e * sg.ldg + sg.col];
      break;
    case C_BIAS_COL_IL:
      for (long long e = tid; e < sg.rows; e += stride) {
        const int rc = (int)e, ri = 4 * (rc % sg.H) + rc / sg.H;
        sg.dst[e] -= sg.lr * sg.grad[(size_t)ri * sg.ldg + sg.col];
      }
      break;
    case C_COPY: {
      const long long n = (long long)sg.rows * sg.cols;
      for (long long e = tid; e < n; e += stride) sg.dst[e] = sg.grad[e];
    } break;
    case C_TAG:
      if (tid == 0) *sg.idst = sg.ival;
      break;
    case C_SPARSE_ROWS: {
      const long long n = (long long)(*sg.nrows) * sg.cols;
      for (long long e = tid; e < n; e += stride) {
        const int k = (int)(e / sg.cols), j = (int)(e - (long long)k * sg.cols);
        sg.dst[(size_t)sg.rows_idx[k] * sg.cols + j] -= sg.lr * sg.grad[(size_t)k * sg.ldg + j];
      }
    } break;
  }
}

__global__ void __launch_bounds__(256, 6) commit_kernel(CommitList cl, const DevStatus *st) {
  pdl_enter();
  if (st->status != 0) return;
  commit_body(cl);
}
// The step's finalize folded into the commit launch: its last block sums the loss rows and writes
// the status word while the commit blocks decide all-or-nothing from the same inputs the status
// is computed from (the minimum failing key and the runtime-error flags), so no block waits for
// another (single-rank steps; with data parallelism the agreed status must precede the commit).
__global__ void __launch_bounds__(256, 6) commit_finalize_kernel(CommitList cl, FinalizeArgs fa, DevStatus *st) {
  pdl_enter();
  if ((int)blockIdx.x == cl.blk[cl.n]) {
    finalize_body(fa.rowloss, fa.rows, fa.gl, st);
    return;
  }
  if (st->key != KEY_PASS || st->runtime_err != 0) return;
  commit_body(cl);
}

static cudaError_t launch_commit_impl(const CommitList &cl0, const FinalizeArgs *fa, DevStatus *st, cudaStream_t s) {
  if (cl0.n <= 0 && !fa) return cudaSuccess;
  CommitList cl = cl0;
  cl.blk[0] = 0;
  for (int k = 0; k < cl.n; ++k) {
    const CommitSeg &g = cl.s[k];
    long long u;
    switch (g.kind) {
      case C_DENSE: case C_DENSE_IL: u = (g.rows + CR_ROWS - 1) / CR_ROWS; break;
      case C_DENSE_IL_T: u = (long long)(((g.ng ? g.ng : 4) * g.H + 31) / 32) * ((g.cols + 63) / 64); break;
      case C_TREE_BIAS: u = (4LL * g.H + 255) / 256; break;
      case C_BIAS_COL: case C_BIAS_COL_IL: u = (g.rows + 255) / 256; break;
      case C_COPY: u = ((long long)g.rows * g.cols + 255) / 256; break;
      case C_TAG: u = 1; break;
      default: u = 8LL * NSM;  // C_SPARSE_ROWS: the row count is known on the device only
    }
    cl.blk[k + 1] = cl.blk[k] + seg_blocks(u);
  }
  {
    const cudaError_t pe_ = fa ? launch_pdl(commit_finalize_kernel, dim3(cl.blk[cl.n] + 1), dim3(256), 0, s, cl, *fa, st)
                               : launch_pdl(commit_kernel, dim3(cl.blk[cl.n]), dim3(256), 0, s, cl,
                                            static_cast<const DevStatus *>(st));
    if (pe_ != cudaSuccess) return pe_;
  }
  return cudaGetLastError();
}
cudaError_t launch_commit(const CommitList &cl, const DevStatus *st, cudaStream_t s) {
  return launch_commit_impl(cl, nullptr, const_cast<DevStatus *>(st), s);
}
cudaError_t launch_commit_finalize(const CommitList &cl, const FinalizeArgs &fa, DevStatus *st, cudaStream_t s) {
  return launch_commit_impl(cl, &fa, st, s);
}

}  // namespace jk
