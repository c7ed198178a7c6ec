// gemm_tc.cu — tcgen05 / TMEM / TMA bf16 GEMM for the batched cell contractions of the LSTM-LM
// and TreeLSTM steps (the only dense contractions on the path: input projections, decoder,
// dgrad and wgrad GEMMs).
//
//   D[M,N] (fp32) = A[M,K] . B[N,K]^T   (+ bias, + existing D), bf16 operands, fp32 accumulate.
//   Either operand may be K-major (K contiguous) or MN-major (M/N contiguous), so wgrad GEMMs
//   (reduction over the token dimension, dW = dz^T x) read the activations in place.
//
// One CTA per 128 x BN output tile, 4 warps: warp0/lane0 issues TMA into a STAGES-deep smem ring
// (128-B swizzle), warp1/lane0 issues tcgen05.mma (M=128, N=BN, K=16) into a TMEM accumulator,
// then all 4 warps drain TMEM (tcgen05.ld 32x32b) and store with the fused epilogue.
#include "common.cuh"
#include "gemm_tc.h"

namespace jk {

template <int BN, int A_MN, int B_MN, int STAGES>
struct GemmCfg {
  static constexpr int BM = 128, BK = 64;
  static constexpr int A_BYTES = BM * BK * 2;  // 16 KB
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

template <int BN, int A_MN, int B_MN, int STAGES>
__global__ void __launch_bounds__(128, 1)
    gemm_bf16_tc_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB, GemmEpilogue ep, int M, int N,
                        int K, const int *K_dev) {
  using C = GemmCfg<BN, A_MN, B_MN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  uint8_t *sA = smem;
  uint8_t *sB = smem + STAGES * C::A_BYTES;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * C::STAGE_BYTES);
  uint64_t *empty = full + STAGES;
  uint64_t *tfull = empty + STAGES;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * C::BM;
  if (K_dev) K = min(K, *K_dev);  // reduction length known only on the device
  const int nk = (K + C::BK - 1) / C::BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES, r = kb / STAGES;
      if (r > 0) mbar_wait(&empty[s], (r - 1) & 1);
      mbar_expect_tx(&full[s], C::STAGE_BYTES);
      const int k0 = kb * C::BK;
      uint8_t *a = sA + s * C::A_BYTES, *b = sB + s * C::B_BYTES;
      if (!A_MN) {
        tma_load_2d(a, &tmA, &full[s], k0, m0);
      } else {
        tma_load_2d(a, &tmA, &full[s], m0, k0);
        tma_load_2d(a + 8192, &tmA, &full[s], m0 + 64, k0);
      }
      if (!B_MN) {
        tma_load_2d(b, &tmB, &full[s], k0, n0);
      } else {
#pragma unroll
        for (int j = 0; j < BN / 64; ++j) tma_load_2d(b + j * 8192, &tmB, &full[s], n0 + 64 * j, k0);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer
    constexpr uint32_t idesc = umma_idesc_bf16(128, BN, A_MN, B_MN);
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES, r = kb / STAGES;
      mbar_wait(&full[s], r & 1);
      tc_fence_after();
      const uint32_t a = smem_u32(sA + s * C::A_BYTES), b = smem_u32(sB + s * C::B_BYTES);
#pragma unroll
      for (int j = 0; j < C::BK / 16; ++j) {
        const uint64_t ad = A_MN ? umma_desc_sw128(a + j * 2048, 8192, 1024)
                                 : umma_desc_sw128(a + j * 32, 16, 1024);
        const uint64_t bd = B_MN ? umma_desc_sw128(b + j * 2048, 8192, 1024)
                                 : umma_desc_sw128(b + j * 32, 16, 1024);
        umma_bf16(tmem, ad, bd, idesc, (kb | j) != 0);
      }
      umma_commit(&empty[s]);
    }
    umma_commit(tfull);
  }

  // ---------------- epilogue: TMEM -> registers -> global
  mbar_wait(tfull, 0);
  __syncwarp();
  tc_fence_after();
  const int m = m0 + warp * 32 + lane;
  const bool row_ok = m < M;
#pragma unroll 1
  for (int c = 0; c < BN / 32; ++c) {
    const int n = n0 + c * 32;
    if (n >= N) break;  // warp-uniform
    float v[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c * 32, v);
    if (nk == 0) {  // empty reduction: the TMEM accumulator was never written
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = 0.f;
    }
    if (!row_ok) continue;
    if (ep.bias_row) {
      const float bv = ep.bias_row[m];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] += bv;
    }
    if (ep.C) {
      float *dst = ep.C + (size_t)m * ep.ldc + n;
      if (n + 32 <= N && (ep.ldc & 3) == 0 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          float4 o = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          if (ep.bias_col) {
            const float4 bb = *reinterpret_cast<const float4 *>(ep.bias_col + n + j);
            o.x += bb.x; o.y += bb.y; o.z += bb.z; o.w += bb.w;
          }
          if (ep.accumulate) {
            const float4 old = *reinterpret_cast<const float4 *>(dst + j);
            o.x += old.x; o.y += old.y; o.z += old.z; o.w += old.w;
          }
          *reinterpret_cast<float4 *>(dst + j) = o;
        }
      } else {
        for (int j = 0; j < 32 && n + j < N; ++j) {
          float o = v[j] + (ep.bias_col ? ep.bias_col[n + j] : 0.f);
          if (ep.accumulate) o += dst[j];
          dst[j] = o;
        }
      }
    }
    if (ep.Cb) {
      __nv_bfloat16 *dst = ep.Cb + (size_t)m * ep.ldcb + n;
      for (int j = 0; j < 32 && n + j < N; ++j)
        dst[j] = __float2bfloat16_rn(v[j] + (ep.bias_col ? ep.bias_col[n + j] : 0.f));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, BN);
}

// ------------------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn g_encode = nullptr;

static bool get_encode() {
  if (g_encode) return true;
  cudaDriverEntryPointQueryResult q;
  void *fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
          cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn)
    return false;
  g_encode = reinterpret_cast<EncodeTiledFn>(fn);
  return true;
}

// 2-D bf16 tensor map: `inner` contiguous elements per row, `outer` rows, row pitch `ld`
// elements, box {64, box_outer}, 128-B swizzle, OOB = zeros.
bool make_tmap_bf16(CUtensorMap *m, const void *ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                    uint32_t box_outer) {
  if (!get_encode()) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {64, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims,
                        strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 3-D view of a row-major bf16 matrix as {64 columns, rows, column chunks}: one TMA op then
// fetches `box_chunks` consecutive 64-column chunks of `box_rows` rows, landing chunk-major in
// shared memory (each chunk = box_rows x 128 B, 128-B swizzled) — the K-major UMMA layout.
// Requires ld >= 64 * n_chunks (the chunk dimension never runs past the row pitch).
bool make_tmap_bf16_chunks(CUtensorMap *m, const void *ptr, uint64_t rows, uint64_t ld,
                           uint64_t n_chunks, uint32_t box_rows, uint32_t box_chunks) {
  if (!get_encode() || ld < 64 * n_chunks) return false;
  cuuint64_t dims[3] = {64, rows, n_chunks};
  cuuint64_t strides[2] = {ld * 2, 128};
  cuuint32_t box[3] = {64, box_rows, box_chunks};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(ptr), dims,
                        strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BN, int A_MN, int B_MN>
static cudaError_t launch(const GemmOp &op, cudaStream_t st) {
  constexpr int STAGES = BN == 256 ? 4 : 5;
  using C = GemmCfg<BN, A_MN, B_MN, STAGES>;
  CUtensorMap ta, tb;
  bool ok = A_MN ? make_tmap_bf16(&ta, op.A, op.M, op.K, op.lda, 64)
                 : make_tmap_bf16(&ta, op.A, op.K, op.M, op.lda, 128);
  ok = ok && (B_MN ? make_tmap_bf16(&tb, op.B, op.N, op.K, op.ldb, 64)
                   : make_tmap_bf16(&tb, op.B, op.K, op.N, op.ldb, BN));
  if (!ok) return cudaErrorInvalidValue;
  auto kern = gemm_bf16_tc_kernel<BN, A_MN, B_MN, STAGES>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((op.N + BN - 1) / BN, (op.M + 127) / 128);
  kern<<<grid, 128, C::SMEM, st>>>(ta, tb, op.ep, op.M, op.N, op.K, op.K_dev);
  return cudaGetLastError();
}

cudaError_t gemm_bf16(const GemmOp &op, cudaStream_t st) {
  if (op.M <= 0 || op.N <= 0) return cudaSuccess;
  if ((op.lda & 7) || (op.ldb & 7) || (reinterpret_cast<uintptr_t>(op.A) & 15) ||
      (reinterpret_cast<uintptr_t>(op.B) & 15))
    return cudaErrorInvalidValue;
  const bool wide = op.N >= 1024;  // BN = 256 for wide outputs (decoder), 128 otherwise
#define JN_G(BN_, AM, BMJ) return launch<BN_, AM, BMJ>(op, st)
  if (wide) {
    if (!op.a_mn && !op.b_mn) JN_G(256, 0, 0);
    if (!op.a_mn && op.b_mn) JN_G(256, 0, 1);
    if (op.a_mn && !op.b_mn) JN_G(256, 1, 0);
    JN_G(256, 1, 1);
  } else {
    if (!op.a_mn && !op.b_mn) JN_G(128, 0, 0);
    if (!op.a_mn && op.b_mn) JN_G(128, 0, 1);
    if (op.a_mn && !op.b_mn) JN_G(128, 1, 0);
    JN_G(128, 1, 1);
  }
#undef JN_G
}

}  // namespace jk
