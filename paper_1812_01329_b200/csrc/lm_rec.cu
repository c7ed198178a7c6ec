// lm_rec.cu — the loop of the Figure 1 program (`for item in sequence: state =
// rnn_cell(state, item)`) executed as ONE persistent launch per layer and direction: the loop
// frame lives on the device — unrolled to the asserted trip count or, in While
// mode, bounded by a trip count computed on the device — with a grid barrier per iteration and no
// host round trip.
//
// Weight-stationary tcgen05 design. CTA j owns hidden units [16j, 16j+16) (all 4 gates):
//   forward : its 64 gate-interleaved rows of W_hh stay in shared memory for all T steps; per step
//             h_{t-1} (bf16, [B x H]) streams in by TMA, D[b, 4u+g] = h_{t-1} . W_slice^T lands in
//             TMEM (M = 128 batch rows, N = 64, K = 16 per MMA), and the cell update runs in the
//             epilogue thread that owns batch row b — c and the fp32 h stay in registers.
//   backward: its 16 columns of W_hh (stored transposed, [units x 4H]) stay in shared memory;
//             per step dz_{t+1} (bf16 [B x 4H]) streams in, D[b, u] = dz_{t+1} . W_hh[:, u] gives the
//             recurrent dh, and the cell backward runs in registers (dc carried in registers).
// Gate-interleaved order: row 4u+g of the working copies = canonical row g*H+u (g = i,f,g,o).
#include "common.cuh"
#include "gemm_tc.h"
#include "lm_rec.h"

namespace jk {

constexpr int REC_THREADS = 128;
constexpr int REC_UPC = 16;     // hidden units per CTA
constexpr int REC_STAGES = 6;   // A-operand ring depth

struct RecSmem {
  // laid out manually from a 1024-aligned base
  static constexpr int A_STAGE = 128 * 128;  // 128 rows x 128 B (MMA reads 128 rows)
};

JN_DEV float tanh_acc(float x) { return tanhf(x); }

// ---------------------------------------------------------------------------------- forward
template <bool MASKED>
__global__ void __launch_bounds__(REC_THREADS, 1)
    lstm_rec_fwd_kernel(const __grid_constant__ CUtensorMap tmH,  // Hs [(T+1)B x H], box {64,B}
                        const __grid_constant__ CUtensorMap tmW,  // W_hh interleaved [4H x H], box {64,64}
                        RecFwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  const int nk = (a.H + 63) / 64;
  uint8_t *sW = base;                                   // nk x 8 KB
  uint8_t *sA = sW + nk * 8192;                         // REC_STAGES x 16 KB
  uint64_t *full = reinterpret_cast<uint64_t *>(sA + REC_STAGES * RecSmem::A_STAGE);
  uint64_t *empty = full + REC_STAGES;
  uint64_t *tfull = empty + REC_STAGES;
  uint64_t *wfull = tfull + 1;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(wfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = threadIdx.x;  // batch row owned in the epilogue
  const int u0 = blockIdx.x * REC_UPC;
  const int B = a.B, H = a.H, G4 = 4 * a.H;
  if (a.fail && *a.fail) return;  // cooperative cancellation: an earlier phase already failed

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmH);
    tma_prefetch_desc(&tmW);
    for (int s = 0; s < REC_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(tfull, 1);
    mbar_init(wfull, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 64);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // resident weight slice: 64 interleaved gate rows x H
  if (threadIdx.x == 0) {
    mbar_expect_tx(wfull, nk * 8192);
    for (int j = 0; j < nk; ++j) tma_load_2d(sW + j * 8192, &tmW, wfull, j * 64, blockIdx.x * 64);
  }

  // initial state -> registers and row block 0 of Hs / Cs (the local copies of P:266)
  float hreg[REC_UPC], creg[REC_UPC];
  const bool row = b < B;
  // `state = self.state` or zeros when it is still None: Switch/Merge on the device
  const bool is_tensor = a.tag == nullptr || *a.tag == 1;
#pragma unroll
  for (int u = 0; u < REC_UPC; ++u) {
    const int gu = u0 + u;
    hreg[u] = (row && gu < H && is_tensor) ? a.h0[(size_t)b * H + gu] : 0.f;
    creg[u] = (row && gu < H && is_tensor) ? a.c0[(size_t)b * H + gu] : 0.f;
    if (row && gu < H) {
      a.Hs[(size_t)b * a.ldh + gu] = __float2bfloat16_rn(hreg[u]);
      a.Cs[(size_t)b * a.ldh + gu] = creg[u];
    }
  }
  const int len_b = (MASKED && row) ? a.lens[b] : 0;
  fence_proxy_async_global();
  unsigned int epoch = 1;
  grid_arrive_wait(a.barrier, epoch * gridDim.x);
  const int T = a.T_dev ? *a.T_dev : a.T;
  constexpr uint32_t idesc = umma_idesc_bf16(128, 64, 0, 0);
  mbar_wait(wfull, 0);

  for (int t = 0; t < T; ++t) {
    if (threadIdx.x == 0) {
      fence_proxy_async_global();
      for (int j = 0; j < nk; ++j) {
        const int q = t * nk + j, s = q % REC_STAGES, r = q / REC_STAGES;
        if (r > 0) mbar_wait(&empty[s], (r - 1) & 1);
        mbar_expect_tx(&full[s], B * 128);
        tma_load_2d(sA + s * RecSmem::A_STAGE, &tmH, &full[s], j * 64, t * B);
      }
    } else if (threadIdx.x == 32) {
      for (int j = 0; j < nk; ++j) {
        const int q = t * nk + j, s = q % REC_STAGES, r = q / REC_STAGES;
        mbar_wait(&full[s], r & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(sA + s * RecSmem::A_STAGE), sw = smem_u32(sW + j * 8192);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_bf16(tmem, umma_desc_sw128(sa + k * 32, 16, 1024),
                    umma_desc_sw128(sw + k * 32, 16, 1024), idesc, (j | k) != 0);
        umma_commit(&empty[s]);
      }
      umma_commit(tfull);
    }
    mbar_wait(tfull, t & 1);
    __syncwarp();
    tc_fence_after();
    float z[64];
    {
      float lo[32], hi[32];
      const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16);
      tmem_ld32(ta, lo);
      tmem_ld32(ta + 32, hi);
#pragma unroll
      for (int i = 0; i < 32; ++i) { z[i] = lo[i]; z[32 + i] = hi[i]; }
    }
    if (row) {
      float *g = a.G + (size_t)(t * B + b) * G4 + (size_t)blockIdx.x * 64;
      const bool valid = !MASKED || t < len_b;
      const int nu = min(REC_UPC, H - u0);
      if (nu == REC_UPC) {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          float4 x = reinterpret_cast<const float4 *>(g)[q];
          z[4 * q] += x.x; z[4 * q + 1] += x.y; z[4 * q + 2] += x.z; z[4 * q + 3] += x.w;
        }
      } else {
        for (int q = 0; q < 4 * nu; ++q) z[q] += g[q];
      }
      __nv_bfloat16 hb[REC_UPC];
#pragma unroll
      for (int u = 0; u < REC_UPC; ++u) {
        const float ig = sigmoidf_(z[4 * u]), fg = sigmoidf_(z[4 * u + 1]);
        const float gg = tanh_acc(z[4 * u + 2]), og = sigmoidf_(z[4 * u + 3]);
        const float c2 = fg * creg[u] + ig * gg;
        const float h2 = og * tanh_acc(c2);
        z[4 * u] = ig; z[4 * u + 1] = fg; z[4 * u + 2] = gg; z[4 * u + 3] = og;
        if (valid) { creg[u] = c2; hreg[u] = h2; }
        hb[u] = __float2bfloat16_rn(hreg[u]);
      }
      // saved activations for the backward pass (in place of the projection)
      if (nu == REC_UPC) {
#pragma unroll
        for (int q = 0; q < 16; ++q)
          reinterpret_cast<float4 *>(g)[q] = make_float4(z[4 * q], z[4 * q + 1], z[4 * q + 2], z[4 * q + 3]);
      } else {
        for (int q = 0; q < 4 * nu; ++q) g[q] = z[q];
      }
      const size_t ro = (size_t)((t + 1) * B + b) * a.ldh + u0;
      for (int u = 0; u < nu; ++u) {
        a.Cs[ro + u] = creg[u];
        a.Hs[ro + u] = hb[u];
      }
    }
    fence_proxy_async_global();
    tc_fence_before();
    ++epoch;
    grid_arrive_wait(a.barrier, epoch * gridDim.x);
    tc_fence_after();
  }
  // final state (committed by the commit phase only if every assumption held)
  if (row) {
    for (int u = 0; u < REC_UPC && u0 + u < H; ++u) {
      a.hT[(size_t)b * H + u0 + u] = hreg[u];
      a.cT[(size_t)b * H + u0 + u] = creg[u];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 64);
}

// ---------------------------------------------------------------------------------- backward
template <bool MASKED>
__global__ void __launch_bounds__(REC_THREADS, 1)
    lstm_rec_bwd_kernel(const __grid_constant__ CUtensorMap tmDZ,  // DZ [T*B x 4H], box {64,B}
                        const __grid_constant__ CUtensorMap tmWT,  // W_hh^T [H x 4H], box {64,16}
                        RecBwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  const int G4 = 4 * a.H;
  const int nk = (G4 + 63) / 64;
  uint8_t *sW = base;                                   // nk x 2 KB (16 rows x 128 B)
  uint8_t *sA = sW + ((nk * 2048 + 1023) & ~1023);      // REC_STAGES x 16 KB
  uint64_t *full = reinterpret_cast<uint64_t *>(sA + REC_STAGES * RecSmem::A_STAGE);
  uint64_t *empty = full + REC_STAGES;
  uint64_t *tfull = empty + REC_STAGES;
  uint64_t *wfull = tfull + 1;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(wfull + 1);

  const int warp = threadIdx.x >> 5;
  const int b = threadIdx.x;
  const int u0 = blockIdx.x * REC_UPC;
  const int B = a.B, H = a.H;
  if (a.fail && *a.fail) return;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmDZ);
    tma_prefetch_desc(&tmWT);
    for (int s = 0; s < REC_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(tfull, 1);
    mbar_init(wfull, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 32);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) {
    mbar_expect_tx(wfull, nk * 2048);
    for (int j = 0; j < nk; ++j) tma_load_2d(sW + j * 2048, &tmWT, wfull, j * 64, u0);
  }
  const int T = a.T_dev ? *a.T_dev : a.T;
  const bool row = b < B;
  const int nu = min(REC_UPC, H - u0);
  // While mode: dz rows of the steps beyond the device trip count must not contribute to wgrads
  if (MASKED && row) {
    for (int t = T; t < a.T; ++t)
      for (int q = 0; q < 4 * nu; ++q)
        a.DZ[(size_t)(t * B + b) * G4 + (size_t)blockIdx.x * 64 + q] = __float2bfloat16_rn(0.f);
  }
  const int len_b = (MASKED && row) ? a.lens[b] : 0;
  float dcreg[REC_UPC], carry[REC_UPC];
#pragma unroll
  for (int u = 0; u < REC_UPC; ++u) { dcreg[u] = 0.f; carry[u] = 0.f; }
  constexpr uint32_t idesc = umma_idesc_bf16(128, 16, 0, 0);
  mbar_wait(wfull, 0);
  unsigned int epoch = 0;
  int q = 0;  // global chunk counter (ring position)

  for (int t = T - 1; t >= 0; --t) {
    const bool has_next = t + 1 < T;  // dz_{t+1} exists
    if (has_next) {
      if (threadIdx.x == 0) {
        fence_proxy_async_global();
        for (int j = 0; j < nk; ++j) {
          const int qq = q + j, s = qq % REC_STAGES, r = qq / REC_STAGES;
          if (r > 0) mbar_wait(&empty[s], (r - 1) & 1);
          mbar_expect_tx(&full[s], B * 128);
          tma_load_2d(sA + s * RecSmem::A_STAGE, &tmDZ, &full[s], j * 64, (t + 1) * B);
        }
      } else if (threadIdx.x == 32) {
        for (int j = 0; j < nk; ++j) {
          const int qq = q + j, s = qq % REC_STAGES, r = qq / REC_STAGES;
          mbar_wait(&full[s], r & 1);
          tc_fence_after();
          const uint32_t sa = smem_u32(sA + s * RecSmem::A_STAGE), sw = smem_u32(sW + j * 2048);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16(tmem, umma_desc_sw128(sa + k * 32, 16, 1024),
                      umma_desc_sw128(sw + k * 32, 16, 1024), idesc, (j | k) != 0);
          umma_commit(&empty[s]);
        }
        umma_commit(tfull);
      }
      q += nk;
    }
    float dh[REC_UPC];
    if (has_next) {
      mbar_wait(tfull, epoch & 1);
      ++epoch;
      __syncwarp();
      tc_fence_after();
      tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16), dh);
    } else {
#pragma unroll
      for (int u = 0; u < REC_UPC; ++u) dh[u] = 0.f;
    }
    if (row) {
      const size_t r = (size_t)(t * B + b);
      const float *din = a.dHin + r * a.ldd + u0;
      const float *g = a.G + r * G4 + (size_t)blockIdx.x * 64;
      const float *ct = a.Cs + (r + B) * a.ldh + u0;
      const float *cp = a.Cs + r * a.ldh + u0;
      __nv_bfloat16 *dz = a.DZ + r * G4 + (size_t)blockIdx.x * 64;
      const bool valid = !MASKED || t < len_b;
      for (int u = 0; u < nu; ++u) {
        const float dhu = dh[u] + din[u] + carry[u];
        const float ig = g[4 * u], fg = g[4 * u + 1], gg = g[4 * u + 2], og = g[4 * u + 3];
        if (valid) {
          const float tc = tanh_acc(ct[u]);
          const float dout = dhu * tc;
          const float dc = dcreg[u] + dhu * og * (1.f - tc * tc);
          const float di = dc * gg, dg = dc * ig, df = dc * cp[u];
          dcreg[u] = dc * fg;
          carry[u] = 0.f;
          dz[4 * u] = __float2bfloat16_rn(di * ig * (1.f - ig));
          dz[4 * u + 1] = __float2bfloat16_rn(df * fg * (1.f - fg));
          dz[4 * u + 2] = __float2bfloat16_rn(dg * (1.f - gg * gg));
          dz[4 * u + 3] = __float2bfloat16_rn(dout * og * (1.f - og));
        } else {
          carry[u] = dhu;  // masked step: (h, c) passed through unchanged
          dz[4 * u] = dz[4 * u + 1] = dz[4 * u + 2] = dz[4 * u + 3] = __float2bfloat16_rn(0.f);
        }
      }
    }
    fence_proxy_async_global();
    tc_fence_before();
    grid_arrive_wait(a.barrier, (unsigned)(T - t) * gridDim.x);
    tc_fence_after();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 32);
}

// ---------------------------------------------------------------------------------- host
static int fwd_smem(int H) { return 1024 + ((H + 63) / 64) * 8192 + REC_STAGES * RecSmem::A_STAGE + 256; }
static int bwd_smem(int H) {
  const int nk = (4 * H + 63) / 64;
  return 1024 + ((nk * 2048 + 1023) & ~1023) + REC_STAGES * RecSmem::A_STAGE + 256;
}

int rec_grid(int H) { return (H + REC_UPC - 1) / REC_UPC; }

static cudaError_t coop_launch(const void *fn, int grid, int smem, void **args, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(REC_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

cudaError_t lstm_rec_fwd(const RecFwdArgs &a, const __nv_bfloat16 *Whh, int ldw, bool masked,
                         cudaStream_t st) {
  if (a.B > 128 || a.B < 1) return cudaErrorInvalidValue;
  CUtensorMap tmH, tmW;
  if (!make_tmap_bf16(&tmH, a.Hs, a.H, (uint64_t)(a.T + 1) * a.B, a.ldh, a.B)) return cudaErrorInvalidValue;
  if (!make_tmap_bf16(&tmW, Whh, a.H, 4ull * a.H, ldw, 64)) return cudaErrorInvalidValue;
  const int smem = fwd_smem(a.H);
  const void *fn = masked ? (const void *)lstm_rec_fwd_kernel<true> : (const void *)lstm_rec_fwd_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  RecFwdArgs aa = a;
  void *args[] = {&tmH, &tmW, &aa};
  return coop_launch(fn, rec_grid(a.H), smem, args, st);
}

cudaError_t lstm_rec_bwd(const RecBwdArgs &a, const __nv_bfloat16 *WhhT, int ldwt, bool masked,
                         cudaStream_t st) {
  if (a.B > 128 || a.B < 1) return cudaErrorInvalidValue;
  CUtensorMap tmDZ, tmWT;
  if (!make_tmap_bf16(&tmDZ, a.DZ, 4ull * a.H, (uint64_t)a.T * a.B, 4ull * a.H, a.B)) return cudaErrorInvalidValue;
  if (!make_tmap_bf16(&tmWT, WhhT, 4ull * a.H, a.H, ldwt, 16)) return cudaErrorInvalidValue;
  const int smem = bwd_smem(a.H);
  const void *fn = masked ? (const void *)lstm_rec_bwd_kernel<true> : (const void *)lstm_rec_bwd_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  RecBwdArgs aa = a;
  void *args[] = {&tmDZ, &tmWT, &aa};
  return coop_launch(fn, rec_grid(a.H), smem, args, st);
}

}  // namespace jk
