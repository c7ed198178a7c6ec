// gemm_tc.cu — tcgen05 / TMEM / TMA bf16 GEMM for the batched cell contractions of the LSTM-LM
// and TreeLSTM steps (the only dense contractions on the path: input projections, decoder,
// dgrad and wgrad GEMMs).
//
//   D[M,N] (fp32) = A[M,K] . B[N,K]^T   (+ bias, + existing D), bf16 operands, fp32 accumulate.
//   Either operand may be K-major (K contiguous) or MN-major (M/N contiguous), so wgrad GEMMs
//   (reduction over the token dimension, dW = dz^T x) read the activations in place.
//
// Persistent, warp-specialised kernel, one CTA per SM (grid <= 148), 6 warps:
//   warp 0 / lane 0 : TMA producer, STAGES-deep smem ring (128-B swizzle), runs across tiles;
//   warp 1 / lane 0 : tcgen05.mma issuer (M=128, N=BN, K=16) into one of TWO TMEM accumulators,
//                     so the epilogue of tile i overlaps the mainloop of tile i+1;
//   warps 2-5       : epilogue, TMEM lanes 32 (w % 4) .. +31 (tcgen05.ld 32x32b) -> fused store.
// Tiles are 128 x BN output blocks, optionally split along K ("splits") when there are too few
// tiles to fill the GPU: each split parks its partial tile in scratch, and the LAST split to
// finish (atomicInc counter, wraps back to 0) adds the partials in split order 0..splits-1 and
// runs the epilogue — deterministic, and no CTA ever waits for another.
// Tile t -> (split = t % splits, m-block fastest), CTA c takes t = c, c + grid, ...
#include <algorithm>
#include <cstring>

#include "common.cuh"
#include "fused_ar.cuh"
#include "gemm_tc.h"

namespace jk {

bool make_tmap_f32_box32(CUtensorMap *m, const void *ptr, uint64_t cols, uint64_t rows, uint64_t ld);

template <int BN, int STAGES, int NMMA = 1, bool PAIR = false>
struct GemmCfg {
  static constexpr int BM = 128, BK = 64;
  static constexpr int A_BYTES = BM * BK * 2;  // 16 KB
  static constexpr int B_BYTES = (PAIR ? BN / 2 : BN) * BK * 2;  // PAIR: this CTA's half of the N rows
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // epilogue staging for TMA stores: per epilogue warp two 32 x 32 fp32 boxes (double buffer)
  static constexpr int EPI_BYTES = 4 * 2 * 32 * 32 * 4;
  static constexpr int SMEM = STAGES * STAGE_BYTES + EPI_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int THREADS = 192 + 32 * (NMMA - 1);  // warp 6: the second MMA warp
  // two accumulators of NMMA x BN columns, allocated as a power of two >= 32 (BN = 192: 512)
  static constexpr int TMEM_NEED = 2 * NMMA * BN;
  static constexpr int TMEM_COLS = TMEM_NEED <= 128 ? 128 : TMEM_NEED <= 256 ? 256 : 512;
};

struct TileMap {
  int Mb, Nb, splits, total;
  JN_DEV void of(int t, int &m_blk, int &n_blk, int &s) const {
    s = t % splits;
    const int mn = t / splits;
    m_blk = mn % Mb;
    n_blk = mn / Mb;
  }
};

// Fused epilogue of 32 consecutive outputs D[m][n .. n+32) of one row (n < N):
// + bias_row[m] + bias_col[n] (+ old C when accumulating), fp32 and / or bf16 stores.
JN_DEV void store_row32(const GemmEpilogue &ep, int m, int n, int N, float (&v)[32], const float *, int) {
  if (ep.bias_row) {
    const float bv = ep.bias_row[m];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] += bv;
  }
  if (ep.C) {
    float *dst = ep.C + (size_t)m * ep.ldc + n;
    if (n + 32 <= N && (ep.ldc & 3) == 0 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
      // every load (bias, old C) is issued before the first store: the stores may alias them in
      // the compiler's view, and interleaving would serialise eight load latencies per call
      float4 add[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) add[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (ep.bias_col) {
        const float4 *b4 = reinterpret_cast<const float4 *>(ep.bias_col + n);
#pragma unroll
        for (int j = 0; j < 8; ++j) add[j] = __ldg(b4 + j);
      }
      if (ep.accumulate) {
        const float4 *o4 = reinterpret_cast<const float4 *>(dst);
        float4 old[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) old[j] = o4[j];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          add[j].x += old[j].x; add[j].y += old[j].y; add[j].z += old[j].z; add[j].w += old[j].w;
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        reinterpret_cast<float4 *>(dst)[j] = make_float4(v[4 * j] + add[j].x, v[4 * j + 1] + add[j].y,
                                                         v[4 * j + 2] + add[j].z, v[4 * j + 3] + add[j].w);
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

// Up to GB_MAX GEMMs with the same operand majors and tile width in one persistent launch
// (grouped): their tiles are concatenated, so small GEMMs fill the machine together.
constexpr int GB_MAX = 8;
struct GemmBatch {
  CUtensorMap ta[GB_MAX], tb[GB_MAX];
  CUtensorMap tc[GB_MAX];        // fp32 D, box {32, 32}, 128-B swizzle (TMA-store epilogue)
  int tma_store[GB_MAX];         // 1: epilogue through tc (fp32 D only, no bf16 copy)
  int split_add[GB_MAX];         // 1: the K splits reduce-add into C (GemmOp::split_add)
  int amn[GB_MAX], bmn[GB_MAX];  // operand majors per GEMM (runtime: one kernel serves all four)
  GemmEpilogue ep[GB_MAX];
  int M[GB_MAX], N[GB_MAX], K[GB_MAX];
  const int *K_dev[GB_MAX];
  TileMap tm[GB_MAX];
  unsigned *counters[GB_MAX];
  float *partials[GB_MAX];
  int tile_start[GB_MAX + 1];
  int n;
};

struct TileRef {
  int g, mb, nb, sp, kb0, kb1, tile;
};

// t: cluster-tile index; with CM > 1 the CM CTAs of a cluster take m-blocks CM * mg + rank of the
// same n-block and K range (they share the B tile through TMA multicast); tm.Mb counts m-groups
template <int BN, int STAGES, int CM = 1>
JN_DEV TileRef tile_ref(const GemmBatch &gb, int t, int rank = 0) {
  TileRef r;
  r.g = 0;
  while (r.g + 1 < gb.n && t >= gb.tile_start[r.g + 1]) ++r.g;
  const TileMap &tm = gb.tm[r.g];
  tm.of(t - gb.tile_start[r.g], r.mb, r.nb, r.sp);
  if (CM > 1) r.mb = r.mb * CM + rank;
  int K = gb.K[r.g];
  if (gb.K_dev[r.g]) K = min(K, *gb.K_dev[r.g]);  // reduction length known only on the device
  const int nk = (K + 63) / 64;
  r.kb0 = (int)((long long)nk * r.sp / tm.splits);
  r.kb1 = (int)((long long)nk * (r.sp + 1) / tm.splits);
  r.tile = r.mb + tm.Mb * CM * r.nb;
  return r;
}

// NMMA = 2 (BN = 128): a second MMA-issuing warp takes the odd ring stages into its own
// accumulators — one warp issues a tcgen05.mma only every ~130 cycles, twice the N = 128 MMA time;
// STAGES is even, so every stage has one fixed owner and no wait can alias a phase
// PAIR (CM == 2, NMMA == 1): the cluster's two CTAs run ONE M = 256 MMA (cta_group::2) per
// k-step: each holds its 128 rows of A and half of the B tile's N rows (32 KB per stage instead of
// 48 KB at BN = 256: six stages in flight), both CTAs' TMA loads complete on the leader's full
// barrier, the leader issues the MMAs and its commits arrive on both CTAs' barriers; each CTA's
// epilogue reads its own 128 accumulator rows and releases the leader's TMEM-empty barrier.
template <int BN, int STAGES, int NMMA, int CM, bool PAIR>
__global__ void __launch_bounds__(192 + 32 * (NMMA - 1), 1) gemm_bf16_tc_kernel(const __grid_constant__ GemmBatch gb) {
  pdl_enter();
  using C = GemmCfg<BN, STAGES, NMMA, PAIR>;
  static_assert(STAGES % NMMA == 0, "stage ownership");
  static_assert(!PAIR || (CM == 2 && NMMA == 1), "CTA pair");
  // CM > 1: clusters of CM CTAs along M share each B tile; CTA r loads rows / k-rows slice r of it
  // with a multicast TMA into every cluster CTA, and a stage is released only when the owning
  // MMA warp of EVERY cluster CTA consumed it (multicast commit into each empty barrier)
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  uint8_t *sA = smem;
  uint8_t *sB = smem + STAGES * C::A_BYTES;
  uint8_t *epi_stage = smem + STAGES * C::STAGE_BYTES;  // [4 warps][2][32 rows][128 B], swizzled
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * C::STAGE_BYTES + C::EPI_BYTES);
  uint64_t *empty = full + STAGES;
  uint64_t *tfull = empty + STAGES;  // [2]
  uint64_t *tempty = tfull + 2;      // [2]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int total = gb.tile_start[gb.n];
  const int rank = CM > 1 ? (int)cluster_ctarank() : 0;
  const int cid = blockIdx.x / CM, ncl = gridDim.x / CM;  // cluster index / count
  constexpr uint16_t cmask = (uint16_t)((1u << CM) - 1);

  if (warp == 0 && lane == 0) {
    for (int g = 0; g < gb.n; ++g) {
      tma_prefetch_desc(&gb.ta[g]);
      tma_prefetch_desc(&gb.tb[g]);
      if (gb.tma_store[g]) tma_prefetch_desc(&gb.tc[g]);
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], PAIR ? 1 : CM);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], NMMA);
      mbar_init(&tempty[i], PAIR ? 8 : 4);  // PAIR: both CTAs' epilogue warps release the leader's
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    if (PAIR) tmem_alloc_pair(tmem_slot, C::TMEM_COLS);
    else tmem_alloc(tmem_slot, C::TMEM_COLS);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (CM > 1) cluster_sync_all();  // peers' barriers exist before any multicast targets them
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {  // ---------------- TMA producer (the warp loops together, lane 0 issues)
    int q = 0;       // ring position, continuous across tiles
    for (int t = cid; t < total; t += ncl) {
      const TileRef tr = tile_ref<BN, STAGES, CM>(gb, t, rank);
      const CUtensorMap *tmA = &gb.ta[tr.g], *tmB = &gb.tb[tr.g];
      const bool A_MN = gb.amn[tr.g], B_MN = gb.bmn[tr.g];
      const int m0 = tr.mb * C::BM, n0 = tr.nb * BN;
      for (int kb = tr.kb0; kb < tr.kb1; ++kb, ++q) {
        const int s = q % STAGES, r = q / STAGES;
        if (PAIR && lane == 0) {
          if (r > 0) mbar_wait(&empty[s], (r - 1) & 1);
          if (rank == 0) mbar_expect_tx(&full[s], 2 * C::STAGE_BYTES);  // both CTAs' loads
          const uint32_t fbar = mapa_shared(smem_u32(&full[s]), 0);      // the leader's barrier
          const int k0 = kb * C::BK;
          uint8_t *a = sA + s * C::A_BYTES, *b = sB + s * C::B_BYTES;
          if (!A_MN) {
            tma_load_2d_pair(a, tmA, fbar, k0, m0);
          } else {
            tma_load_2d_pair(a, tmA, fbar, m0, k0);
            tma_load_2d_pair(a + 8192, tmA, fbar, m0 + 64, k0);
          }
          const int nh = n0 + rank * (BN / 2);  // my half of the tile's N rows
          if (!B_MN) {
            tma_load_2d_pair(b, tmB, fbar, k0, nh);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 128; ++j) tma_load_2d_pair(b + j * 8192, tmB, fbar, nh + 64 * j, k0);
          }
        } else if (lane == 0) {
          if (r > 0) mbar_wait(&empty[s], (r - 1) & 1);
          mbar_expect_tx(&full[s], C::STAGE_BYTES);
          const int k0 = kb * C::BK;
          uint8_t *a = sA + s * C::A_BYTES, *b = sB + s * C::B_BYTES;
          if (!A_MN) {
            tma_load_2d(a, tmA, &full[s], k0, m0);
          } else {
            tma_load_2d(a, tmA, &full[s], m0, k0);
            tma_load_2d(a + 8192, tmA, &full[s], m0 + 64, k0);
          }
          if (CM == 1) {
            if (!B_MN) {
              tma_load_2d(b, tmB, &full[s], k0, n0);
            } else {
#pragma unroll
              for (int j = 0; j < BN / 64; ++j) tma_load_2d(b + j * 8192, tmB, &full[s], n0 + 64 * j, k0);
            }
          } else if (!B_MN) {  // my slice of N rows, multicast to the cluster
            constexpr int RS = BN / CM;
            tma_load_2d_mc(b + rank * RS * 128, tmB, &full[s], k0, n0 + rank * RS, cmask);
          } else {  // my slice of the K rows of every 64-column chunk, multicast
            constexpr int KS = 64 / CM;
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_2d_mc(b + j * 8192 + rank * KS * 128, tmB, &full[s], n0 + 64 * j, k0 + rank * KS, cmask);
          }
        }
        __syncwarp();
      }
    }
  } else if (PAIR && warp == 1) {  // ---------------- the pair's MMA issuer (leader, lane 0)
    int q = 0, i = 0;
    if (rank == 0)
      for (int t = cid; t < total; t += ncl, ++i) {
        const TileRef tr = tile_ref<BN, STAGES, CM>(gb, t, rank);
        const int A_MN = gb.amn[tr.g], B_MN = gb.bmn[tr.g];
        const uint32_t idesc = umma_idesc_bf16(256, BN, A_MN, B_MN);
        const int buf = i & 1;
        if (i >= 2) mbar_wait(&tempty[buf], ((i >> 1) - 1) & 1);  // both CTAs drained this buffer
        tc_fence_after();
        const uint32_t acc = tmem + (uint32_t)(buf * BN);
        bool first = true;
        for (int kb = tr.kb0; kb < tr.kb1; ++kb, ++q) {
          const int s = q % STAGES, r = q / STAGES;
          mbar_wait(&full[s], r & 1);
          tc_fence_after();
          if (elect_one_sync()) {
            const uint32_t a = smem_u32(sA + s * C::A_BYTES), b = smem_u32(sB + s * C::B_BYTES);
            static_assert(C::BK == 64, "one umma_bf16_pair_k64 per k-block");
            umma_bf16_pair_k64(acc, A_MN ? umma_desc_sw128(a, 8192, 1024) : umma_desc_sw128(a, 16, 1024),
                               B_MN ? umma_desc_sw128(b, 8192, 1024) : umma_desc_sw128(b, 16, 1024), idesc,
                               first ? 0u : 1u, A_MN ? 128 : 2, B_MN ? 128 : 2);
            umma_commit_pair(&empty[s]);
          }
          first = false;
          __syncwarp();
        }
        if (lane == 0) umma_commit_pair(&tfull[buf]);  // arrives even without a k-block
        __syncwarp();
      }
  } else if (warp == 1 || warp >= 6) {  // ---------------- MMA issuers (lane 0 issues)
    const int mw = warp == 1 ? 0 : warp - 5;  // which of the NMMA issuing warps
    int q = 0, i = 0;
    for (int t = cid; t < total; t += ncl, ++i) {
      const TileRef tr = tile_ref<BN, STAGES, CM>(gb, t, rank);
      const int A_MN = gb.amn[tr.g], B_MN = gb.bmn[tr.g];
      const uint32_t idesc = umma_idesc_bf16(128, BN, A_MN, B_MN);
      const int buf = i & 1;
      if (i >= 2) mbar_wait(&tempty[buf], ((i >> 1) - 1) & 1);  // epilogue drained this buffer
      tc_fence_after();
      const uint32_t acc = tmem + (uint32_t)((buf * NMMA + mw) * BN);
      bool first = true;
      for (int kb = tr.kb0; kb < tr.kb1; ++kb, ++q) {
        if (q % NMMA != mw) continue;
        const int s = q % STAGES, r = q / STAGES;
        mbar_wait(&full[s], r & 1);
        tc_fence_after();
        if (elect_one_sync()) {
          const uint32_t a = smem_u32(sA + s * C::A_BYTES), b = smem_u32(sB + s * C::B_BYTES);
          static_assert(C::BK == 64, "one umma_bf16_k64 per k-block");
          umma_bf16_k64(acc, A_MN ? umma_desc_sw128(a, 8192, 1024) : umma_desc_sw128(a, 16, 1024),
                        B_MN ? umma_desc_sw128(b, 8192, 1024) : umma_desc_sw128(b, 16, 1024), idesc,
                        first ? 0u : 1u, A_MN ? 128 : 2, B_MN ? 128 : 2);
          if (CM == 1) umma_commit(&empty[s]);
          else umma_commit_mc(&empty[s], cmask);
        }
        first = false;
        __syncwarp();
      }
      if (lane == 0) umma_commit(&tfull[buf]);  // arrives even without a k-block of its own
      __syncwarp();
    }
  } else {
    // ---------------- epilogue: TMEM -> registers -> global (warps 2-5)
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    int i = 0, qe = 0;          // qe: ring position of the tile's first k-block (as the MMA warps)
    // this warp is done reading accumulator buffer `buf` (PAIR: on the leader's barrier)
    auto release_tmem = [&](int buf) {
      if (PAIR) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[buf]), 0));
      else mbar_arrive(&tempty[buf]);
    };
    for (int t = cid; t < total; t += ncl, ++i) {
      const TileRef tr = tile_ref<BN, STAGES, CM>(gb, t, rank);
      const int nkt = tr.kb1 > tr.kb0 ? tr.kb1 - tr.kb0 : 0;
      const int qt = qe;
      qe += nkt;
      // accumulator columns of chunk c: the owners of the tile's first min(NMMA, nkt) k-blocks
      auto ld_acc = [&](int c, float (&v)[32]) {
        const uint32_t base = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(((i & 1) * NMMA) * BN) + c * 32;
        tmem_ld32(base + (uint32_t)((qt % NMMA) * BN), v);
        if (NMMA > 1 && nkt > 1) {
          float w[32];
          tmem_ld32(base + (uint32_t)(((qt + 1) % NMMA) * BN), w);
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] += w[j];
        }
      };
      // Pipelined accumulator reads: chunk c + 1's TMEM loads are in flight while chunk c is
      // stored (a tcgen05.ld + wait per chunk serialised eight TMEM round trips per tile and made
      // the epilogue, not the MMAs, the bound of the short-K GEMMs)
      uint32_t pf[NMMA][32];
      auto acc_issue = [&](int c) {
        const uint32_t base = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(((i & 1) * NMMA) * BN) + c * 32;
        tmem_ld32_nw(base + (uint32_t)((qt % NMMA) * BN), pf[0]);
        if (NMMA > 1 && nkt > 1) tmem_ld32_nw(base + (uint32_t)(((qt + 1) % NMMA) * BN), pf[NMMA - 1]);
      };
      auto acc_take = [&](float (&v)[32]) {
        tmem_ld_wait();
        tmem_pin(pf[0]);
        if (NMMA > 1) tmem_pin(pf[NMMA - 1]);
#pragma unroll
        for (int j = 0; j < 32; ++j)
          v[j] = __uint_as_float(pf[0][j]) + (NMMA > 1 && nkt > 1 ? __uint_as_float(pf[NMMA - 1][j]) : 0.f);
      };
      const GemmEpilogue &ep = gb.ep[tr.g];
      const int M = gb.M[tr.g], N = gb.N[tr.g];
      const int splits = gb.tm[tr.g].splits;
      const int m0 = tr.mb * C::BM, n0 = tr.nb * BN;
      const bool empty_k = tr.kb1 <= tr.kb0;  // no MMA wrote the accumulator
      const int buf = i & 1;
      mbar_wait(&tfull[buf], (i >> 1) & 1);
      __syncwarp();
      tc_fence_after();
      const int m = m0 + quad * 32 + lane;
      const bool row_ok = m < M;
      const bool sadd = gb.split_add[tr.g] != 0;
      if ((splits == 1 || sadd) && gb.tma_store[tr.g]) {
        // TMA-store epilogue: each 32 x 32 block of this warp's rows goes registers -> swizzled
        // smem box -> one bulk tensor store (or reduce-add when accumulating), asynchronously;
        // two boxes per warp alternate (wait_group.read 1 before a box is rewritten)
        uint8_t *stg0 = epi_stage + (size_t)(warp - 2) * 2 * 4096;
        const int mrow0 = m0 + quad * 32;
        const float bv = (ep.bias_row && row_ok) ? ep.bias_row[m] : 0.f;
        const int nch = min(BN / 32, (N - n0 + 31) / 32);  // chunks inside N (warp-uniform)
        // one 32-column chunk: bias, swizzled staging box, bulk tensor store
        // column bias: lane l holds bias[n + l] of a chunk, loaded one chunk ahead (its L2 latency
        // was the epilogue's critical path: measured, the FADDs waiting on it were the top stall),
        // and is broadcast with shuffles
        const bool add_bias = ep.bias_col && (!sadd || tr.sp == 0);  // split_add: split 0 adds it
        auto bias_of = [&](int c) {
          const int n = n0 + c * 32 + lane;
          return (add_bias && c < nch && n < N) ? __ldg(ep.bias_col + n) : 0.f;
        };
        float bnext = bias_of(0);
        auto store_chunk = [&](int c, float (&v)[32]) {
          const int n = n0 + c * 32;
          if (empty_k) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = 0.f;
          }
          const float bcur = bnext;
          bnext = bias_of(c + 1);
          if (add_bias) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += __shfl_sync(0xffffffffu, bcur, j);
          }
          if (ep.bias_row && (!sadd || tr.sp == 0)) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += bv;
          }
          uint8_t *stg = stg0 + (c & 1) * 4096;
          if (lane == 0 && c >= 2) bulk_wait_group_read1();  // this box's previous store has read it
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j)  // row `lane`, 16-B granule j at its 128-B-swizzled slot
            *reinterpret_cast<float4 *>(stg + lane * 128 + ((j ^ (lane & 7)) << 4)) =
                make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          fence_proxy_async_shared();
          __syncwarp();
          if (lane == 0) {
            if (ep.accumulate || sadd) tma_reduce_add_2d(&gb.tc[tr.g], stg, n, mrow0);
            else tma_store_2d(&gb.tc[tr.g], stg, n, mrow0);
            bulk_commit_group();
          }
        };
        if constexpr (NMMA == 1) {
          // 64 accumulator columns per tcgen05.ld (x64): measured, eight x32 loads per tile and
          // warp cost the decoder GEMM 13 us over the MMAs alone, four x64 loads nothing
          uint32_t pf64[64];
          const uint32_t abase = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)((i & 1) * BN);
          const int ngp = (nch + 1) / 2;
          if (ngp > 0) tmem_ld64_nw(abase, pf64);
#pragma unroll 1
          for (int p = 0; p < ngp; ++p) {
            float v0[32], v1[32];
            tmem_ld_wait();
            tmem_pin(pf64);
#pragma unroll
            for (int j = 0; j < 32; ++j) { v0[j] = __uint_as_float(pf64[j]); v1[j] = __uint_as_float(pf64[32 + j]); }
            if (p + 1 < ngp) tmem_ld64_nw(abase + (uint32_t)((p + 1) * 64), pf64);
            store_chunk(2 * p, v0);
            if (2 * p + 1 < nch) store_chunk(2 * p + 1, v1);
          }
        } else {
          if (nch > 0) acc_issue(0);
#pragma unroll 1
          for (int c = 0; c < nch; ++c) {
            float v[32];
            acc_take(v);
            if (c + 1 < nch) acc_issue(c + 1);
            store_chunk(c, v);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) release_tmem(buf);
        if (ep.fr.win) {
          // fused cross-rank reduction (NEXT-3): the tile's stores must have COMPLETED (not only
          // read their boxes) before the owner may read it; then the per-tile protocol
          if (lane == 0) {
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            fence_proxy_async_global();  // the tile's TMA (async-proxy) writes -> generic loads
          }
          __syncwarp();
          fr_tile(ep.fr, tr.tile, m0, n0, BN, M, N, ep.ldc, quad * 32 + lane);
        } else {
          if (lane == 0) bulk_wait_group_read0();  // both boxes free before the next tile
          __syncwarp();
        }
      } else if (splits == 1 && !ep.C && !ep.Cb && ep.dev_x64) {
        // dev experiment: drain with 64-column loads
        const uint32_t base = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(((i & 1) * NMMA) * BN);
        for (int c = 0; c < BN / 64; ++c) {
          uint32_t r[64];
          tmem_ld64_nw(base + c * 64, r);
          tmem_ld_wait();
          tmem_pin(r);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) release_tmem(buf);
      } else if (splits == 1) {
        const int nch = ep.dev_no_drain ? 0 : min(BN / 32, (N - n0 + 31) / 32);
        if (nch > 0) acc_issue(0);
#pragma unroll 1
        for (int c = 0; c < nch; ++c) {
          const int n = n0 + c * 32;
          float v[32];
          acc_take(v);
          if (c + 1 < nch) acc_issue(c + 1);
          if (empty_k) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = 0.f;
          }
          if (row_ok) store_row32(ep, m, n, N, v, nullptr, 0);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) release_tmem(buf);
      } else {
        // split-K: park this split's partial tile; the last split to arrive adds the splits in
        // order 0 .. splits-1 (deterministic) and runs the epilogue
        float *partials = gb.partials[tr.g];
        float *pt = partials + ((size_t)tr.tile * splits + tr.sp) * (128 * BN);
        const int rl = quad * 32 + lane;  // tile-local row
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          float v[32];
          ld_acc(c, v);
          if (empty_k) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = 0.f;
          }
          float4 *d4 = reinterpret_cast<float4 *>(pt + (size_t)rl * BN + c * 32);
#pragma unroll
          for (int j = 0; j < 8; ++j) d4[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) release_tmem(buf);
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        __shared__ unsigned s_last;
        if (warp == 2 && lane == 0)
          s_last = atomicInc(&gb.counters[tr.g][tr.tile], (unsigned)splits - 1) == (unsigned)splits - 1;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (s_last) {
          __threadfence();
          const float *p0 = partials + (size_t)tr.tile * splits * (128 * BN) + (size_t)rl * BN;
#pragma unroll 1
          for (int c = 0; c < BN / 32; ++c) {
            const int n = n0 + c * 32;
            if (n >= N) break;
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = 0.f;
            for (int qq = 0; qq < splits; ++qq) {
              const float4 *s4 = reinterpret_cast<const float4 *>(p0 + (size_t)qq * (128 * BN) + c * 32);
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float4 x = __ldcg(s4 + j);
                v[4 * j] += x.x; v[4 * j + 1] += x.y; v[4 * j + 2] += x.z; v[4 * j + 3] += x.w;
              }
            }
            if (row_ok) store_row32(ep, m, n, N, v, nullptr, 0);
          }
        }
      }
    }
  }
  if (warp >= 2 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores done
  tc_fence_before();
  __syncthreads();
  if (CM > 1) cluster_sync_all();  // no CTA leaves while peers may still signal its barriers
  if (warp == 1) {
    if (PAIR) tmem_dealloc_pair(tmem, C::TMEM_COLS);
    else tmem_dealloc(tmem, C::TMEM_COLS);
  }
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

// 2-D fp32 tensor map for the TMA-store epilogue: box {32 columns, 32 rows}, 128-B swizzle
// (a 32-float row is exactly one 128-B swizzle row). Out-of-bounds box parts are not written.
bool make_tmap_f32_box32(CUtensorMap *m, const void *ptr, uint64_t cols, uint64_t rows, uint64_t ld) {
  if (!get_encode()) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(ptr), dims, strides, box,
                        es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
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

static int g_num_sms = 0;
static bool g_tma_store_ok = getenv("JANUS_GEMM_TMA_STORE") == nullptr || getenv("JANUS_GEMM_TMA_STORE")[0] != '0';

// K splits: the fewest persistent rounds per unit of work, each split >= 4 k-blocks, and the
// partial tiles must fit the caller's scratch
static int choose_splits(int tiles, int nk, int nsm, size_t cap_tiles) {
  // Automatic split-K is off: the last-arriver reduction of the partial tiles measured slower
  // than the unsplit GEMM for every shape of the step (scripts/gemm_check.py); explicit
  // GemmOp::splits still selects it (tests/test_gpu_gemm.py::test_gemm_splitk*).
  if (getenv("JANUS_GEMM_AUTOSPLIT") == nullptr) return 1;
  if (tiles >= nsm || nk < 64) return 1;
  int best = 1;
  double best_cost = (double)((tiles + nsm - 1) / nsm);
  for (int s = 2; s <= 8 && nk / s >= 4 && (size_t)tiles * s <= cap_tiles; ++s) {
    const double cost = (double)((tiles * s + nsm - 1) / nsm) / s + 0.08 * s;  // + partial traffic
    if (cost < best_cost - 1e-9) { best_cost = cost; best = s; }
  }
  return best;
}

// may this op run split-K (single launch with scratch, explicit or automatic splits)?
static bool op_wants_split(const GemmOp &op) {
  if (op.split_add) return false;  // no scratch: the split rides the normal (clustered) kernel
  return op.flags && op.partials && (op.splits > 1 || (op.splits <= 0 && getenv("JANUS_GEMM_AUTOSPLIT")));
}

template <int BN, int CM, bool PAIR = false>
static cudaError_t launch_cm(const GemmOp *ops, int n, cudaStream_t st) {
  // PAIR halves a CTA's B stage: six (BN = 256) / eight (BN = 128) stages fit instead of 4 / 6
  // (BN = 192, for launches whose tile count 256-wide tiles would round badly onto 148 SMs:
  // 40 KB stages, four of them)
  constexpr int STAGES = PAIR ? (BN == 256 ? 6 : 8) : (BN == 256 ? 4 : BN == 192 ? 4 : 6);
  constexpr int NMMA = PAIR ? 1 : (BN == 128 ? 2 : 1);
  using C = GemmCfg<BN, STAGES, NMMA, PAIR>;
  auto kern = gemm_bf16_tc_kernel<BN, STAGES, NMMA, CM, PAIR>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  GemmBatch gb;  // ~1.5 KB of kernel parameters (copied at launch)
  memset(&gb, 0, sizeof(gb));
  gb.n = n;
  int total = 0;
  for (int g = 0; g < n; ++g) {
    const GemmOp &op = ops[g];
    bool ok = op.a_mn ? make_tmap_bf16(&gb.ta[g], op.A, op.M, op.K, op.lda, 64)
                      : make_tmap_bf16(&gb.ta[g], op.A, op.K, op.M, op.lda, 128);
    // B boxes: multicast (CM > 1) loads 1/CM of the tile into every CTA; PAIR loads this CTA's
    // half of the N rows (all K rows of each 64-column chunk when MN-major)
    ok = ok && (op.b_mn ? make_tmap_bf16(&gb.tb[g], op.B, op.N, op.K, op.ldb, PAIR ? 64 : 64 / CM)
                        : make_tmap_bf16(&gb.tb[g], op.B, op.K, op.N, op.ldb, BN / CM));
    gb.amn[g] = op.a_mn ? 1 : 0;
    gb.bmn[g] = op.b_mn ? 1 : 0;
    if (!ok) return cudaErrorInvalidValue;
    gb.tma_store[g] = 0;
    if (op.ep.C && !op.ep.Cb && (op.ep.ldc & 3) == 0 && (reinterpret_cast<uintptr_t>(op.ep.C) & 15) == 0 &&
        g_tma_store_ok)
      gb.tma_store[g] = make_tmap_f32_box32(&gb.tc[g], op.ep.C, op.N, op.M, op.ep.ldc) ? 1 : 0;
    // dev measurement knob: "1" drains the accumulators and stores nothing, "2" does not even
    // read them (the mainloop bound)
    static const int epi_skip = getenv("JANUS_GEMM_EPI_SKIP") ? atoi(getenv("JANUS_GEMM_EPI_SKIP")) : 0;
    if (epi_skip) {
      gb.tma_store[g] = 0;
      gb.ep[g] = GemmEpilogue{};
      gb.ep[g].dev_no_drain = epi_skip == 2;
      gb.ep[g].dev_x64 = epi_skip == 3;
    }
    TileMap &tm = gb.tm[g];
    tm.Mb = ((op.M + 127) / 128 + CM - 1) / CM;  // m-groups of CM blocks (ghost blocks: OOB)
    tm.Nb = (op.N + BN - 1) / BN;
    const int nk = (op.K + 63) / 64;
    const size_t cap_tiles = op.partials ? op.partials_cap / (128 * BN) : 0;
    int splits = 1;
    if (op.ep.fr.win && !gb.tma_store[g]) return cudaErrorInvalidValue;  // fused reduction: TMA-store path
    gb.split_add[g] = 0;
    if (op.split_add && op.splits == 2 && gb.tma_store[g] && !op.ep.accumulate && !op.ep.fr.win) {
      splits = 2;  // K halves reduce-added into the zeroed C
      gb.split_add[g] = 1;
    } else
    // split-K only for single launches (own scratch); with clusters (multicast / CTA pairs) only
    // when asked for explicitly: both CTAs of a cluster take the same split of K
    if (n == 1 && op.flags && op.partials && !op.ep.fr.win && (CM == 1 || op.splits > 1)) {
      splits = op.splits > 0 ? op.splits : choose_splits(tm.Mb * tm.Nb, nk, g_num_sms, cap_tiles);
      splits = std::max(1, std::min(splits, 64));
      if ((size_t)tm.Mb * CM * tm.Nb * splits > cap_tiles) splits = 1;  // tile ids span Mb * CM rows
    }
    tm.splits = splits;
    tm.total = tm.Mb * tm.Nb * splits;
    if (!epi_skip) gb.ep[g] = op.ep;
    gb.M[g] = op.M; gb.N[g] = op.N; gb.K[g] = op.K;
    gb.K_dev[g] = op.K_dev;
    gb.counters[g] = op.flags;
    gb.partials[g] = op.partials;
    gb.tile_start[g] = total;
    total += tm.total;
  }
  gb.tile_start[n] = total;
  if (total == 0) return cudaSuccess;
  if (CM == 1) {
    const int grid = std::min(total, g_num_sms);
    return launch_pdl(kern, dim3(grid), dim3(C::THREADS), C::SMEM, st, gb);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(std::min(total, g_num_sms / CM) * CM);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CM;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // see pdl_enter (common.cuh)
  at[1].val.programmaticStreamSerializationAllowed = pdl_on() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, gb);
}

// Clusters of two CTAs along M share the B tile (multicast TMA): the tensor pipe of these
// GEMMs is fed at L2 -> smem rates, and halving B's share of that traffic is the lever.
// JANUS_GEMM_CM=1 disables it.
static int g_gemm_cm = getenv("JANUS_GEMM_CM") ? atoi(getenv("JANUS_GEMM_CM")) : 2;

// CTA pairs (cta_group::2) for launches whose reductions are long (every K >= 1024: the weight
// gradients K = T*B, dh_top K = V): measured at C2, wgrad 81.6 -> 72.8 us, dh 60.4 -> 58.9 us,
// while the short-K (650) decoder and input projection are a little slower paired (57.8 -> 59.7
// us). JANUS_GEMM_PAIR (dev knob): "1" pairs for every launch, "0" never.
static int g_gemm_pair = getenv("JANUS_GEMM_PAIR") ? atoi(getenv("JANUS_GEMM_PAIR")) : -1;
static bool want_pair(const GemmOp *ops, int n) {
  if (g_gemm_pair >= 0) return g_gemm_pair == 1;
  for (int g = 0; g < n; ++g)
    if (ops[g].K < 1024 || ops[g].M <= 128) return false;  // (one 128-row block: a pair would idle half)
  return true;
}

template <int BN>
static cudaError_t launch(const GemmOp *ops, int n, cudaStream_t st) {
  static_assert(BN == 128 || BN == 192 || BN == 256, "tile width");
  bool split = false;
  for (int g = 0; g < n; ++g) split = split || (op_wants_split(ops[g]) && n == 1);
  // an explicit split of a long-K single launch keeps the CTA pair (same split on both CTAs)
  const bool pair_split = split && n == 1 && ops[0].splits > 1 && want_pair(ops, n);
  if constexpr (BN != 192) {  // CTA pairs split B's N rows in 64-row halves: BN = 128 / 256
    if (g_gemm_cm == 2 && pair_split) return launch_cm<BN, 2, true>(ops, n, st);
    if (g_gemm_cm == 2 && !split && want_pair(ops, n)) return launch_cm<BN, 2, true>(ops, n, st);
  }
  if (g_gemm_cm == 2 && !split) return launch_cm<BN, 2>(ops, n, st);
  return launch_cm<BN, 1>(ops, n, st);
}

static cudaError_t check_op(const GemmOp &op) {
  if ((op.lda & 7) || (op.ldb & 7) || (reinterpret_cast<uintptr_t>(op.A) & 15) ||
      (reinterpret_cast<uintptr_t>(op.B) & 15))
    return cudaErrorInvalidValue;
  return cudaSuccess;
}

// Tile width: one tcgen05.mma issue costs ~130 cycles whatever N is (scripts/bench_mma.cu), so
// BN = 256 tiles keep the tensor pipe busiest — as long as the launch still has enough tiles to
// occupy the SMs (else BN = 128 for twice the tiles). Decided per launch (grouped GEMMs together).
static bool wide_of(const GemmOp &op) { return op.N > 128; }
static bool use_bn256(const GemmOp *ops, int n);
void gemm_group_tiling(const GemmOp *ops, int n, int *bn, int *mblocks, int *nblocks) {
  const int BN = use_bn256(ops, n) ? 256 : 128;
  bool split = false;
  for (int g = 0; g < n; ++g) split = split || (op_wants_split(ops[g]) && n == 1);
  const int CM = (g_gemm_cm == 2 && !split) ? 2 : 1;
  *bn = BN;
  for (int g = 0; g < n; ++g) {
    mblocks[g] = (((ops[g].M + 127) / 128 + CM - 1) / CM) * CM;
    nblocks[g] = (ops[g].N + BN - 1) / BN;
  }
}
static bool use_bn256(const GemmOp *ops, int n) {
  long tiles = 0;
  for (int i = 0; i < n; ++i) {
    if (!wide_of(ops[i])) return false;
    tiles += (long)((ops[i].M + 127) / 128) * ((ops[i].N + 255) / 256);
  }
  return tiles >= 100;
}

cudaError_t gemm_bf16_group(const GemmOp *ops, int n, cudaStream_t st) {
  GemmOp live[GB_MAX];
  int m = 0;
  for (int i = 0; i < n; ++i) {
    if (ops[i].M <= 0 || ops[i].N <= 0) continue;
    const cudaError_t e = check_op(ops[i]);
    if (e != cudaSuccess) return e;
    live[m++] = ops[i];
  }
  if (m == 0) return cudaSuccess;
  if (m > GB_MAX) return cudaErrorInvalidValue;
  // one launch for the whole group (the operand majors are per-GEMM runtime properties)
  static const int bn_env = getenv("JANUS_GEMM_BN") ? atoi(getenv("JANUS_GEMM_BN")) : 0;  // dev knob
  int bn = m == 1 ? (bn_env ? bn_env : live[0].bn) : 0;
  if (m == 1 && bn == 0 && wide_of(live[0])) {
    // a single launch takes the tile width with the least work per SM: rounds of tiles over the
    // SMs x tile width (ties to the wider tile). The 2240 x 2600 input projection: 256-wide
    // tiles are 198 = 1.34 rounds, 192-wide 252 = 1.7 rounds
    const int mb = (live[0].M + 127) / 128;
    long best = -1;
    for (int w : {256, 192, 128}) {
      const long tiles = (long)mb * ((live[0].N + w - 1) / w);
      const long cost = (tiles + 147) / 148 * w;
      if (best < 0 || cost < best) { best = cost; bn = w; }
    }
  }
  if (bn == 256) return launch<256>(live, m, st);
  if (bn == 192) return launch<192>(live, m, st);
  if (bn == 128) return launch<128>(live, m, st);
  if (use_bn256(live, m)) return launch<256>(live, m, st);
  return launch<128>(live, m, st);
}

cudaError_t gemm_bf16(const GemmOp &op, cudaStream_t st) { return gemm_bf16_group(&op, 1, st); }

size_t gemm_flags_count(int M, int N) { return (size_t)((M + 127) / 128) * ((N + 127) / 128); }

}  // namespace jk
