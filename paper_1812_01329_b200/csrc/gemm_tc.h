// gemm_tc.h — host interface of the tcgen05 bf16 GEMM (gemm_tc.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace jk {

// NEXT-3: gradient reduction fused into the weight-gradient GEMM's epilogue (P:298 — the
// collective inside the step — done over NVLink peer memory, tile by tile, as the tiles finish).
// C lives in an NCCL symmetric window (load/store accessible on every rank of the node); tile t
// is owned by rank t mod nranks: every rank signals the owner when its tile t is written, the
// owner sums the ranks' tiles in rank order (deterministic, bit-identical everywhere), writes
// the sum into every rank's window and signals each rank. Flags are epoch counters: never reset.
struct FusedReduce {
  void *win = nullptr;   // ncclWindow_t of the arena (nullptr: no fused reduction)
  size_t c_off = 0;      // byte offset of this GEMM's C inside the arena window
  void *fwin = nullptr;  // ncclWindow_t of the tile flags
  size_t flag_off = 0;   // byte offset of this GEMM's flags (2 x u32 per tile: ready, reduced)
  int nranks = 1, rank = 0;
  unsigned epoch = 0;    // this step's epoch (1, 2, ...): ready counts reach epoch * nranks
  int force_pull = 0;    // test hook: run the owner's pull / sum / push even with one rank
};

struct GemmEpilogue {
  float *C = nullptr;               // fp32 output [M, ldc] (row-major), may be null
  int ldc = 0;
  __nv_bfloat16 *Cb = nullptr;      // optional bf16 copy of the output
  int ldcb = 0;
  const float *bias_col = nullptr;  // + bias[n]
  const float *bias_row = nullptr;  // + bias[m]
  int accumulate = 0;               // C += result
  FusedReduce fr;                   // fused cross-rank reduction of C (TMA-store path only)
  int dev_no_drain = 0;             // dev measurement (JANUS_GEMM_EPI_SKIP=2): release TMEM unread
  int dev_x64 = 0;                  // dev measurement (JANUS_GEMM_EPI_SKIP=3): drain with x64 loads
};

// D[M,N] = A[M,K] . B[N,K]^T.
//  a_mn == 0: A stored [M][lda] (K contiguous);  a_mn == 1: A stored [K][lda] (M contiguous).
//  b_mn == 0: B stored [N][ldb] (K contiguous);  b_mn == 1: B stored [K][ldb] (N contiguous).
// lda/ldb multiples of 8 elements; base pointers 16-B aligned. Out-of-range K/M/N reads are
// zero-filled by TMA.
struct GemmOp {
  int M = 0, N = 0, K = 0;
  const __nv_bfloat16 *A = nullptr;
  int lda = 0, a_mn = 0;
  const __nv_bfloat16 *B = nullptr;
  int ldb = 0, b_mn = 0;
  GemmEpilogue ep;
  const int *K_dev = nullptr;  // optional device-resident K (<= K): data-dependent reductions
  // split-K (deterministic: partials added in split order): `flags` = gemm_flags_count(M, N)
  // ZERO-INITIALISED counters (every launch leaves them zero again) and `partials` = fp32
  // scratch of partials_cap floats, both private to the stream; null disables splitting.
  // splits: 0 = automatic, >= 1 forces the count (capped by the scratch).
  unsigned *flags = nullptr;
  float *partials = nullptr;
  size_t partials_cap = 0;
  int splits = 0;
  int bn = 0;  // tile width: 0 = automatic, 128 or 256 forces it (single launches)
  // split_add (with splits = 2): each K half reduce-adds its tile into C through the TMA store
  // (cp.reduce.async.bulk .add) — no partials, no fixup pass; C must be ZERO on entry. Two
  // addends onto zero give the same bits in either order, so the result stays deterministic.
  int split_add = 0;
};

cudaError_t gemm_bf16(const GemmOp &op, cudaStream_t st);
// Several GEMMs in one persistent launch (tiles concatenated; <= 4 ops). Ops sharing the kernel
// configuration (operand majors, tile width) are grouped; split-K applies to single launches only.
cudaError_t gemm_bf16_group(const GemmOp *ops, int n, cudaStream_t st);
size_t gemm_flags_count(int M, int N);  // flags needed by a split-K launch of an M x N GEMM
// Tile geometry a grouped launch uses for each op (BN, M blocks incl. cluster ghosts, N blocks):
// the fused reduction's tile ids are mb + mblocks * nb.
void gemm_group_tiling(const GemmOp *ops, int n, int *bn, int *mblocks, int *nblocks);
bool make_tmap_bf16(CUtensorMap *m, const void *ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                    uint32_t box_outer);
bool make_tmap_bf16_chunks(CUtensorMap *m, const void *ptr, uint64_t rows, uint64_t ld,
                           uint64_t n_chunks, uint32_t box_rows, uint32_t box_chunks);

}  // namespace jk
