// step_kernels.h — SIMT kernels of the speculative step: status/guards (AssertOps), operand
// preparation, embedding gather, softmax cross-entropy, embedding-gradient segmented sum,
// loss/status finalisation and the predicated all-or-nothing commit.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace jk {

// Device status word (16-byte aligned; copied to the host once per step).
struct DevStatus {
  unsigned long long key;  // min over failing (assumption_id << 40 | element index); ~0 = pass
  long long observed;      // value of the failing element (filled by finalize)
  int runtime_err;         // nonzero: runtime error in a node (bad id) -> ERR_RUNTIME
  int status;              // janus_status computed on the device (OK / ASSUMPTION_FAILED / RUNTIME)
  float loss;
  int trip;                // device trip count of the While loop (diagnostic)
  unsigned int flags;
  int pad[3];
};
static_assert(sizeof(DevStatus) == 48, "DevStatus layout");

constexpr unsigned long long KEY_PASS = ~0ull;
constexpr int IDX_BITS = 40;

// A RUNTIME assumption evaluated on the device (AssertOp).
enum GuardKind { G_ALL_EQ = 0, G_FIRST_EQ = 1, G_RANGE = 2, G_FORCED = 3,
                 G_TREE = 4 /* evaluated by the forest guard; listed for the observed lookup */,
                 G_FIRST_TRUTH = 5 /* (data[0] != 0) == (value != 0): a branch arm */ };
struct GuardDesc {
  int kind;
  unsigned int id;
  const int *data;
  long long n;
  long long value, lo, hi;
  const int *data2;  // G_TREE: element i >= n is data2[i - n]
};
constexpr int MAX_GUARDS = 8;
struct GuardList {
  int n;
  GuardDesc g[MAX_GUARDS];
};

// status word := PASS; zeroes words 0, stride, 2 stride, ... < nbar of the step-flag area
cudaError_t launch_step_init(DevStatus *st, unsigned int *barriers, int nbar, cudaStream_t s, int stride = 1);
cudaError_t launch_guards(const GuardList &gl, DevStatus *st, cudaStream_t s);
// init + guards in one single-block launch (the step's first launch)
cudaError_t launch_step_init_guards(DevStatus *st, unsigned int *barriers, int nbar, int stride,
                                    const GuardList &gl, cudaStream_t s);

// gather X[t*B+b] = rb(E[tok[b][t]]) (bf16, ld) with X[:, E] = 1 (ones column for bias grads);
// ids outside [0,V) set runtime_err and read row 0.
cudaError_t launch_gather(const float *E, int V, int Edim, const int *tok, int B, int W, int T,
                          const int *T_dev, __nv_bfloat16 *X, int ldx, DevStatus *st,
                          cudaStream_t s);
// While mode: device trip count st->trip = min(max(lens), W) (the LoopCond bound).
cudaError_t launch_trip(const int *lens, int B, int W, DevStatus *st, cudaStream_t s);

// x (fp32, canonical rows) -> bf16 copies: interleaved rows (4u+g <- g*H+u) and/or transposed.
// Fused per-step operand preparation (one launch): see prep_kernel in step_kernels.cu.
enum PrepKind { P_CAST_ROWS = 0, P_CAST_T_IL = 1, P_BIAS_IL = 2, P_FILL_COL = 3 };
struct PrepSeg {
  int kind;
  const float *src;      // fp32 source (CAST_ROWS, CAST_T_IL, BIAS_IL)
  __nv_bfloat16 *dst;    // bf16 destination (CAST_ROWS, CAST_T_IL, FILL_COL)
  float *fdst;           // fp32 destination (BIAS_IL)
  int rows, cols;        // CAST_ROWS: dst rows, valid source columns; FILL_COL: rows, ones column
  int ld_src, ld_dst;    // pitches (elements); FILL_COL zeroes (cols, ld_dst)
  int H;                 // CAST_ROWS: > 0 gate-interleaves rows; CAST_T_IL / BIAS_IL: hidden size
};
constexpr int MAX_PREP = 24;
struct PrepList {
  int n;
  PrepSeg s[MAX_PREP];
  int blk[MAX_PREP + 1];  // set by launch_prep: segment k owns blocks [blk[k], blk[k+1]) of the 1-D grid
};
cudaError_t launch_prep(const PrepList &pl, cudaStream_t s);
// launch_prep and launch_gather in one launch (prep blocks first, then the gather's)
cudaError_t launch_prep_gather(const PrepList &pl, const float *E, int V, int Edim, const int *tok, int B, int W,
                              int T, const int *T_dev, __nv_bfloat16 *X, int ldx, DevStatus *st, cudaStream_t s);
cudaError_t launch_cast_rows(const float *src, int R, int Cc, int ld_src, __nv_bfloat16 *dst,
                             int ld_dst, int interleave_H, cudaStream_t s);
cudaError_t launch_cast_transpose_interleaved(const float *W, int H, __nv_bfloat16 *WT, int ldwt,
                                              cudaStream_t s);
cudaError_t launch_bias_interleave(const float *b, int H, float *out, cudaStream_t s);
cudaError_t launch_fill_col(__nv_bfloat16 *X, int rows, int ld, int col, float v, int zero_to,
                            cudaStream_t s);

// per-row softmax cross-entropy: rowloss[r], dy = mask (softmax - onehot) / n_valid (bf16).
// Row r = t*B + b targets tgt[b][t]; in While mode rows with t >= len_b (or t >= *T_dev) are
// masked. n_valid: host constant, or computed from lens on the device when lens != nullptr.
// Inverted dropout (Zaremba [51]; masks: philox.cuh, reading R14) of rows [0, rows) of a
// time-major matrix (global row r = t * B + b), columns [0, cols): bf16 mode: dst = rb(src * m / (1 -
// p)) with the columns cols .. ld copied unchanged (the ones column); f32 mode: x *= m / (1 - p) in
// place. key: device i32[2].
cudaError_t launch_dropout_bf16(const __nv_bfloat16 *src, __nv_bfloat16 *dst, int rows, int cols, int ld,
                                const int *key, int site, float p, cudaStream_t s);
cudaError_t launch_dropout_f32(float *x, int rows, int cols, int ld, const int *key, int site, float p,
                               cudaStream_t s, int row0 = 0);  // row0: global index of row 0
uint32_t dropout_threshold(float p);  // floor(p * 2^32), saturated
// zero / zero_n4 (optional): a float4 buffer the kernel zero-fills on the side (the reduce-add
// target of the next GEMM), so no separate memset sits on the step's critical path
cudaError_t launch_xent(const float *logits, int V, int ldl, int rows, const int *tgt, int B, int W,
                        const int *lens, const int *T_dev, float n_valid, __nv_bfloat16 *dy,
                        int lddy, float *rowloss, DevStatus *st, cudaStream_t s,
                        float4 *zero = nullptr, long long zero_n4 = 0);

// embedding gradient: seg_word[k] (k < *nseg, slot order unspecified) lists the distinct ids of
// the step; seg_grad[k][ldg] = sum of the dX rows of that id, summed in a fixed order
// (deterministic). owner: V + 2 T*B + 1 ints of scratch. seg_word slots are in order of first
// occurrence (deterministic).
cudaError_t launch_embed_grad(const int *tok, int B, int W, int T, const int *T_dev, int V,
                              const float *dX, int ldx, int Edim, int *seg_word, int *owner,
                              float *seg_grad, int ldg, int *nseg, cudaStream_t s,
                              int part = 0);  // part 1: the bucketing only, 2: the segment sums only

// loss = sum(rowloss) / n_valid... rowloss already carries the 1/n_valid scale; status decode.
cudaError_t launch_finalize(const float *rowloss, int rows, const GuardList &gl, DevStatus *st,
                            int world_size, cudaStream_t s);

// data-parallel abort agreement (host_dp.cpp): scratch[0] = packed key (MIN over ranks),
// scratch[1] = runtime error (MAX), scratch[2] = observed of the winning rank (MAX), scratch[3] =
// this rank's packed key. DevStatus.pad[0] receives the failing rank.
// Global abort agreement (reading Q12 / R7), the arithmetic shared by the device kernels and
// the host transport of the protocol test (host_dp.cpp). scratch: [0] packed key (MIN over
// ranks), [1] runtime-error flag (MAX), [2] observed value of the winning rank (MAX), [3] this
// rank's own packed key. Packed key = assumption id << 48 | rank << 40 | element index.
__host__ __device__ inline void dp_pack(const DevStatus &st, long long *sc, int rank) {
  unsigned long long p = KEY_PASS;
  if (st.key != KEY_PASS)
    p = ((st.key >> IDX_BITS) << 48) | ((unsigned long long)(rank & 0xff) << IDX_BITS) |
        (st.key & ((1ull << IDX_BITS) - 1));
  sc[0] = (long long)p;
  sc[1] = st.runtime_err;
  sc[3] = (long long)p;
}
__host__ __device__ inline void dp_observed(const DevStatus &st, long long *sc) {
  const bool mine = sc[3] == sc[0] && (unsigned long long)sc[0] != KEY_PASS;
  sc[2] = mine ? st.observed : (long long)(-9223372036854775807LL - 1);
}
__host__ __device__ inline void dp_unpack(DevStatus &st, const long long *sc) {
  const unsigned long long p = (unsigned long long)sc[0];
  if (p != KEY_PASS) {
    st.key = ((p >> 48) << IDX_BITS) | (p & ((1ull << IDX_BITS) - 1));
    st.pad[0] = (int)((p >> IDX_BITS) & 0xff);
    st.observed = sc[2];
    st.status = 1;
  } else {
    st.key = KEY_PASS;
    st.runtime_err = (int)sc[1];
    st.status = sc[1] ? 4 : 0;
  }
}
// A failure decided on the host (dispatch guard of a null step); id ~0 = invalid arguments on
// this rank, agreed as a runtime error (no commit).
__host__ __device__ inline void dp_set_failure(DevStatus &st, unsigned id, long long index, long long observed) {
  if (id == 0xffffffffu) {
    st.key = KEY_PASS;
    st.runtime_err = 1;
    st.status = 4;
    return;
  }
  const unsigned long long idx = index < 0 ? (1ull << IDX_BITS) - 1 : (unsigned long long)index;
  st.key = ((unsigned long long)id << IDX_BITS) | idx;
  st.observed = observed;
  st.status = 1;
}
cudaError_t launch_dp_pack(const DevStatus *st, long long *scratch, int rank, cudaStream_t s);
cudaError_t launch_dp_observed(const DevStatus *st, long long *scratch, cudaStream_t s);
cudaError_t launch_dp_unpack(DevStatus *st, const long long *scratch, cudaStream_t s);
// a dispatch failure on this rank inside a data-parallel null step (id 0xffffffff: this rank's
// arguments were invalid; it joins the agreement as a runtime error)
cudaError_t launch_set_failure(DevStatus *st, unsigned id, long long index, long long observed,
                               cudaStream_t s);
// dense embedding gradient for the data-parallel allreduce: zero + scatter the segment sums
cudaError_t launch_scatter_rows(const float *seg_grad, int ldg, const int *seg_word, const int *nseg,
                                float *dense, int V, int cols, cudaStream_t s);

// commit segments (P:164 all-or-nothing, P:282 deferred update)
enum CommitKind { C_DENSE = 0, C_DENSE_IL = 1, C_BIAS_COL = 2, C_BIAS_COL_IL = 3, C_COPY = 4,
                  C_TAG = 5, C_SPARSE_ROWS = 6, C_TREE_BIAS = 7,
                  C_DENSE_IL_T = 8 /* C_DENSE_IL with a transposed copy: 32 x 64 tiles */ };
struct CommitSeg {
  int kind;
  float *dst;          // master (fp32) or state destination
  const float *grad;   // gradient / copy source
  int rows, cols;      // master shape (canonical)
  int ldg;             // gradient row pitch
  int col;             // C_BIAS_COL*: gradient column holding the bias gradient
  int H;               // interleave H (C_*_IL)
  float lr;            // learning rate / n_ranks
  const int *rows_idx; // C_SPARSE_ROWS: word id per gradient row
  const int *nrows;    // C_SPARSE_ROWS: device count of rows
  int *idst;           // C_TAG
  int ival;
  int ng;              // C_DENSE_IL: gates per unit (0 = 4)
  const float *grad2;  // C_TREE_BIAS: leaf wgrad (bias column col2, pitch ldg2)
  int ldg2, col2;
  const int *pred;     // device predicate (`if training:` Switch): skip the segment when *pred == 0
  // bf16 working copies refreshed from the committed masters (R1), so the next step needs no cast:
  __nv_bfloat16 *bcopy; int ldb;  // row copy: row ri (interleaved, C_DENSE_IL*) or rc (C_DENSE)
  __nv_bfloat16 *tcopy; int ldt;  // C_DENSE_IL_T: transposed copy, tcopy[k][ri] (ri = ng*u + g, ng = 4 if 0)
};
constexpr int MAX_COMMIT = 24;
struct CommitList {
  int n;
  CommitSeg s[MAX_COMMIT];
  int blk[MAX_COMMIT + 1];  // set by launch_commit: segment k owns blocks [blk[k], blk[k+1])
};
cudaError_t launch_commit(const CommitList &cl, const DevStatus *st, cudaStream_t s);
// finalize (loss sum, status word) folded into the commit launch as one extra block; the commit
// blocks take their all-or-nothing decision from the key and runtime-error flags (single rank)
struct FinalizeArgs {
  const float *rowloss;
  int rows;
  GuardList gl;
};
cudaError_t launch_commit_finalize(const CommitList &cl, const FinalizeArgs &fa, DevStatus *st, cudaStream_t s);

}  // namespace jk
