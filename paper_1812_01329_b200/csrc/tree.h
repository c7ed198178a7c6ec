// tree.h — level-batched TreeLSTM device program (tree.cu): the recursive InvokeOp of the TreeNN
// program (P:224, P:316 fn6) flattened into a height schedule and executed level by level.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "step_kernels.h"

namespace jk {

constexpr int TREE_MAX_LEVELS = 130;  // heights < 128 (<= 127 nodes per tree)

// Device schedule (reading Q8): level = height; order = stable sort of node ids by height.
struct TreeSched {
  int *height;     // [N]
  int *order;      // [N] node id at level-order position
  int *irank;      // [N] rank among internal nodes in level order (-1 for leaves)
  int *pslot;      // [N] (irank(parent) << 1 | side), -1 for roots
  int *lvl_off;    // [TREE_MAX_LEVELS + 1] level offsets over all nodes
  int *meta;       // [0] = number of levels (max height + 1), [1] = N, [2] = #leaves, [3] = #internal
  int *tree_of;    // [N] tree index of each node
  int *pcount;     // [N] scratch: parent counts (guard)
};

struct TreeDims {
  int N, B, V, E, H, C;
  int Ep;   // x_leaf pitch (bf16) >= E + 1, multiple of 64
  int P2;   // stage_h pitch (bf16) >= 2H + 1, multiple of 64
  int P5;   // DZ_int pitch >= 5H, multiple of 64
  int P3;   // DZ_leaf pitch >= 3H, multiple of 64
  int Nmax; // rows allocated for the node arrays (the tensor maps span Nmax rows: step-invariant)
  int rnn;  // 1: TreeRNN cell (one tanh gate, leaves = word vectors), 0: TreeLSTM
};

struct TreeBufs {
  const int *kind, *left, *right, *word, *off, *label;
  const float *E;              // frozen embedding table [V][E] fp32
  const float *b;              // bias [4H] blocks (i, f, o, u)
  const float *Wc, *bc;        // classifier [C][H], [C]
  __nv_bfloat16 *x_leaf;       // [N][Ep] leaf inputs in level-0 order (+ ones column at E)
  __nv_bfloat16 *stage_h;      // [N_int][P2] children h (h_l | h_r), ones column at 2H
  float *stage_c;              // [N_int][2H] children c
  float *gates_int;            // [N_int][5H] (i, f_l, f_r, o, u) per unit, interleaved 5u+g
  float *c_int;                // [N_int][H] (TreeRNN: h of the internal nodes)
  float *gates_leaf;           // [n_leaf][3H] (i, o, u) interleaved 3u+g
  float *c_leaf;               // [n_leaf][H]
  float *root_h;               // [B][H]
  float *dh_node, *dc_node;    // [N][H]
  __nv_bfloat16 *DZ_int;       // [N_int][P5] rb(dz), interleaved 5u+g
  __nv_bfloat16 *DZ_leaf;      // [n_leaf][P3] rb(dz), interleaved 3u+g
  float *gWc, *gbc;            // classifier gradients [C][H], [C]
  float *rowloss;              // [B]
  float *root_part;            // [ceil(B/8)][C*H + C] per-block classifier-gradient partials
  unsigned int *barrier;       // grid barrier counters (zeroed by step init)
  unsigned int *bwd_lvl;       // backward per-level arrival counters (one 128-B line per level; zeroed by the forward)
  unsigned long long *dbg;     // dev hook (janus_dev_set_probe): per-barrier arrival / release
                               // %globaltimer of every CTA, [2 kernels][256 syncs][256 CTAs][2]
};

cudaError_t launch_tree_guard(const TreeBufs &t, const TreeDims &d, const TreeSched &s, unsigned id,
                              long long V, long long max_nodes, DevStatus *st, cudaStream_t str);
cudaError_t launch_tree_guard_schedule(const TreeBufs &t, const TreeDims &d, const TreeSched &s, unsigned id,
                                       long long V, long long max_nodes, DevStatus *st, cudaStream_t str);
cudaError_t launch_tree_schedule(const TreeBufs &t, const TreeDims &d, const TreeSched &s,
                                 const DevStatus *st, cudaStream_t str);
// forward: leaf gather, leaf level, internal levels (one cooperative launch)
cudaError_t launch_tree_fwd(const TreeBufs &t, const TreeDims &d, const TreeSched &s,
                            const __nv_bfloat16 *Wl_il, const __nv_bfloat16 *U_il, int grid,
                            const DevStatus *st, cudaStream_t str);
// root classifier + softmax xent (mean over trees) + its backward (dh of the roots)
cudaError_t launch_tree_root(const TreeBufs &t, const TreeDims &d, const TreeSched &s,
                             DevStatus *st, cudaStream_t str);
// backward: internal levels top-down (cell backward, then dz . U scattered to the children),
// then the leaf cell backward (one cooperative launch)
cudaError_t launch_tree_bwd(const TreeBufs &t, const TreeDims &d, const TreeSched &s,
                            const __nv_bfloat16 *UT_il, int grid, const DevStatus *st,
                            cudaStream_t str);
// bf16 working copies: rows interleaved by `ng` gates (row ng*u+g <- g*H+u), optional transpose
cudaError_t launch_cast_il(const float *src, int H, int ng, int cols, __nv_bfloat16 *dst, int ld,
                           cudaStream_t s);
// the three above for one TreeLSTM step in one launch (W_leaf rows, U rows, U^T tiles)
cudaError_t launch_tree_cast3(const float *Wl, __nv_bfloat16 *Wl_il, int ldw, const float *U,
                              __nv_bfloat16 *U_il, int ldu, __nv_bfloat16 *UT_il, int ldut, int H, int E,
                              cudaStream_t s);
cudaError_t launch_cast_il_T(const float *src, int H, int ng, int cols, __nv_bfloat16 *dst, int ld,
                             cudaStream_t s);

}  // namespace jk
