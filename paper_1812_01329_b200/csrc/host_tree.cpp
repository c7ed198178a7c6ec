// host_tree.cpp — speculative lowering and device program of the TreeLSTM training step
// (Table 2 TreeLSTM on SST; recursion through InvokeOp, P:224, P:316 fn6).
//
// lower_tree recognises the generic graph of the recursive program (function 1 = node(n): a
// Switch/Merge on kind[n] between a TREELSTM_LEAF arm and a TREELSTM_CELL arm over two recursive
// INVOKEs; main = loop over trees, root classifier LINEAR + SOFTMAX_XENT, SGD_APPLY effects) and,
// under the TREE_BINARY assumption, replaces the recursion by a device-built level schedule and
// level-batched tensor-core evaluation (tree.cu). Without TREE_BINARY the graph has no device
// lowering (ERR_UNSUPPORTED; the imperative path still runs it).
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>

#include "gemm_tc.h"
#include "host.h"
#include "imp_kernels.h"
#include "step_kernels.h"
#include "tree.h"

namespace jk {

static int r8(int x) { return (x + 7) & ~7; }
static int r64(int x) { return (x + 63) & ~63; }
static size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

static bool slot_dims(const Graph &g, int node, int *slot, int64_t d[4]) {
  const int o = producer_origin(g, node);
  if (o < 0 || g.ops[o].kind != JOP_STATE_READ) return false;
  *slot = (int)g.ops[o].iattr[0];
  for (int k = 0; k < 4; ++k) d[k] = g.ops[o].iattr[3 + k];
  return true;
}

bool lower_tree(Graph &g, std::string &why) {
  TreePlan &p = g.tree;
  p = TreePlan();
  int leaf = -1, cell = -1, rcell = -1, self_invoke = 0, main_invoke = -1, xent = -1;
  for (int i = 0; i < (int)g.ops.size(); ++i) {
    const janus_op &o = g.ops[i];
    if (o.func == 1 && o.kind == JOP_TREELSTM_LEAF) leaf = i;
    if (o.func == 1 && o.kind == JOP_TREELSTM_CELL) cell = i;
    if (o.func == 1 && o.kind == JOP_TREERNN_CELL) rcell = i;
    if (o.func == 1 && o.kind == JOP_INVOKE && o.iattr[0] == 1) ++self_invoke;
    if (o.func == 0 && o.kind == JOP_INVOKE && o.iattr[0] == 1) main_invoke = i;
    if (o.func == 0 && o.kind == JOP_SOFTMAX_XENT) xent = i;
  }
  // TreeRNN (Table 2): the leaf arm is the word vector itself, the internal arm a
  // TREERNN_CELL; TreeLSTM: TREELSTM_LEAF / TREELSTM_CELL
  p.rnn = rcell >= 0 && leaf < 0 && cell < 0;
  if ((!p.rnn && (leaf < 0 || cell < 0)) || self_invoke != 2 || main_invoke < 0 || xent < 0) {
    why = "not the recursive TreeLSTM / TreeRNN pattern";
    return false;
  }
  for (const auto &a : g.asms)
    if (a.kind == JA_DTYPE_EQ && a.target >= 0 && a.target <= 5) {
      if (a.dtype != JANUS_I32 && a.dtype != JANUS_I64) {
        why = "forest / label arguments must be int32 or int64";
        return false;
      }
      p.arg_dtype[a.target] = a.dtype;
    }
  const janus_op &inv = g.ops[main_invoke];
  if (inv.n_in != (p.rnn ? 8 : 9)) { why = "node() arity"; return false; }
  for (int k = 1; k <= 4; ++k) {
    const int o = producer_origin(g, inv.in_node[k]);
    if (g.ops[o].kind != JOP_ARG || g.ops[o].iattr[0] != k - 1) { why = "forest arguments"; return false; }
  }
  int64_t d[4];
  if (!slot_dims(g, inv.in_node[5], &p.slot_E, d)) { why = "embedding slot"; return false; }
  p.V = (int)d[0]; p.E = (int)d[1];
  if (p.rnn) {
    if (!slot_dims(g, inv.in_node[6], &p.slot_U, d)) { why = "W slot"; return false; }
    p.H = (int)d[0];
    if (d[1] != 2 * p.H || p.E != p.H) { why = "TreeRNN W must be [H, 2H] with E = H (leaves are word vectors)"; return false; }
    if (!slot_dims(g, inv.in_node[7], &p.slot_b, d) || d[0] != p.H) { why = "b shape"; return false; }
  } else {
    if (!slot_dims(g, inv.in_node[6], &p.slot_Wleaf, d)) { why = "W_leaf slot"; return false; }
    p.H = (int)(d[0] / 3);
    if (d[0] != 3 * p.H || d[1] != p.E) { why = "W_leaf shape"; return false; }
    if (!slot_dims(g, inv.in_node[7], &p.slot_U, d) || d[0] != 5 * p.H || d[1] != 2 * p.H) { why = "U shape"; return false; }
    if (!slot_dims(g, inv.in_node[8], &p.slot_b, d) || d[0] != 4 * p.H) { why = "b shape"; return false; }
  }
  if (p.H > 1024) { why = "hidden size > 1024 (the forward keeps the bias in shared memory)"; return false; }
  const janus_op &x = g.ops[xent];
  const janus_op &lin = g.ops[x.in_node[0]];
  if (lin.kind != JOP_LINEAR) { why = "classifier"; return false; }
  if (!slot_dims(g, lin.in_node[1], &p.slot_Wc, d) || d[1] != p.H) { why = "W_c"; return false; }
  p.C = (int)d[0];
  if (!slot_dims(g, lin.in_node[2], &p.slot_bc, d) || d[0] != p.C) { why = "b_c"; return false; }
  const int lab = producer_origin(g, x.in_node[1]);
  if (g.ops[lab].kind != JOP_ARG || g.ops[lab].iattr[0] != 5) { why = "labels"; return false; }
  for (const auto &o : g.ops) {
    if (o.func != 0) continue;
    if (o.kind == JOP_SGD_APPLY) {
      const int s = (int)o.iattr[0];
      const float lr = (float)o.fattr[0];
      if (s == p.slot_Wleaf && s >= 0) p.lr_Wleaf = lr;
      else if (s == p.slot_U) p.lr_U = lr;
      else if (s == p.slot_b) p.lr_b = lr;
      else if (s == p.slot_Wc) p.lr_Wc = lr;
      else if (s == p.slot_bc) p.lr_bc = lr;
      else { why = "SGD on an unsupported slot (the embedding table is frozen, reading Q5)"; return false; }
    }
    if (o.kind == JOP_STATE_WRITE) { why = "state writes in the tree program"; return false; }
  }
  p.B = -1;
  for (const auto &a : g.asms) {
    if (a.kind == JA_TREE_BINARY && a.target == 0) {
      p.tree_guard = true;
      p.tree_guard_id = a.id;
      p.max_nodes = (int)a.value;
      if (a.hi != p.V) { why = "TREE_BINARY word bound != V"; return false; }
    }
    if (a.kind == JA_SHAPE_MATCH && a.target == 4 && a.ndim == 1 && a.dims[0] > 0) p.B = (int)a.dims[0] - 1;
    if (a.kind == JA_SHAPE_MATCH && a.target == 5 && a.ndim == 1 && a.dims[0] > 0 && p.B < 0) p.B = (int)a.dims[0];
  }
  if (!p.tree_guard) { why = "no TREE_BINARY assumption: recursion cannot be flattened"; return false; }
  if (p.B <= 0) { why = "batch of trees not fixed by a SHAPE_MATCH assumption"; return false; }
  if (p.max_nodes < 1 || p.max_nodes > 127) { why = "max nodes per tree must be in [1, 127]"; return false; }
  if (g.opts.gemm_dtype == JANUS_F32) { why = "tree program runs the bf16 tensor-core path only"; return false; }
  for (const auto &a : g.asms) {
    if (a.mode != JANUS_MODE_RUNTIME || a.kind == JA_TREE_BINARY) continue;
    if (a.kind != JA_VALUE_EQ && a.kind != JA_RANGE) { why = "unsupported runtime assumption"; return false; }
    LmPlan::RG r{};
    r.id = a.id; r.value = a.value; r.lo = a.lo; r.hi = a.hi; r.arg = a.target; r.slot = -1;
    r.ref_arg = a.ref_arg; r.ref_dim = a.ref_dim;
    r.kind = a.kind == JA_RANGE ? G_RANGE : G_FIRST_EQ;
    if (!g.opts.strip_asserts) p.runtime_guards.push_back(r);
  }
  if (g.opts.fail_assert_id >= 0)
    for (const auto &a : g.asms)
      if ((int)a.id == g.opts.fail_assert_id && a.mode == JANUS_MODE_RUNTIME) {
        LmPlan::RG r{};
        r.kind = G_FORCED; r.id = a.id; r.arg = -1; r.slot = -1;
        p.runtime_guards.push_back(r);
      }
  if (g.opts.strip_asserts) p.tree_guard = false;
  if ((int)p.runtime_guards.size() + (p.tree_guard ? 1 : 0) > MAX_GUARDS) { why = "too many runtime guards"; return false; }
  p.max_N = p.max_nodes * p.B;
  // ------------------------------------------------------------------ workspace layout
  const int N = p.max_N, H = p.H, E = p.E, V = p.V;
  const int NG = p.rnn ? 1 : 5;  // gates per unit of the internal cell
  const size_t NL = p.rnn ? 0 : (size_t)N;  // rows of the leaf-GEMM buffers (none for the TreeRNN)
  p.Ep = r64(E + 1); p.P2 = r64(2 * H + 1); p.P5 = r64(NG * H); p.P3 = r64(3 * H);
  p.ldgU = r8(2 * H + 1); p.ldgW = r8(E + 1);
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = a256(o + bytes); return r; };
  p.off.status = take(sizeof(DevStatus));
  // 64 grid-barrier words, then one 128-B line per level: the forward's per-level arrival counters
  // (+ the backward's per-level arrival counters, one line per level)
  p.off.barriers = take((64 + 2 * (size_t)TREE_MAX_LEVELS * 32) * sizeof(unsigned));
  p.off.stage_args = take((4ull * N + 2ull * (p.B + 1)) * sizeof(int));
  p.off.height = take((size_t)N * 4); p.off.order = take((size_t)N * 4); p.off.irank = take((size_t)N * 4);
  p.off.pslot = take((size_t)N * 4); p.off.tree_of = take((size_t)N * 4); p.off.pcount = take((size_t)N * 4);
  p.off.lvl_off = take((TREE_MAX_LEVELS + 2) * 4); p.off.meta = take(64);
  p.off.x_leaf = take(NL * p.Ep * 2);
  p.off.stage_h = take((size_t)N * p.P2 * 2);
  p.off.stage_c = take(NL * 2 * H * 4);
  p.off.gates_int = take(NL * 5 * H * 4);
  p.off.c_int = take((size_t)N * H * 4);
  p.off.gates_leaf = take(NL * 3 * H * 4);
  p.off.c_leaf = take(NL * H * 4);
  p.off.root_h = take((size_t)p.B * H * 4);
  p.off.root_part = take((size_t)((p.B + 7) / 8) * (p.C * H + p.C) * 4);  // root classifier partials
  p.off.dh_node = take((size_t)N * H * 4);
  p.off.dc_node = take((size_t)N * H * 4);
  p.off.DZ_int = take((size_t)(N + 64) * p.P5 * 2);
  p.off.DZ_leaf = take(p.rnn ? 0 : (size_t)(N + 64) * p.P3 * 2);
  p.off.rowloss = take((size_t)p.B * 4);
  p.off.U_il = take((size_t)NG * H * p.P2 * 2);
  p.off.UT_il = take((size_t)2 * H * p.P5 * 2);
  p.off.Wl_il = take(p.rnn ? 0 : (size_t)3 * H * p.Ep * 2);
  p.off.arena_begin = o;
  p.off.gU = take((size_t)NG * H * p.ldgU * 4);
  p.off.gWl = take(p.rnn ? 0 : (size_t)3 * H * p.ldgW * 4);
  p.off.gWc = take((size_t)p.C * H * 4);
  p.off.gbc = take((size_t)p.C * 4);
  p.off.arena_end = o;
  p.off.dp_scratch = take(64);
  p.ws_bytes = o;
  (void)V;
  char buf[512];
  snprintf(buf, sizeof buf,
           "%s: V=%d E=%d H=%d C=%d B=%d max_nodes/tree=%d guards=%zu+tree_binary "
           "phases=[init,guards,tree_guard,schedule,cast,tree_fwd(leaf level + internal levels, "
           "cooperative),root_xent,tree_bwd(levels top-down, cooperative),gemm_dU,gemm_dWleaf,"
           "finalize,commit]",
           p.rnn ? "treernn" : "treelstm", p.V, p.E, p.H, p.C, p.B, p.max_nodes, p.runtime_guards.size());
  g.describe = buf;
  return true;
}

#define TCHK(name, x)                             \
  do {                                            \
    g.prof.mark(name, st);                        \
    cudaError_t e_ = (x);                         \
    g.launches++;                                 \
    if (e_ != cudaSuccess) return JANUS_ERR_CUDA; \
  } while (0)

janus_status run_tree(Graph &g, const janus_tensor *args, int n_args, const janus_tensor *state,
                      const janus_tensor *outs, int n_outs, const janus_tensor &ws, cudaStream_t st,
                      janus_failure *fail) {
  const TreePlan &p = g.tree;
  if (n_args < 6 || !ws.data || (size_t)ws.shape[0] * (ws.dtype == JANUS_U8 ? 1 : 4) < p.ws_bytes)
    return JANUS_ERR_INVALID;
  uint8_t *W = static_cast<uint8_t *>(ws.data);
  const int N = (int)args[0].shape[0], B = p.B, H = p.H, E = p.E;
  if (args[0].ndim != 1 || N < 1 || N > p.max_N) return JANUS_ERR_INVALID;
  for (int a = 0; a < 6; ++a) {
    const int64_t n = a < 4 ? N : (a == 4 ? B + 1 : B);
    if (args[a].ndim != 1 || args[a].shape[0] != n || args[a].dtype != p.arg_dtype[a]) return JANUS_ERR_INVALID;
  }
  // arguments: device pointers, or host buffers staged through the workspace; int64 arguments
  // of a type-specialised graph are narrowed on the device into the same staging area
  const int *argp[6];
  int *stage = reinterpret_cast<int *>(W + p.off.stage_args);
  for (int a = 0; a < 6; ++a) {
    const int64_t n = a < 4 ? N : (a == 4 ? B + 1 : B);
    if (p.arg_dtype[a] == JANUS_I64) {
      if (!is_device_ptr(args[a].data)) return JANUS_ERR_INVALID;
      if (imp::i64_to_i32(stage, static_cast<const long long *>(args[a].data), n, st) != cudaSuccess)
        return JANUS_ERR_CUDA;
      g.launches++;
      argp[a] = stage;
      stage += n;
      continue;
    }
    if (is_device_ptr(args[a].data)) { argp[a] = static_cast<const int *>(args[a].data); continue; }
    if (cudaMemcpyAsync(stage, args[a].data, n * 4, cudaMemcpyHostToDevice, st) != cudaSuccess) return JANUS_ERR_CUDA;
    argp[a] = stage;
    stage += n;
  }
  auto sf = [&](int slot, int64_t n) -> float * {
    const janus_tensor &t = state[slot];
    int64_t k = 1;
    for (int i = 0; i < t.ndim; ++i) k *= t.shape[i];
    if (t.dtype != JANUS_F32 || k != n || !is_device_ptr(t.data)) return nullptr;
    return static_cast<float *>(t.data);
  };
  const int NG = p.rnn ? 1 : 5;
  float *Emb = sf(p.slot_E, (int64_t)p.V * E), *Wl = p.rnn ? nullptr : sf(p.slot_Wleaf, 3LL * H * E),
        *U = sf(p.slot_U, 2LL * NG * H * H), *bb = sf(p.slot_b, (p.rnn ? 1LL : 4LL) * H),
        *Wc = sf(p.slot_Wc, (int64_t)p.C * H), *bc = sf(p.slot_bc, p.C);
  if (!Emb || (!Wl && !p.rnn) || !U || !bb || !Wc || !bc) return JANUS_ERR_INVALID;
  auto bf = [&](size_t off) { return reinterpret_cast<__nv_bfloat16 *>(W + off); };
  auto fp = [&](size_t off) { return reinterpret_cast<float *>(W + off); };
  auto ip = [&](size_t off) { return reinterpret_cast<int *>(W + off); };
  DevStatus *dst = reinterpret_cast<DevStatus *>(W + p.off.status);
  unsigned *bars = reinterpret_cast<unsigned *>(W + p.off.barriers);
  if (dp_enabled(g)) {
    janus_status r = dp_init(g);
    if (r != JANUS_OK) return r;
  }
  TreeDims d{N, B, p.V, E, H, p.C, p.Ep, p.P2, p.P5, p.P3, p.max_N, p.rnn ? 1 : 0};
  TreeSched s{ip(p.off.height), ip(p.off.order), ip(p.off.irank), ip(p.off.pslot), ip(p.off.lvl_off),
              ip(p.off.meta), ip(p.off.tree_of), ip(p.off.pcount)};
  TreeBufs t{};
  t.kind = argp[0]; t.left = argp[1]; t.right = argp[2]; t.word = argp[3]; t.off = argp[4]; t.label = argp[5];
  t.E = Emb; t.b = bb; t.Wc = Wc; t.bc = bc;
  t.x_leaf = bf(p.off.x_leaf); t.stage_h = bf(p.off.stage_h); t.stage_c = fp(p.off.stage_c);
  t.gates_int = fp(p.off.gates_int); t.c_int = fp(p.off.c_int); t.gates_leaf = fp(p.off.gates_leaf);
  t.c_leaf = fp(p.off.c_leaf); t.root_h = fp(p.off.root_h); t.dh_node = fp(p.off.dh_node);
  t.dc_node = fp(p.off.dc_node); t.DZ_int = bf(p.off.DZ_int); t.DZ_leaf = bf(p.off.DZ_leaf);
  t.gWc = fp(p.off.gWc); t.gbc = fp(p.off.gbc); t.rowloss = fp(p.off.rowloss); t.barrier = bars;
  t.bwd_lvl = bars + 64 + TREE_MAX_LEVELS * 32;
  t.dbg = g.probe;
  t.root_part = fp(p.off.root_part);

  // guards (AssertOps): forest structure + any other runtime assumption
  GuardList gl{};
  for (const auto &r : p.runtime_guards) {
    GuardDesc gd{};
    gd.kind = r.kind; gd.id = r.id; gd.value = r.value; gd.lo = r.lo; gd.hi = r.hi;
    if (r.kind != G_FORCED) {
      gd.data = argp[r.arg];
      int64_t n = 1;
      for (int k = 0; k < args[r.arg].ndim; ++k) n *= args[r.arg].shape[k];
      gd.n = n;
    }
    gl.g[gl.n++] = gd;
  }
  if (p.tree_guard) {  // observed value of a forest failure: kind[n] (node) or tree_off[t] (offset)
    GuardDesc gd{};
    gd.kind = G_TREE; gd.id = p.tree_guard_id; gd.data = argp[0]; gd.n = N; gd.data2 = argp[4];
    gl.g[gl.n++] = gd;
  }
  TCHK("init", launch_step_init_guards(dst, bars, 64, 1, gl, st));  // (the forward zeroes its level counters)
  if (p.tree_guard) TCHK("schedule", launch_tree_guard_schedule(t, d, s, p.tree_guard_id, p.V, p.max_nodes, dst, st));
  else TCHK("schedule", launch_tree_schedule(t, d, s, dst, st));
  // bf16 operand copies (R1): re-cast unless the last commit of this graph refreshed them and
  // no state-writing call came since (host.h copies_epoch; as the LM step)
  static const bool recast_env = [] { const char *e = getenv("JANUS_RECAST"); return e && e[0] == '1'; }();
  const void *srcs[9] = {U, p.rnn ? nullptr : Wl};
  bool copies_ok = !recast_env && g.copies_in && g.copies_W == W;
  for (int k = 0; k < 9; ++k) copies_ok = copies_ok && g.copies_src[k] == srcs[k];
  const bool refresh = !recast_env;
  g.copies_out = refresh;
  g.copies_W = W;
  for (int k = 0; k < 9; ++k) g.copies_src[k] = srcs[k];
  if (copies_ok) {
  } else if (p.rnn) {  // W rows and W^T (one gate: no interleave)
    TCHK("cast", launch_cast_il(U, H, 1, 2 * H, bf(p.off.U_il), p.P2, st));
    TCHK("cast_T", launch_cast_il_T(U, H, 1, 2 * H, bf(p.off.UT_il), p.P5, st));
  } else {
    TCHK("cast", launch_tree_cast3(Wl, bf(p.off.Wl_il), p.Ep, U, bf(p.off.U_il), p.P2, bf(p.off.UT_il), p.P5, H, E, st));
  }
  // one CTA per SM: the leaf level of a B=25 forest already has ~76 tiles. opts.tree_grid = n
  // (ablation only: the paper's +PARL) runs the level loops on n CTAs
  const int grid = g.opts.tree_grid > 0 ? std::min(148, g.opts.tree_grid) : 148;
  TCHK("tree_fwd", launch_tree_fwd(t, d, s, bf(p.off.Wl_il), bf(p.off.U_il), grid, dst, st));
  TCHK("root_xent", launch_tree_root(t, d, s, dst, st));
  TreeBufs tb = t;
  tb.barrier = bars + 16;  // the backward launch has its own grid-barrier counter
  TCHK("tree_bwd", launch_tree_bwd(tb, d, s, bf(p.off.UT_il), grid, dst, st));
  {
    GemmOp a;  // dU | db_int = rb(dz_int)^T [h_l h_r | 1]  (K = number of internal nodes, on device)
    a.M = NG * H; a.N = 2 * H + 1; a.K = N; a.K_dev = s.meta + 3;
    a.A = bf(p.off.DZ_int); a.lda = p.P5; a.a_mn = 1;
    a.B = bf(p.off.stage_h); a.ldb = p.P2; a.b_mn = 1;
    a.ep.C = fp(p.off.gU); a.ep.ldc = p.ldgU;

    GemmOp b2;  // dW_leaf | db_leaf = rb(dz_leaf)^T [x | 1]  (K = number of leaves)
    b2.M = 3 * H; b2.N = E + 1; b2.K = N; b2.K_dev = s.meta + 2;
    b2.A = bf(p.off.DZ_leaf); b2.lda = p.P3; b2.a_mn = 1;
    b2.B = bf(p.off.x_leaf); b2.ldb = p.Ep; b2.b_mn = 1;
    b2.ep.C = fp(p.off.gWl); b2.ep.ldc = p.ldgW;
    // one grouped launch: each GEMM alone has too few (long-K) tiles to occupy the GPU
    const GemmOp both[2] = {a, b2};
    TCHK("gemm_wgrad", gemm_bf16_group(both, p.rnn ? 1 : 2, st));  // TreeRNN: no leaf weights
  }
  if (g.nccl) {
    g.prof.mark("dp_allreduce", st);
    janus_status r = JANUS_OK;
    for (const DpSeg &sg : dp_segments(g))
      if (r == JANUS_OK) r = dp_allreduce_sum(g, fp(sg.begin), (sg.end - sg.begin) / 4, st);
    if (r != JANUS_OK) return r;
  }
  // single rank: the finalize runs as one extra block of the commit launch (below)
  if (g.nccl) TCHK("finalize", launch_finalize(fp(p.off.rowloss), B, gl, dst, g.opts.world_size, st));
  if (g.nccl) {
    janus_status r = dp_agree(g, dst, reinterpret_cast<long long *>(W + p.off.dp_scratch), st);
    if (r != JANUS_OK) return r;
  }
  // observed value of a TREE_BINARY failure: kind[n] (node) or off[t] (offset entry)
  CommitList cl{};
  auto add = [&](CommitSeg sg) { cl.s[cl.n++] = sg; };
  const float nr = (float)g.opts.world_size;
  CommitSeg sg{};
  if (p.lr_Wleaf != 0) {
    sg = {}; sg.kind = C_DENSE_IL; sg.ng = 3; sg.dst = Wl; sg.grad = fp(p.off.gWl); sg.rows = 3 * H; sg.cols = E; sg.ldg = p.ldgW; sg.H = H; sg.lr = p.lr_Wleaf / nr;
    if (refresh) { sg.bcopy = bf(p.off.Wl_il); sg.ldb = p.Ep; }
    add(sg);
  }
  if (p.lr_U != 0) {  // + the row copy and the transposed copy the backward streams
    sg = {}; sg.kind = refresh ? C_DENSE_IL_T : C_DENSE_IL; sg.ng = NG; sg.dst = U; sg.grad = fp(p.off.gU); sg.rows = NG * H; sg.cols = 2 * H; sg.ldg = p.ldgU; sg.H = H; sg.lr = p.lr_U / nr;
    if (refresh) { sg.bcopy = bf(p.off.U_il); sg.ldb = p.P2; sg.tcopy = bf(p.off.UT_il); sg.ldt = p.P5; }
    add(sg);
  }
  if (p.lr_b != 0 && p.rnn) { sg = {}; sg.kind = C_BIAS_COL; sg.dst = bb; sg.grad = fp(p.off.gU); sg.rows = H; sg.cols = 1; sg.ldg = p.ldgU; sg.col = 2 * H; sg.lr = p.lr_b / nr; add(sg); }
  if (p.lr_b != 0 && !p.rnn) { sg = {}; sg.kind = C_TREE_BIAS; sg.dst = bb; sg.grad = fp(p.off.gU); sg.ldg = p.ldgU; sg.col = 2 * H; sg.grad2 = fp(p.off.gWl); sg.ldg2 = p.ldgW; sg.col2 = E; sg.H = H; sg.lr = p.lr_b / nr; add(sg); }
  if (p.lr_Wc != 0) { sg = {}; sg.kind = C_DENSE; sg.dst = Wc; sg.grad = fp(p.off.gWc); sg.rows = p.C; sg.cols = H; sg.ldg = H; sg.lr = p.lr_Wc / nr; add(sg); }
  if (p.lr_bc != 0) { sg = {}; sg.kind = C_DENSE; sg.dst = bc; sg.grad = fp(p.off.gbc); sg.rows = 1; sg.cols = p.C; sg.ldg = p.C; sg.lr = p.lr_bc / nr; add(sg); }
  if (g.nccl) TCHK("commit", launch_commit(cl, dst, st));
  else TCHK("commit", launch_commit_finalize(cl, FinalizeArgs{fp(p.off.rowloss), B, gl}, dst, st));
  return finish(g, dst, outs, n_outs, st, fail);
}

// Null step of a data-parallel TreeLSTM rank whose DISPATCH guards failed or whose arguments were
// invalid: no compute, but the same collective sequence as a full step (arena allreduce, then the
// agreement), so its peers cannot block; its failure reaches every rank through the agreement.
janus_status run_tree_null(Graph &g, const janus_failure &f, const janus_tensor &ws, cudaStream_t st,
                           janus_failure *fail) {
  const TreePlan &p = g.tree;
  if (!ws.data || (size_t)ws.shape[0] * (ws.dtype == JANUS_U8 ? 1 : 4) < p.ws_bytes) return JANUS_ERR_INVALID;
  janus_status r = dp_init(g);
  if (r != JANUS_OK) return r;
  uint8_t *W = static_cast<uint8_t *>(ws.data);
  DevStatus *dst = reinterpret_cast<DevStatus *>(W + p.off.status);
  unsigned *bars = reinterpret_cast<unsigned *>(W + p.off.barriers);
  TCHK("init", launch_step_init(dst, bars, 64, st));
  TCHK("set_failure", launch_set_failure(dst, f.assumption_id, f.index, f.observed, st));
  for (const DpSeg &sg : dp_segments(g)) {  // the same collective sequence as a full step
    r = dp_allreduce_sum(g, reinterpret_cast<float *>(W + sg.begin), (sg.end - sg.begin) / 4, st);
    if (r != JANUS_OK) return r;
  }
  r = dp_agree(g, dst, reinterpret_cast<long long *>(W + p.off.dp_scratch), st);
  if (r != JANUS_OK) return r;
  return finish(g, dst, nullptr, 0, st, fail);
}

}  // namespace jk
