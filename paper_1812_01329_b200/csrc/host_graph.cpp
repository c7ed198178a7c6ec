// host_graph.cpp — C ABI entry points (include/janus.h), structural validation of the op list
// (arity, ports, no cycles except through NextIteration, unique effect sequence
// numbers), DISPATCH assumption checks at graph lookup and the lowering dispatch.
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <functional>
#include <set>
#include <string>

#include "host.h"
#include "../../include/janus_dev.h"
#include "lm_rec.h"

#define TREE_MAX_LEVELS_HOST 130  // tree.h TREE_MAX_LEVELS

namespace jk {

std::atomic<unsigned long long> state_epoch{0};

static int arity(int k) {
  switch (k) {
    case JOP_ARG: case JOP_CONST: case JOP_STATE_READ: case JOP_TA_NEW: return 0;
    case JOP_STATE_WRITE: case JOP_OUTPUT: case JOP_MAX_REDUCE: case JOP_LEN: case JOP_SUM: case JOP_ZEROS_LIKE:
    case JOP_TA_STACK: case JOP_ENTER: case JOP_EXIT: case JOP_NEXT_ITERATION: case JOP_LOOP_COND:
    case JOP_IDENTITY: case JOP_SGD_APPLY: return 1;
    case JOP_ADD: case JOP_LESS: case JOP_EQ: case JOP_COLUMN: case JOP_ELEMENT: case JOP_EMBEDDING:
    case JOP_SEQ_MASK: case JOP_TIME_MAJOR: case JOP_SWITCH: return 2;
    case JOP_LINEAR: case JOP_TREELSTM_LEAF: case JOP_SOFTMAX_XENT: case JOP_TA_WRITE: case JOP_DROPOUT: return 3;
    case JOP_TREERNN_CELL: return 4;
    case JOP_TREELSTM_CELL: return 6;
    case JOP_LSTM_CELL: return 7;
    case JOP_MERGE: return -2;   // >= 2
    default: return -1;          // INVOKE, RETURN: any
  }
}

static int n_ports(const Graph &g, int node) {
  const janus_op &o = g.ops[node];
  switch (o.kind) {
    case JOP_SWITCH: case JOP_MERGE: case JOP_LSTM_CELL: case JOP_TREELSTM_LEAF:
    case JOP_TREELSTM_CELL: return 2;
    case JOP_STATE_WRITE: case JOP_OUTPUT: case JOP_SGD_APPLY: case JOP_RETURN: return 0;
    case JOP_INVOKE: {
      for (const auto &r : g.ops)
        if (r.kind == JOP_RETURN && r.func == (int)o.iattr[0]) return r.n_in;
      return 0;
    }
    default: return 1;
  }
}

const janus_op &op_at(const Graph &g, int node) { return g.ops[node]; }

int producer_origin(const Graph &g, int node) {
  for (int guard = 0; guard < 64 && node >= 0; ++guard) {
    const janus_op &o = g.ops[node];
    if (o.kind == JOP_ENTER || o.kind == JOP_IDENTITY || o.kind == JOP_SWITCH || o.kind == JOP_MERGE ||
        o.kind == JOP_LOOP_COND || o.kind == JOP_EXIT)
      node = o.in_node[0];
    else
      return node;
  }
  return node;
}

janus_status cuda_status(cudaError_t e) { return e == cudaSuccess ? JANUS_OK : JANUS_ERR_CUDA; }

bool is_device_ptr(const void *p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

janus_status validate_graph(Graph &g, std::string &err) {
  const int n = (int)g.ops.size();
  char buf[256];
  std::set<int64_t> seqs;
  std::set<uint32_t> aids;
  int max_arg = -1, max_slot = -1;
  for (int i = 0; i < n; ++i) {
    const janus_op &o = g.ops[i];
    if (o.kind < 0 || o.kind >= JOP__COUNT) {
      snprintf(buf, sizeof buf, "node %d: unknown op kind %d", i, o.kind);
      err = buf;
      return JANUS_ERR_INVALID;
    }
    const int a = arity(o.kind);
    if (o.n_in < 0 || o.n_in > JANUS_MAX_IN || (a >= 0 && o.n_in != a) || (a == -2 && o.n_in < 2)) {
      snprintf(buf, sizeof buf, "node %d (kind %d): bad arity %d", i, o.kind, o.n_in);
      err = buf;
      return JANUS_ERR_INVALID;
    }
    for (int k = 0; k < o.n_in; ++k) {
      const int p = o.in_node[k];
      if (p < 0 || p >= n || g.ops[p].func != o.func || o.in_port[k] < 0 ||
          o.in_port[k] >= n_ports(g, p)) {
        snprintf(buf, sizeof buf, "node %d input %d: bad producer (%d, port %d)", i, k, p, o.in_port[k]);
        err = buf;
        return JANUS_ERR_INVALID;
      }
    }
    if (o.kind == JOP_ARG && o.func == 0) max_arg = std::max(max_arg, (int)o.iattr[0]);
    if (o.kind == JOP_STATE_READ || o.kind == JOP_STATE_WRITE || o.kind == JOP_SGD_APPLY)
      max_slot = std::max(max_slot, (int)o.iattr[0]);
    if (o.kind == JOP_STATE_WRITE || o.kind == JOP_SGD_APPLY) {
      if (!seqs.insert(o.iattr[1]).second) {
        snprintf(buf, sizeof buf, "node %d: duplicate effect sequence number %lld", i, (long long)o.iattr[1]);
        err = buf;
        return JANUS_ERR_INVALID;
      }
    }
    if (o.kind == JOP_ENTER && o.iattr[0] <= 0) {
      snprintf(buf, sizeof buf, "node %d: Enter frame id must be > 0", i);
      err = buf;
      return JANUS_ERR_INVALID;
    }
    if (o.kind == JOP_INVOKE) {
      bool found = false;
      for (const auto &r : g.ops) found |= (r.kind == JOP_RETURN && r.func == (int)o.iattr[0]);
      if (!found || o.iattr[0] <= 0) {
        snprintf(buf, sizeof buf, "node %d: Invoke of unknown function %lld", i, (long long)o.iattr[0]);
        err = buf;
        return JANUS_ERR_INVALID;
      }
    }
  }
  // data edges must be acyclic except through NextIteration (tagged-frame back edges)
  std::vector<int> state(n, 0);
  std::function<bool(int)> dfs = [&](int v) -> bool {
    state[v] = 1;
    const janus_op &o = g.ops[v];
    for (int k = 0; k < o.n_in; ++k) {
      const int p = o.in_node[k];
      if (g.ops[p].kind == JOP_NEXT_ITERATION) continue;
      if (state[p] == 1) return false;
      if (state[p] == 0 && !dfs(p)) return false;
    }
    state[v] = 2;
    return true;
  };
  for (int i = 0; i < n; ++i)
    if (state[i] == 0 && !dfs(i)) {
      err = "data-edge cycle not passing through NextIteration";
      return JANUS_ERR_INVALID;
    }
  for (const auto &a : g.asms) {
    if (!aids.insert(a.id).second) {
      snprintf(buf, sizeof buf, "duplicate assumption id %u", a.id);
      err = buf;
      return JANUS_ERR_INVALID;
    }
    if (a.kind < JA_DTYPE_EQ || a.kind > JA_BRANCH_ARM || (a.mode != 0 && a.mode != 1)) {
      snprintf(buf, sizeof buf, "assumption %u: bad kind/mode", a.id);
      err = buf;
      return JANUS_ERR_INVALID;
    }
    if (a.id >= 0xffffu) {  // the data-parallel agreement packs the id into 16 bits
      snprintf(buf, sizeof buf, "assumption id %u: ids must be < 65535", a.id);
      err = buf;
      return JANUS_ERR_INVALID;
    }
    if (a.kind == JA_SHAPE_MATCH && (a.ndim < 0 || a.ndim > 4)) {
      snprintf(buf, sizeof buf, "assumption %u: SHAPE_MATCH ndim %d outside [0, 4]", a.id, a.ndim);
      err = buf;
      return JANUS_ERR_INVALID;
    }
    if (a.mode == JANUS_MODE_DISPATCH && a.kind != JA_DTYPE_EQ && a.kind != JA_SHAPE_MATCH) {
      snprintf(buf, sizeof buf, "assumption %u: only DTYPE_EQ/SHAPE_MATCH are dispatch-checkable", a.id);
      err = buf;
      return JANUS_ERR_INVALID;
    }
  }
  g.n_args = max_arg + 1;
  g.n_state = max_slot + 1;
  return JANUS_OK;
}

// DISPATCH assumptions on tensor metadata, ascending id. No device access.
bool check_dispatch(const Graph &g, const janus_tensor *args, int n_args, janus_failure *fail) {
  std::vector<const janus_assumption *> v;
  for (const auto &a : g.asms)
    if (a.mode == JANUS_MODE_DISPATCH) v.push_back(&a);
  std::sort(v.begin(), v.end(), [](auto *x, auto *y) { return x->id < y->id; });
  const bool forced_dispatch = [&] {
    for (auto *a : v) if ((int)a->id == g.opts.fail_assert_id) return true;
    return false;
  }();
  for (auto *a : v) {
    if (a->target < 0 || a->target >= n_args) {
      *fail = {a->id, g.opts.rank, -1, -1};
      return false;
    }
    const janus_tensor &t = args[a->target];
    if (a->kind == JA_DTYPE_EQ) {
      if (t.dtype != a->dtype) {
        *fail = {a->id, g.opts.rank, -1, t.dtype};
        return false;
      }
    } else if (a->kind == JA_SHAPE_MATCH) {
      if (t.ndim != a->ndim) {
        *fail = {a->id, g.opts.rank, -1, t.ndim};
        return false;
      }
      for (int k = 0; k < a->ndim; ++k)
        if (a->dims[k] != -1 && a->dims[k] != t.shape[k]) {
          *fail = {a->id, g.opts.rank, k, t.shape[k]};
          return false;
        }
    }
  }
  if (forced_dispatch) {
    *fail = {(uint32_t)g.opts.fail_assert_id, g.opts.rank, -1, -1};
    return false;
  }
  return true;
}

}  // namespace jk

using namespace jk;


extern "C" {

int32_t janus_abi_version(void) { return JANUS_ABI_VERSION; }

const char *janus_status_str(janus_status s) {
  switch (s) {
    case JANUS_OK: return "OK";
    case JANUS_ASSUMPTION_FAILED: return "ASSUMPTION_FAILED";
    case JANUS_ERR_INVALID: return "ERR_INVALID";
    case JANUS_ERR_UNSUPPORTED: return "ERR_UNSUPPORTED";
    case JANUS_ERR_RUNTIME: return "ERR_RUNTIME";
    case JANUS_ERR_CUDA: return "ERR_CUDA";
    case JANUS_ERR_NCCL: return "ERR_NCCL";
    case JANUS_ERR_WORKSPACE: return "ERR_WORKSPACE";
  }
  return "UNKNOWN";
}

static void set_err(char *err, size_t len, const std::string &m) {
  if (err && len) {
    strncpy(err, m.c_str(), len - 1);
    err[len - 1] = 0;
  }
}

janus_status janus_graph_build(const janus_op *ops, int32_t n_ops, const janus_assumption *asms,
                               int32_t n_asms, const janus_build_opts *opts, janus_graph **out,
                               char *err, size_t err_len) {
  if (!out || (!ops && n_ops) || (!asms && n_asms) || n_ops < 0 || n_asms < 0) {
    set_err(err, err_len, "null argument");
    return JANUS_ERR_INVALID;
  }
  *out = nullptr;
  janus_graph *g = new janus_graph();
  g->ops.assign(ops, ops + n_ops);
  g->asms.assign(asms, asms + n_asms);
  if (opts) g->opts = *opts;
  else {
    g->opts.world_size = 1;
    g->opts.gemm_dtype = JANUS_BF16;
    g->opts.fail_assert_id = -1;
  }
  if (g->opts.world_size < 1) g->opts.world_size = 1;
  std::string e;
  janus_status s = validate_graph(*g, e);
  if (s != JANUS_OK) {
    set_err(err, err_len, e);
    delete g;
    return s;
  }
  g->dp = dp_wanted(g->opts);
  std::string why_lm, why_tree;
  if (lower_lm(*g, why_lm)) {
    g->kind = "lstm_lm";
    const LmPlan &p = g->lm;  // the fused reduction rides on the grouped weight-gradient launch
    g->fused_ar = g->dp && g->opts.fused_allreduce && p.bf16 && p.L == 2 && p.B <= 64 && p.key_arg < 0 &&
                  !g->opts.serial_layers && rec_bwd_wf_grid(p.H) <= 148;
  }
  else if (lower_tree(*g, why_tree)) g->kind = "treelstm";
  else g->unsupported_reason = "lstm_lm: " + why_lm + "; treelstm: " + why_tree;
  g->imp_ws_bytes = imperative_ws_bytes(*g);
  size_t plan = g->kind == "lstm_lm" ? g->lm.ws_bytes : g->kind == "treelstm" ? g->tree.ws_bytes : 0;
  g->ws_bytes = std::max(plan, g->imp_ws_bytes);
  *out = g;  // pinned status buffer is allocated lazily on the first run (build needs no GPU)
  if (g->kind.empty()) {
    set_err(err, err_len, g->unsupported_reason);
    return JANUS_ERR_UNSUPPORTED;
  }
  return JANUS_OK;
}

janus_status janus_workspace_bytes(const janus_graph *g, size_t *bytes) {
  if (!g || !bytes) return JANUS_ERR_INVALID;
  *bytes = g->ws_bytes;
  return JANUS_OK;
}

janus_status janus_run(janus_graph *g, const janus_tensor *args, int32_t n_args,
                       const janus_tensor *state, int32_t n_state, const janus_tensor *outs,
                       int32_t n_outs, janus_tensor workspace, void *cuda_stream,
                       janus_failure *fail) {
  if (!g || (!args && n_args) || (!state && n_state)) return JANUS_ERR_INVALID;
  if (g->kind.empty()) return JANUS_ERR_UNSUPPORTED;
  if (n_args < g->n_args || n_state < g->n_state) return JANUS_ERR_INVALID;
  janus_failure f{};
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  // the bf16 operand copies the last commit refreshed are current iff no state-writing call
  // (this one excepted) happened since (host.h copies_epoch)
  const unsigned long long e0 = state_epoch.fetch_add(1);
  g->copies_in = e0 == g->copies_epoch;
  g->copies_out = false;
  g->copies_epoch = ~0ull;
  // a workspace this graph has not initialised (new, or written by the imperative executor or
  // another graph since) is zero-filled first: the device program relies on zero pads
  auto ready = [&]() -> janus_status {
    if (g->ws_ready == workspace.data) return JANUS_OK;
    const size_t have = (size_t)workspace.shape[0] * (workspace.dtype == JANUS_U8 ? 1 : 4);
    if (!workspace.data || have < g->ws_bytes) return JANUS_ERR_INVALID;
    if (cudaMemsetAsync(workspace.data, 0, g->ws_bytes, st) != cudaSuccess) return JANUS_ERR_CUDA;
    g->gflags_ws = nullptr;
    g->copies_in = false;
    g->ws_ready = workspace.data;
    return JANUS_OK;
  };
  // data parallel: a rank that cannot run the step still joins its collectives (null step, the
  // same sequence as a full step) so its peers cannot block; the failure reaches every rank
  // through the agreement (reading Q12)
  const bool dp_null = dp_enabled(*g) && (g->kind == "treelstm" || g->lm.bf16);
  auto null_step = [&](const janus_failure &nf) -> janus_status {
    janus_status r = ready();
    if (r != JANUS_OK) return r;
    return g->kind == "lstm_lm" ? run_lm_null(*g, nf, workspace, st, fail)
                                : run_tree_null(*g, nf, workspace, st, fail);
  };
  if (!check_dispatch(*g, args, n_args, &f)) {
    g->aborts++;
    if (dp_null) {
      const janus_status r = null_step(f);
      return r == JANUS_OK ? JANUS_ASSUMPTION_FAILED : r;
    }
    // cache miss: nothing is launched, nothing mutated
    if (g->copies_in) g->copies_epoch = e0 + 1;
    if (fail) *fail = f;
    return JANUS_ASSUMPTION_FAILED;
  }
  janus_status r = ready();
  if (r != JANUS_OK) return r;
  if (g->kind == "lstm_lm") r = run_lm(*g, args, state, outs, n_outs, workspace, st, fail);
  else r = run_tree(*g, args, n_args, state, outs, n_outs, workspace, st, fail);
  if (r == JANUS_ERR_INVALID && dp_null) {
    // argument validation failed on this rank before any collective was issued
    janus_failure nf{NULL_STEP_INVALID_ARGS, g->opts.rank, -1, -1};
    const janus_status rn = null_step(nf);
    return rn == JANUS_OK || rn == JANUS_ERR_RUNTIME ? JANUS_ERR_INVALID : rn;
  }
  if (r == JANUS_ASSUMPTION_FAILED) g->aborts++;
  // the commit kept the copies current, or nothing committed (all-or-nothing)
  if (g->copies_out && (r == JANUS_OK || r == JANUS_ASSUMPTION_FAILED || r == JANUS_ERR_RUNTIME))
    g->copies_epoch = e0 + 1;
  return r;
}

janus_status janus_state_changed(void) {
  state_epoch.fetch_add(1);
  return JANUS_OK;
}

janus_status janus_run_imperative(janus_graph *g, const janus_tensor *args, int32_t n_args,
                                  const janus_tensor *state, int32_t n_state,
                                  const janus_tensor *outs, int32_t n_outs,
                                  janus_tensor workspace, void *cuda_stream) {
  if (!g || (!args && n_args) || (!state && n_state)) return JANUS_ERR_INVALID;
  if (g->ws_ready == workspace.data) g->ws_ready = nullptr;
  state_epoch.fetch_add(1);
  return run_imperative(*g, args, n_args, state, n_state, outs, n_outs, workspace,
                        static_cast<cudaStream_t>(cuda_stream));
}

janus_status janus_counters(const janus_graph *g, uint64_t *launches, uint64_t *host_syncs,
                            uint64_t *aborts) {
  if (!g) return JANUS_ERR_INVALID;
  if (launches) *launches = g->launches;
  if (host_syncs) *host_syncs = g->host_syncs;
  if (aborts) *aborts = g->aborts;
  return JANUS_OK;
}

janus_status janus_describe(const janus_graph *g, char *buf, size_t buf_len) {
  if (!g || !buf || !buf_len) return JANUS_ERR_INVALID;
  std::string d = g->kind.empty() ? "no device program: " + g->unsupported_reason : g->describe;
  set_err(buf, buf_len, d);
  return JANUS_OK;
}

/* dev hooks (include/janus_dev.h) */
int32_t janus_dev_set_probe(janus_graph *g, void *dev_buf) {
  if (!g) return -1;
  g->probe = static_cast<unsigned long long *>(dev_buf);
  return 0;
}

/* named workspace regions (tests compare device-internal integer results bit-exactly) */
int32_t janus_dev_workspace_region(const janus_graph *g, const char *name, size_t *offset,
                                   size_t *bytes) {
  if (!g || !name || !offset || !bytes) return -1;
  const std::string n(name);
  const TreePlan &t = g->tree;
  const size_t N = (size_t)t.max_N * 4;
  struct R { const char *k; size_t off, len; } rs[] = {
      {"tree.height", t.off.height, N},   {"tree.order", t.off.order, N},
      {"tree.irank", t.off.irank, N},     {"tree.pslot", t.off.pslot, N},
      {"tree.lvl_off", t.off.lvl_off, (TREE_MAX_LEVELS_HOST + 2) * 4},
      {"tree.meta", t.off.meta, 16},      {"status", g->kind == "treelstm" ? t.off.status : g->lm.off.status, sizeof(DevStatus)},
      {"tree.dh_node", t.off.dh_node, (size_t)t.max_N * t.H * 4},
      {"tree.dc_node", t.off.dc_node, (size_t)t.max_N * t.H * 4},
      {"tree.root_h", t.off.root_h, (size_t)t.B * t.H * 4},
  };
  for (const auto &r : rs)
    if (n == r.k && (g->kind == "treelstm" || n == "status")) {
      *offset = r.off;
      *bytes = r.len;
      return 0;
    }
  if (g->kind == "treelstm") {  // gradient arena members (fp32, padded pitches)
    struct R2 { const char *k; size_t off, len; } ts[] = {
        {"tree.gU", t.off.gU, (size_t)5 * t.H * t.ldgU * 4}, {"tree.gWl", t.off.gWl, (size_t)3 * t.H * t.ldgW * 4},
        {"tree.gWc", t.off.gWc, (size_t)t.C * t.H * 4},     {"tree.gbc", t.off.gbc, (size_t)t.C * 4},
        {"arena", t.off.arena_begin, t.off.arena_end - t.off.arena_begin}};
    for (const auto &r : ts)
      if (n == r.k) { *offset = r.off; *bytes = r.len; return 0; }
  }
  if (g->kind == "lstm_lm" && g->lm.bf16) {
    const LmPlan &p = g->lm;
    const size_t G4 = (size_t)4 * p.H;
    if (n == "arena") { *offset = p.off.arena_begin; *bytes = p.off.arena_end - p.off.arena_begin; return 0; }
    if (n == "lm.gWdec") { *offset = p.off.gWdec; *bytes = (size_t)p.V * p.Hp * 4; return 0; }
    if (n == "lm.dEd" && p.off.dEd) { *offset = p.off.dEd; *bytes = (size_t)p.V * p.E * 4; return 0; }
    for (int l = 0; l < p.L; ++l) {
      const std::string sl = std::to_string(l);
      if (n == "lm.gWih" + sl) { *offset = p.off.gWih[l]; *bytes = G4 * (l ? p.Hp : p.Ep) * 4; return 0; }
      if (n == "lm.gWhh" + sl) { *offset = p.off.gWhh[l]; *bytes = G4 * p.Hp * 4; return 0; }
    }
  }
  return -1;
}

/* per-phase device timing */
int32_t janus_dev_profile(janus_graph *g, int32_t enable) {
  if (!g) return -1;
  g->prof.on = enable != 0;
  g->prof.acc.clear();
  return 0;
}

int32_t janus_dev_phase_report(const janus_graph *g, char *buf, size_t len) {
  if (!g || !buf || !len) return -1;
  std::string r;
  char tmp[160];
  for (const auto &kv : g->prof.acc) {
    snprintf(tmp, sizeof tmp, "%s:%.6f:%ld;", kv.first.c_str(), kv.second.first, kv.second.second);
    r += tmp;
  }
  set_err(buf, len, r);
  return (int32_t)g->prof.acc.size();
}

void janus_graph_destroy(janus_graph *g) {
  if (!g) return;
  g->cg.reset();
  dp_destroy(*g);
  if (g->bk_side) {
    cudaStreamSynchronize(g->bk_side);
    cudaStreamDestroy(g->bk_side);
  }
  if (g->ev_bk_fork) cudaEventDestroy(g->ev_bk_fork);
  if (g->ev_bk_join) cudaEventDestroy(g->ev_bk_join);
  if (g->h_status) cudaFreeHost(g->h_status);
  delete g;
}

}  // extern "C"
