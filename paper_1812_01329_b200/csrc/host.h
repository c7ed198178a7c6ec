// host.h — host runtime of libjanus: the graph object, speculative lowering plans, dispatch.
#pragma once
#include <atomic>
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <string>
#include <vector>

#include "../../include/janus.h"
#include "fused_ar.h"
#include "step_kernels.h"

namespace jk {

// Lowered device program for the Figure 1 LSTM language model (unrolled or device While loop).
struct LmPlan {
  int V = 0, E = 0, H = 0, L = 0, B = 0;
  int T = 0;        // unrolled trip count (TRIP_COUNT) or maximum width W (While mode)
  bool while_mode = false;
  bool tag_specialised = false;  // TYPE_TAG assumed; otherwise the tag Switch runs on the device
  // `if training:` around the optimizer update: argument index of the flag (-1 = no such branch);
  // specialised by VALUE_EQ(training == 1), otherwise the commit reads the flag on the device
  int train_arg = -1;
  bool train_specialised = false;
  bool bf16 = true;              // tcgen05 path; false = single-CTA fp32 SIMT path
  // dtype of the index arguments (tokens, targets, lengths) fixed by DTYPE_EQ: JANUS_I32, or
  // JANUS_I64 (the type-specialised graph narrows them on the device first, as R10)
  int arg_dtype[3] = {JANUS_I32, JANUS_I32, JANUS_I32};
  // state slots
  int slot_E = -1, slot_Wih[4] = {-1, -1, -1, -1}, slot_Whh[4] = {-1, -1, -1, -1},
      slot_b[4] = {-1, -1, -1, -1}, slot_Wdec = -1, slot_bdec = -1;
  int slot_h[4] = {-1, -1, -1, -1}, slot_c[4] = {-1, -1, -1, -1}, slot_tag = -1;
  // learning rates (0 = parameter not updated / frozen)
  float lr_E = 0, lr_Wih[4] = {}, lr_Whh[4] = {}, lr_b[4] = {}, lr_Wdec = 0, lr_bdec = 0;
  bool write_h = false, write_tag = false;
  // dropout on the non-recurrent connections (Zaremba [51]; DROPOUT sites 0 .. L, reading R14):
  // keep probability 1 - dropout, masks from Philox4x32-10 keyed by argument key_arg (i32[2])
  float dropout = 0.f;
  int key_arg = -1;
  // device guards
  struct RG { int kind; uint32_t id; int arg; int slot; int64_t value, lo, hi; int ref_arg, ref_dim; };
  std::vector<RG> runtime_guards;
  // workspace layout (bytes)
  size_t ws_bytes = 0;
  struct Off {
    size_t status = 0, barriers = 0, stage_args = 0;
    size_t Wih_b[4], Whh_b[4], WhhT_b[4], bil[4], Wdec_b = 0, WihT_b1 = 0;
    size_t X = 0, Hs[4], Cs[4], G[4], DZ[4], dX[4], Hsw[4], DZsw[4];
    size_t Xd[5] = {0, 0, 0, 0, 0};  // dropout: masked bf16 copy of the input of layer l (1..L-1) / the decoder (L)
    size_t logits = 0, dy = 0, rowloss = 0, dHtop = 0, hT[4], cT[4];
    size_t gWih[4], gWhh[4], gWdec = 0;
    size_t seg_word = 0, seg_grad = 0, nseg = 0, ehist = 0, gflags = 0, gpart = 0;
    size_t small_ws = 0;
    size_t arena_begin = 0, arena_end = 0, dEd = 0, dp_scratch = 0;
    size_t arena_early_end = 0;  // [arena_begin, arena_early_end): dW_dec, allreduced during the backward
  } off;
  int Ep = 0, Hp = 0, Gz = 0;  // padded row pitches (elements)
  int nbar = 0;
};

// Lowered device program for the TreeLSTM (recursive InvokeOp flattened to level batches).
struct TreePlan {
  int V = 0, E = 0, H = 0, C = 0, B = 0, max_nodes = 127, max_N = 0;
  bool bf16 = true;
  bool rnn = false;  // TreeRNN cell (TREERNN_CELL; slot_U = W [H, 2H], b [H], no W_leaf)
  int arg_dtype[6] = {JANUS_I32, JANUS_I32, JANUS_I32, JANUS_I32, JANUS_I32, JANUS_I32};
  int slot_E = -1, slot_Wleaf = -1, slot_U = -1, slot_b = -1, slot_Wc = -1, slot_bc = -1;
  float lr_Wleaf = 0, lr_U = 0, lr_b = 0, lr_Wc = 0, lr_bc = 0;
  uint32_t tree_guard_id = 0;
  bool tree_guard = false;
  std::vector<LmPlan::RG> runtime_guards;
  size_t ws_bytes = 0;
  int Ep = 0, P2 = 0, P5 = 0, P3 = 0, ldgU = 0, ldgW = 0;  // row pitches (elements)
  struct Off {
    size_t status = 0, barriers = 0, stage_args = 0;
    size_t height = 0, order = 0, irank = 0, pslot = 0, tree_of = 0, pcount = 0, lvl_off = 0, meta = 0;
    size_t x_leaf = 0, stage_h = 0, stage_c = 0, gates_int = 0, c_int = 0, gates_leaf = 0, c_leaf = 0;
    size_t root_part = 0;
    size_t root_h = 0, dh_node = 0, dc_node = 0, DZ_int = 0, DZ_leaf = 0, rowloss = 0;
    size_t U_il = 0, UT_il = 0, Wl_il = 0;
    size_t arena_begin = 0, arena_end = 0, gU = 0, gWl = 0, gWc = 0, gbc = 0, dp_scratch = 0;
  } off;
};

// Optional per-phase device timing: a CUDA event is recorded on the launch stream before every
// phase; after the step's single synchronisation the gaps are accumulated per phase name.
struct PhaseProf {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  std::vector<std::string> pending;  // phase name per recorded event ("" = end marker)
  std::map<std::string, std::pair<double, long>> acc;  // name -> (total ms, launches)
  void mark(const char *name, cudaStream_t st) {
    if (!on) return;
    if (pending.size() == pool.size()) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) { on = false; return; }
      pool.push_back(e);
    }
    cudaEventRecord(pool[pending.size()], st);
    pending.push_back(name ? name : "");
  }
  void collect() {
    if (!on) { pending.clear(); return; }
    for (size_t i = 0; i + 1 < pending.size(); ++i) {
      if (pending[i].empty()) continue;
      float ms = 0;
      cudaEventElapsedTime(&ms, pool[i], pool[i + 1]);
      auto &a = acc[pending[i]];
      a.first += ms;
      a.second += 1;
    }
    pending.clear();
  }
  ~PhaseProf() {
    for (auto e : pool) cudaEventDestroy(e);
  }
};

// Identity of a captured step: the same workspace, state tensors, batch width and stream replay
// the same graph (every argument is staged into fixed workspace slots first).
struct GraphKey {
  const void *W = nullptr;
  const void *state[64] = {};
  int width = 0;
  const void *stream = nullptr;
  bool cast = true;  // the step re-casts the bf16 operand copies (false: the last commit refreshed them)
  bool operator==(const GraphKey &o) const {
    if (W != o.W || width != o.width || stream != o.stream || cast != o.cast) return false;
    for (int k = 0; k < 64; ++k)
      if (state[k] != o.state[k]) return false;
    return true;
  }
};
struct StepGraph {
  void *exec = nullptr;  // cudaGraphExec_t
  GraphKey key;
  uint64_t kernels = 0;  // launches one replay stands for
  bool seen = false;     // a direct run with seen_key happened: the next one captures
  GraphKey seen_key;
  bool failed = false;   // capture not possible: direct launches only
  void reset() {
    if (exec) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(exec));
    exec = nullptr;
  }
};

struct Graph {
  PhaseProf prof;
  std::vector<janus_op> ops;
  std::vector<janus_assumption> asms;
  janus_build_opts opts{};
  int n_args = 0, n_state = 0;
  std::string kind;  // "lstm_lm" | "treelstm" | "" (no device lowering)
  std::string unsupported_reason;
  LmPlan lm;
  TreePlan tree;
  size_t ws_bytes = 0;       // max over graph path and imperative path
  size_t imp_ws_bytes = 0;
  // counters
  uint64_t launches = 0, host_syncs = 0, aborts = 0;
  // pinned status readback
  DevStatus *h_status = nullptr;
  void *nccl = nullptr;  // ncclComm_t when world_size > 1
  void *nccl2 = nullptr; // second communicator (split) for the collective that overlaps the backward
  cudaStream_t side = nullptr;             // stream of the overlapped collective
  cudaStream_t bk_side = nullptr;          // single-rank LM: the embedding-gradient bucketing beside the forward
  cudaEvent_t ev_bk_fork = nullptr, ev_bk_join = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool dp = false;       // data-parallel collectives in the step (fixed at build)
  bool fused_ar = false; // NEXT-3: weight gradients reduced in the wgrad GEMM epilogue (fixed at build)
  FusedArena far;        // its NCCL symmetric windows (created with the communicator)
  // protocol-test transport (janus_dev_dp_set_host_collective): host buffers, caller's allreduce
  int32_t (*host_coll)(void *ctx, void *buf, int64_t count, int32_t dtype, int32_t op) = nullptr;
  void *host_coll_ctx = nullptr;
  std::string describe;
  const void *gflags_ws = nullptr;        // workspace whose split-K counters were zeroed
  // workspace the device program last initialised (zero-filled on first use by janus_run; the
  // imperative executor writes anywhere in it, so running it on the same buffer clears this)
  const void *ws_ready = nullptr;
  unsigned long long *probe = nullptr;  // dev hook: recurrent-kernel timeline buffer (2*128*16*T u64)
  StepGraph cg;                         // the LM step captured as one CUDA graph (host_lm.cpp)
  // bf16 operand copies (R1) kept current by the commit: valid for the next run when no library
  // call that may write state (any graph, the imperative executor) and no janus_state_changed
  // happened since this graph's last run, on the same workspace and the same master pointers
  unsigned long long copies_epoch = ~0ull;  // state_epoch value after the run that left them valid
  bool copies_in = false;                   // set by janus_run for run_lm: the copies match the masters
  bool copies_out = false;                  // set by run_lm: the enqueued step leaves them matching
  const void *copies_W = nullptr;
  const void *copies_src[9] = {};
};

// bumped by every library call that may write a state tensor, and by janus_state_changed
extern std::atomic<unsigned long long> state_epoch;

// host_graph.cpp
janus_status validate_graph(Graph &g, std::string &err);
bool check_dispatch(const Graph &g, const janus_tensor *args, int n_args, janus_failure *fail);

// host_lm.cpp
bool lower_lm(Graph &g, std::string &why);
janus_status run_lm(Graph &g, const janus_tensor *args, const janus_tensor *state,
                    const janus_tensor *outs, int n_outs, const janus_tensor &ws,
                    cudaStream_t st, janus_failure *fail);

// host_tree.cpp
bool lower_tree(Graph &g, std::string &why);
janus_status run_tree(Graph &g, const janus_tensor *args, int n_args, const janus_tensor *state,
                      const janus_tensor *outs, int n_outs, const janus_tensor &ws,
                      cudaStream_t st, janus_failure *fail);

// host_imperative.cpp
size_t imperative_ws_bytes(const Graph &g);
janus_status run_imperative(Graph &g, const janus_tensor *args, int n_args,
                            const janus_tensor *state, int n_state, const janus_tensor *outs,
                            int n_outs, const janus_tensor &ws, cudaStream_t st);

// host_dp.cpp: NCCL data parallelism
bool dp_enabled(const Graph &g);
bool dp_wanted(const janus_build_opts &o);  // decided once, at build time
janus_status dp_init(Graph &g);
void dp_destroy(Graph &g);
janus_status dp_allreduce_sum(Graph &g, float *buf, size_t n, cudaStream_t st);
// the same on the second communicator (issued on the side stream by the step, on the launch
// stream by a null step — the per-communicator order is the same on every rank)
janus_status dp_allreduce_sum2(Graph &g, float *buf, size_t n, cudaStream_t st);
bool dp_overlap(const Graph &g);  // the backward's early allreduce is in use
// The step's gradient-arena allreduces in issue order (identical on every rank and for the null
// step): comm 1 = the main communicator on the launch stream, comm 2 = the split communicator
// (issued on the side stream, overlapping the backward, by a full step). Byte offsets into the
// workspace.
enum { DP_OP_SUM = 0, DP_OP_MIN = 1, DP_OP_MAX = 2 };  // janus_allreduce_fn ops
struct DpSeg {
  int comm;
  size_t begin, end;
};
std::vector<DpSeg> dp_segments(const Graph &g);
janus_status dp_agree(Graph &g, DevStatus *st_dev, long long *scratch, cudaStream_t st);
// a data-parallel rank whose DISPATCH guards failed still joins every collective (null step)
janus_status run_lm_null(Graph &g, const janus_failure &f, const janus_tensor &ws, cudaStream_t st,
                         janus_failure *fail);
janus_status run_tree_null(Graph &g, const janus_failure &f, const janus_tensor &ws, cudaStream_t st,
                           janus_failure *fail);
constexpr uint32_t NULL_STEP_INVALID_ARGS = 0xffffffffu;  // failure id of a rank with invalid arguments

// one D2H of the status word + stream sync; decodes the failure (host_lm.cpp)
janus_status finish(Graph &g, DevStatus *dst, const janus_tensor *outs, int n_outs,
                    cudaStream_t st, janus_failure *fail);

// helpers
int producer_origin(const Graph &g, int node);     // follows Enter/Identity/Switch/Merge(in0)
const janus_op &op_at(const Graph &g, int node);
janus_status cuda_status(cudaError_t e);
bool is_device_ptr(const void *p);

}  // namespace jk

// the opaque handle of janus.h is the host graph object
struct janus_graph : public jk::Graph {};
