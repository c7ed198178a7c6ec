/*
 * janus.h — C ABI of the B200-native speculative-graph executor (JANUS, arXiv 1812.01329).
 *
 * The library executes the *speculatively specialised* symbolic dataflow graph of an imperative
 * DL training step on one B200 (§2.3 "generates a symbolic graph tailored for the
 * assumptions"; §3.1 "the Speculative Graph Executor executes the symbolic graph"), checks
 * the assumptions on the device (§3.2 AssertOp), commits state all-or-nothing
 * (§3.2; §4.2.3) and offers the imperative per-op GPU executor as the fallback
 * (§3.2, Figure 2 (E)).
 *
 * Citations: P:NNN = line of the paper text, S:NNN = line of SPEC.md.
 *
 * Conventions
 *  - Every pointer argument is BORROWED for the duration of the call unless stated otherwise.
 *  - janus_tensor.data may point to device memory (normal case) or, for `args` and `outs` only,
 *    to host memory: the library then stages the bytes through the workspace (H2D before the
 *    step, D2H after), inside the same call. State tensors and the workspace must be device memory.
 *  - Strides are in elements. Every tensor passed to janus_run must be contiguous (row-major).
 *  - No call allocates device memory. The caller (PyTorch caching allocator) owns args, state,
 *    outs and the workspace; the graph object owns host metadata only.
 *  - Errors: every call returns a janus_status. JANUS_ERR_* codes never leave state modified.
 */
#ifndef JANUS_H
#define JANUS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define JANUS_ABI_VERSION 1

/* ---------------------------------------------------------------------------------------------
 * Status codes. ASSUMPTION_FAILED is the AssertOp abort of P:168 ("aborts the graph execution if
 * the given condition fails. It also reports which assumption has been broken"). ERR_RUNTIME is a
 * runtime error inside a pure node (index out of range), reported distinctly from an assumption
 * failure as in S:429; it also commits nothing.
 * ------------------------------------------------------------------------------------------- */
typedef enum {
  JANUS_OK = 0,
  JANUS_ASSUMPTION_FAILED = 1,
  JANUS_ERR_INVALID = 2,      /* malformed op list / bad arguments (text in err buffer)      */
  JANUS_ERR_UNSUPPORTED = 3,  /* graph valid but the device path cannot run it exactly       */
  JANUS_ERR_RUNTIME = 4,      /* runtime error in a node (bad token id, bad child id)         */
  JANUS_ERR_CUDA = 5,
  JANUS_ERR_NCCL = 6,
  JANUS_ERR_WORKSPACE = 7     /* janus_session_step: workspace smaller than the dispatched
                                 graph needs; nothing ran (required bytes in the step info) */
} janus_status;

typedef enum { JANUS_F32 = 0, JANUS_BF16 = 1, JANUS_I32 = 2, JANUS_I64 = 3, JANUS_U8 = 4 } janus_dtype;

typedef struct {
  void *data;         /* device pointer (or host pointer for args/outs, see conventions) */
  int32_t dtype;      /* janus_dtype */
  int32_t ndim;       /* 0..4 */
  int64_t shape[4];
  int64_t stride[4];  /* elements; must describe a contiguous row-major tensor */
} janus_tensor;

/* ---------------------------------------------------------------------------------------------
 * Op kinds of the symbolic graph. A graph is an array of janus_op; a node is referenced by its
 * index in that array. The graph vocabulary follows the paper's conversion rules:
 *   ARG = PlaceholderOp for input parameters; CONST = ConstantOp for literals;
 *   STATE_READ/STATE_WRITE = PyGetAttrOp/PySetAttrOp with local copies (Figure 5);
 *   SWITCH/MERGE = `if`; ENTER/EXIT/NEXT_ITERATION/LOOP_COND = `while`/`for` frames
 *   (P:222); INVOKE = function call / recursion (InvokeOp); the whitelisted framework
 *   functions are EMBEDDING, LINEAR, LSTM_CELL, TREELSTM_LEAF, TREELSTM_CELL, TREERNN_CELL,
 *   SOFTMAX_XENT; SGD_APPLY is the automatically inserted differentiation + parameter update
 *    and, being a state mutation, is deferred until all assumptions hold.
 *
 * Port conventions: SWITCH output port 0 = false branch, port 1 = true branch (TF SwitchOp).
 * MERGE output port 0 = value, port 1 = index of the live input. LSTM_CELL/TREELSTM_* output
 * port 0 = h, port 1 = c.
 *
 * Attribute table (iattr[k] / fattr[k]); "scalar" means an int32 or f32 0-d value:
 *   ARG            iattr0 = argument index
 *   CONST          iattr0 = dtype (JANUS_I32 | JANUS_F32); scalar value in fattr0
 *   STATE_READ     iattr0 = state slot, iattr1 = dtype, iattr2 = ndim, iattr3..6 = dims
 *   STATE_WRITE    in0 = value; iattr0 = state slot, iattr1 = effect sequence number
 *   OUTPUT         in0 = value; iattr0 = output index
 *   ADD, LESS, EQ  in0, in1 (scalar ∘ scalar, or scalar ∘ vector elementwise; LESS/EQ give int32)
 *   MAX_REDUCE     in0 int32 vector -> int32 scalar
 *   LEN            in0 tensor -> int32 scalar = shape[0] (the whitelisted `len`)
 *   SUM            in0 f32 tensor -> f32 scalar (sum of all elements)
 *   ZEROS_LIKE     in0 -> zeros of the same dtype/shape
 *   COLUMN         in0 = matrix [B,T], in1 = scalar t -> vector [B] = in0[:, t]
 *   ELEMENT        in0 = vector, in1 = scalar i -> scalar in0[i]
 *   EMBEDDING      in0 = table [V,E] f32, in1 = int ids (scalar or [n]) -> rows [n,E]
 *   LINEAR         in0 = x [n,K], in1 = W [N,K], in2 = b [N] -> x W^T + b  [n,N]
 *   LSTM_CELL      in0 = x [B,E], in1 = h [B,H], in2 = c [B,H], in3 = W_ih [4H,E],
 *                  in4 = W_hh [4H,H], in5 = b [4H] (gate blocks i,f,g,o), in6 = valid mask int32 [B]
 *                  (rows with valid==0 carry h,c unchanged)
 *   TREELSTM_LEAF  in0 = x [1,E], in1 = W_leaf [3H,E] (blocks i,o,u), in2 = b [4H] (blocks i,f,o,u)
 *   TREELSTM_CELL  in0 = h_l, in1 = c_l, in2 = h_r, in3 = c_r ([1,H] each), in4 = U [5H,2H]
 *                  (blocks i,f_l,f_r,o,u), in5 = b [4H]
 *   TREERNN_CELL   in0 = h_l, in1 = h_r ([1,H] each), in2 = W [H,2H], in3 = b [H] -> h [1,H] =
 *                  tanh([h_l; h_r] W^T + b) (TreeRNN [37], Table 2; one output port)
 *   DROPOUT        in0 = x [n,D] f32, in1 = key i32[2], in2 = scalar step t; iattr0 = site,
 *                  fattr0 = p -> x * m / (1 - p): inverted dropout of a non-recurrent connection
 *                  (Zaremba et al. [51]). m[r][j] = 1 iff word j mod 4 of Philox4x32-10
 *                  (counter = (j / 4, t * n + r, site, 0), key) >= floor(p * 2^32).
 *   SOFTMAX_XENT   in0 = logits [n,C], in1 = targets int32 [n], in2 = mask int32 [n] -> f32
 *                  scalar: mean over masked rows of (logsumexp(logits_r) - logits_r[target_r])
 *   SEQ_MASK       in0 = lengths [B], in1 = scalar T -> int32 [T*B], row t*B+b = (t < len_b)
 *   TIME_MAJOR     in0 = int matrix [B,W], in1 = scalar T -> int32 [T*B], row t*B+b = in0[b,t]
 *   TA_NEW         -> empty tensor array (list)
 *   TA_WRITE       in0 = array, in1 = scalar index, in2 = value -> array with element set
 *   TA_STACK       in0 = array of n values [k, D] -> [n*k, D] (concatenate rows in index order)
 *   SWITCH         in0 = data, in1 = int predicate scalar
 *   MERGE          in0.. = candidate inputs (n_in >= 2)
 *   ENTER          in0 = value; iattr0 = frame id (>0), iattr1 = 1 if loop-invariant
 *   EXIT, NEXT_ITERATION, LOOP_COND, IDENTITY: in0
 *   INVOKE         iattr0 = callee function id; inputs = callee arguments; output port k =
 *                  the callee's RETURN input k
 *   RETURN         inputs = return values of the enclosing function (func > 0)
 *   SGD_APPLY      in0 = scalar loss; iattr0 = state slot of the parameter, iattr1 = effect seq;
 *                  fattr0 = learning rate. Effect: slot -= lr * (d loss / d value read from slot),
 *                  averaged over data-parallel ranks ("average of gradients").
 * janus_op.func = id of the function body the node belongs to (0 = main program). Function
 * bodies use ARG nodes for their parameters (iattr0 = parameter index) and one RETURN node.
 * ------------------------------------------------------------------------------------------- */
typedef enum {
  JOP_ARG = 0, JOP_CONST = 1, JOP_STATE_READ = 2, JOP_STATE_WRITE = 3, JOP_OUTPUT = 4,
  JOP_ADD = 5, JOP_LESS = 6, JOP_EQ = 7, JOP_MAX_REDUCE = 8, JOP_SUM = 9, JOP_ZEROS_LIKE = 10,
  JOP_COLUMN = 11, JOP_ELEMENT = 12,
  JOP_EMBEDDING = 13, JOP_LINEAR = 14, JOP_LSTM_CELL = 15, JOP_TREELSTM_LEAF = 16,
  JOP_TREELSTM_CELL = 17, JOP_SOFTMAX_XENT = 18, JOP_SEQ_MASK = 19, JOP_TIME_MAJOR = 20,
  JOP_TA_NEW = 21, JOP_TA_WRITE = 22, JOP_TA_STACK = 23,
  JOP_SWITCH = 24, JOP_MERGE = 25, JOP_ENTER = 26, JOP_EXIT = 27, JOP_NEXT_ITERATION = 28,
  JOP_LOOP_COND = 29, JOP_IDENTITY = 30, JOP_INVOKE = 31, JOP_RETURN = 32,
  JOP_SGD_APPLY = 33, JOP_LEN = 34, JOP_TREERNN_CELL = 35, JOP_DROPOUT = 36,
  JOP__COUNT = 37
} janus_op_kind;

#define JANUS_MAX_IN 12
typedef struct {
  int32_t kind;                  /* janus_op_kind */
  int32_t func;                  /* function body id, 0 = main */
  int32_t n_in;
  int32_t in_node[JANUS_MAX_IN]; /* producer node index into the ops array */
  int32_t in_port[JANUS_MAX_IN]; /* producer output port */
  int64_t iattr[8];
  double fattr[2];
} janus_op;

/* ---------------------------------------------------------------------------------------------
 * Assumptions ("the optimized graph and the assumption that were used to generate the
 * graph"; Figure 4 specialisation hierarchy P:240-248).
 *   mode DISPATCH: validated from tensor metadata before launch ("checked when retrieving
 *                  the graph from the graph cache"); failure launches nothing.
 *   mode RUNTIME : validated on the device by AssertOps over input data.
 *
 *   JA_DTYPE_EQ     args[target].dtype == dtype                                    (DISPATCH)
 *   JA_SHAPE_MATCH  args[target] has ndim dims and dims[k] == -1 ('?') or equal    (DISPATCH)
 *                   (Figure 4: (4,8) relaxed to (?,8))
 *   JA_TRIP_COUNT   every element of int32 args[target] == value: the loop whose trip count is
 *                   max(lengths) runs exactly `value` iterations with no masked rows; the graph is
 *                   unrolled ("unrolls the loop with this fixed iteration count, and adds
 *                   an assertion operation")                                          (RUNTIME)
 *   JA_TYPE_TAG     int32 state[target][0] == value: the `self.state is None` branch takes the
 *                   tensor arm (P:226-228 single-arm branch; P:238 attribute type)    (RUNTIME)
 *   JA_RANGE        lo <= args[target][i] <= hi for all i; if ref_arg >= 0 then also
 *                   args[target][i] <= args[ref_arg].shape[ref_dim]                   (RUNTIME)
 *   JA_TREE_BINARY  the forest args (kind,left,right,word,tree_off = args target..target+4) is a
 *                   list of binary trees in per-tree post-order: every node is a leaf (kind 0,
 *                   0 <= word < hi) or binary (kind 1, two distinct children with ids in
 *                   [tree_off[t], node), each node having exactly one parent), tree root = last
 *                   node, at most `value` nodes per tree — the structure the level-batched
 *                   lowering of the recursive InvokeOp (P:224, P:316 fn6) relies on (RUNTIME)
 *   JA_VALUE_EQ     int32 args[target][0] == value (constant promotion)        (RUNTIME)
 *   JA_BRANCH_ARM   the Switch whose predicate is int32 args[target][0] (taken when != 0, as the
 *                   SWITCH op reads it) takes arm `value` (1: true arm, 0: false arm): the
 *                   untaken arm is dropped and the branch asserted ("speculates the
 *                   branch ... single arm"); unlike VALUE_EQ any non-zero predicate satisfies the
 *                   true arm; observed = the predicate value                            (RUNTIME)
 * ------------------------------------------------------------------------------------------- */
typedef enum {
  JA_DTYPE_EQ = 0, JA_SHAPE_MATCH = 1, JA_TRIP_COUNT = 2, JA_TYPE_TAG = 3, JA_RANGE = 4,
  JA_TREE_BINARY = 5, JA_VALUE_EQ = 6, JA_BRANCH_ARM = 7
} janus_assumption_kind;

enum { JANUS_MODE_DISPATCH = 0, JANUS_MODE_RUNTIME = 1 };

typedef struct {
  uint32_t id;        /* assumption id reported on failure (smaller id wins) */
  int32_t kind;       /* janus_assumption_kind */
  int32_t mode;       /* JANUS_MODE_* */
  int32_t target;     /* argument index (state slot for JA_TYPE_TAG) */
  int32_t dtype;      /* JA_DTYPE_EQ */
  int32_t ndim;       /* JA_SHAPE_MATCH */
  int64_t dims[4];    /* JA_SHAPE_MATCH, -1 = '?' */
  int64_t lo, hi, value;
  int32_t ref_arg, ref_dim; /* JA_RANGE optional shape bound, -1 = none */
} janus_assumption;

/* Failure report. observed = the offending value (dim size, dtype code, element value);
 * index = dim index (DISPATCH) or flat element index (RUNTIME). */
typedef struct {
  uint32_t assumption_id;
  int32_t rank;
  int64_t index;
  int64_t observed;
} janus_failure;

typedef struct {
  int32_t world_size;        /* data-parallel ranks; 1 = single GPU                 */
  int32_t rank;
  uint8_t nccl_id[128];      /* ncclUniqueId bytes from rank 0 (ignored when world_size==1) */
  int32_t gemm_dtype;        /* JANUS_BF16: bf16 operands, fp32 accumulate (tcgen05);
                                JANUS_F32: fp32 SIMT everywhere                             */
  int32_t strip_asserts;     /* test/ablation only: drop RUNTIME AssertOps (P:392 overhead) */
  int32_t fail_assert_id;    /* fault injection: force this assumption id to fail, -1 = off */
  /* Ablation / test switches; 0 = the default build (Figure 7 arms):              */
  int32_t serial_layers;     /* 1: stacked LSTM layers one after the other, forward and backward
                                (no layer wavefront: the layer-parallelism analogue of +PARL)   */
  int32_t tree_grid;         /* CTAs of the level-batched tree kernels: 0 = one per SM; 1 = the
                                -PARL arm (no parallelism across the nodes of a level)          */
  int32_t force_dp;          /* 1 with world_size == 1: run the data-parallel collective path
                                (arena allreduce, agreement, null step) on a 1-rank communicator */
  int32_t no_dp_overlap;     /* 1: no early dW_dec allreduce on the split communicator          */
  int32_t fused_allreduce;   /* 1 (data parallel, 2-layer LM): the weight gradients are reduced
                                across ranks inside the weight-gradient GEMM's epilogue over
                                NVLink peer memory (NCCL symmetric windows, NCCL-owned), tile by
                                tile as the tiles finish (NEXT-3); else one NCCL allreduce      */
} janus_build_opts;

typedef struct janus_graph janus_graph;

/* Validate the op list, split assumptions into DISPATCH/RUNTIME, specialise (unroll trip-count
 * loops, drop single-arm branches, lower recursive INVOKE to level-batched tree evaluation) and
 * encode the device program. Keeps the generic op list for janus_run_imperative.
 * On JANUS_ERR_INVALID / JANUS_ERR_UNSUPPORTED a message is written to err (if err_len > 0) and
 * *out is NULL — except that ERR_UNSUPPORTED still returns a graph usable by
 * janus_run_imperative (the device graph is absent; janus_run then returns ERR_UNSUPPORTED). */
janus_status janus_graph_build(const janus_op *ops, int32_t n_ops, const janus_assumption *asms,
                               int32_t n_asms, const janus_build_opts *opts, janus_graph **out,
                               char *err, size_t err_len);

/* Device bytes the caller must allocate for `workspace` (graph path and imperative path). The
 * first janus_run on a workspace zero-fills it (the device program keeps zero pads and counters
 * there across steps); later runs reuse it as left, so the caller must not modify it between
 * calls. janus_run_imperative may write anywhere in it; the next janus_run re-initialises. */
janus_status janus_workspace_bytes(const janus_graph *g, size_t *bytes);

/* One speculative graph step. Enqueues on cuda_stream (a cudaStream_t; NULL = default)
 * and returns after ONE stream synchronisation on the 16-byte status word.
 *   JANUS_OK                : outputs written; every STATE_WRITE / SGD_APPLY effect committed.
 *   JANUS_ASSUMPTION_FAILED : *fail filled (minimum failing id); every state tensor is
 *                             byte-identical to its value before the call; outs unspecified.
 *   JANUS_ERR_RUNTIME       : nothing committed.
 * With world_size > 1 the call is collective: every rank gets the same status. */
janus_status janus_run(janus_graph *g, const janus_tensor *args, int32_t n_args,
                       const janus_tensor *state, int32_t n_state, const janus_tensor *outs,
                       int32_t n_outs, janus_tensor workspace, void *cuda_stream,
                       janus_failure *fail);

/* Imperative fallback (Figure 2 (E)): runs the generic op list op by op, one kernel
 * launch per op instance, control predicates read back to the host (TF-Eager analogue). No
 * assumptions; never returns ASSUMPTION_FAILED; commits unless ERR_RUNTIME.
 * With world_size > 1 the call is collective: each rank runs its own shard, then ONE
 * allreduce(sum) of [every SGD-updated slot's gradient, ascending slot | runtime-error count]
 * over the graph's communicator; every rank returns ERR_RUNTIME if any rank hit one, otherwise
 * every rank applies W -= (lr / world_size) * summed gradient. A rank that fails before the
 * collective still joins it. Every SGD-updated state slot must be F32. */
janus_status janus_run_imperative(janus_graph *g, const janus_tensor *args, int32_t n_args,
                                  const janus_tensor *state, int32_t n_state,
                                  const janus_tensor *outs, int32_t n_outs,
                                  janus_tensor workspace, void *cuda_stream);

/* The caller wrote a state tensor outside the library (an optimizer, a checkpoint load, an
 * in-place update). The LM step keeps bf16 working copies of its weight matrices (R1)
 * that its own commit refreshes (P:164 commit, P:282 deferred update), so a step skips the re-cast
 * while the masters were written only by the library since its last run; this call makes the
 * next step of every graph re-cast. Required after any such write; never fails. (The Python
 * binding calls it itself when a state tensor's version counter moved.) */
janus_status janus_state_changed(void);

/* Cumulative counters of this graph: kernel launches issued by the library, host
 * synchronisations, and aborts (ASSUMPTION_FAILED returns). */
janus_status janus_counters(const janus_graph *g, uint64_t *launches, uint64_t *host_syncs,
                            uint64_t *aborts);

/* Human-readable description of the lowered device program (phases), for tests and docs. */
janus_status janus_describe(const janus_graph *g, char *buf, size_t buf_len);

void janus_graph_destroy(janus_graph *g); /* NULL-safe */
const char *janus_status_str(janus_status s);
int32_t janus_abi_version(void);

/* ---------------------------------------------------------------------------------------------
 * Graph cache + relaxation driver (Figure 2 of the paper).
 *
 * A session owns the generic op list and a cache of speculatively specialised graphs, each saved
 * with the assumptions it was generated under ("the optimized graph and the assumption that
 * were used to generate the graph are saved into the graph cache"). Every step:
 *   1. Dispatch: the first active entry whose DISPATCH assumptions hold for the argument
 *      metadata runs janus_run. No entry matches = cache miss: the step runs imperatively
 *      (janus_run_imperative of a graph built without assumptions).
 *   2. An AssertOp failure falls back to the imperative executor in the same call
 *      ("falls back to the imperative executor"), so a step always returns the imperative
 *      result when an assumption breaks.
 *   3. Policy ("gives up further optimizations that rely on the assumptions that
 *      repeatedly break"; SPEC S:516-524 threshold 2): once the SAME assumption of an entry has
 *      failed `fail_threshold` times (only failures whose fallback committed count), the entry is
 *      retired and regenerated with that assumption relaxed one level (janus_relax); once the
 *      same dispatch key has missed `fail_threshold` times, a graph specialised to the observed
 *      key is generated — a shape-only miss first tries the per-dim join of Figure 4 (P:246-248,
 *      "(4, 8) and (3, 8)" -> "(?, 8)") and replaces the old entry if the joined graph still has
 *      a device program; otherwise the new entry coexists with the old one (one specialised graph
 *      per key, as the cache keys on argument types).
 *   A generated graph without a device program (janus_graph_build ERR_UNSUPPORTED) is cached as
 *   an imperative-only entry: its key dispatches straight to the imperative executor.
 * Entries are never re-specialised once relaxed (relaxation is monotone; with at most 2 levels
 * per assumption the number of aborts per assumption is bounded by 2 * fail_threshold).
 * Single-GPU only (world_size must be 1): regeneration would need a fresh NCCL communicator.
 * A session is not thread-safe; one step at a time (as janus_run).
 * ------------------------------------------------------------------------------------------- */
typedef struct janus_session janus_session;

typedef struct {
  int32_t fail_threshold;  /* failures (misses) of one assumption (key) before regeneration; <=0 -> 2 */
  int32_t cache_max;       /* active entries kept (least recently dispatched retired); <=0 -> unlimited */
  int32_t reserved[6];
} janus_session_opts;

enum { JANUS_PATH_GRAPH = 0, JANUS_PATH_IMPERATIVE = 1 };
enum {
  JANUS_EV_HIT = 0,               /* dispatched, every assumption held: graph result       */
  JANUS_EV_MISS = 1,              /* no entry matched: imperative (P:162 cache miss)       */
  JANUS_EV_ABORT = 2,             /* dispatched, an AssertOp failed: imperative fallback   */
  JANUS_EV_IMPERATIVE_ENTRY = 3   /* dispatched to an entry without a device program       */
};

typedef struct {
  int32_t path;             /* JANUS_PATH_* that produced the returned result                */
  int32_t event;            /* JANUS_EV_*                                                    */
  int32_t entry;            /* id of the dispatched entry, -1 on a miss                      */
  int32_t generated;        /* id of the entry generated by this step, -1 if none            */
  janus_failure fail;       /* MISS: first failing DISPATCH assumption of the first active
                               entry; ABORT: the AssertOp failure (zeroed on a HIT)          */
  uint64_t workspace_bytes; /* bytes the step needs (always set; see JANUS_ERR_WORKSPACE)    */
} janus_step_info;

/* Copies the op list and assumptions, builds the initial entry (the caller's assumptions, i.e.
 * the profiled context of P:150) and the assumption-free graph used for cache misses.
 * Status as janus_graph_build for the op list; the initial entry may lack a device program.
 * opts may be NULL (defaults); bopts as for janus_graph_build (world_size must be 1). */
janus_status janus_session_create(const janus_op *ops, int32_t n_ops, const janus_assumption *asms,
                                  int32_t n_asms, const janus_build_opts *bopts,
                                  const janus_session_opts *opts, janus_session **out, char *err,
                                  size_t err_len);

/* Largest workspace any active entry (or the miss path) of the session currently needs. */
janus_status janus_session_workspace_bytes(const janus_session *s, size_t *bytes);

/* One step through the cache (see above). Arguments as janus_run. Returns the status of the
 * result that was committed (JANUS_OK, or the imperative executor's ERR_RUNTIME / ERR_*); never
 * JANUS_ASSUMPTION_FAILED. JANUS_ERR_WORKSPACE: nothing ran and no counter moved; grow the
 * workspace to info->workspace_bytes and call again. info may be NULL. */
janus_status janus_session_step(janus_session *s, const janus_tensor *args, int32_t n_args,
                                const janus_tensor *state, int32_t n_state,
                                const janus_tensor *outs, int32_t n_outs, janus_tensor workspace,
                                void *cuda_stream, janus_step_info *info);

/* JSON report (SPEC S:508-516 analogue): calls, graph/imperative calls, misses, aborts by
 * assumption id, generated entries and every entry (id, active, device, hits, assumptions). */
janus_status janus_session_stats(const janus_session *s, char *buf, size_t buf_len);

void janus_session_destroy(janus_session *s); /* NULL-safe */

/* Relax one failed assumption one level up the specialisation hierarchy (Figure 4, P:240-248;
 * SPEC S:253-261 relax). `observed` = metadata of the offending argument (DISPATCH kinds; may be
 * NULL otherwise; only dtype/ndim/shape are read, data is never touched).
 *   DTYPE_EQ    -> DTYPE_EQ on the observed dtype (the cache keys on argument types)
 *   SHAPE_MATCH -> per-dim join with the observed shape: dims that differ become -1 ('?');
 *                  a rank mismatch drops the assumption (kind level)
 *   TRIP_COUNT  -> RANGE [1, value] on the same argument: the loop is regenerated as a bounded
 *                  device While (P:222 Enter/Exit/NextIteration) instead of unrolled
 *   TYPE_TAG, VALUE_EQ, BRANCH_ARM, RANGE, TREE_BINARY -> dropped (the construct is evaluated on the
 *                  device or the graph loses its device program)
 * *out receives the relaxed assumption (same id) unless *dropped = 1. Pure host function. */
janus_status janus_relax(const janus_assumption *a, const janus_tensor *observed,
                         janus_assumption *out, int32_t *dropped);

#ifdef __cplusplus
}
#endif
#endif /* JANUS_H */
