// host_lm.cpp — speculative lowering and device program of the Figure 1 LSTM language model
// (Table 2 LSTM on PTB).
//
// lower_lm recognises the generic graph built by the imperative program (loop frame over
// time steps with LSTM_CELL layers, embedding lookup, decoder LINEAR + SOFTMAX_XENT, SGD_APPLY
// effects, STATE_WRITE of the carried state) and specialises it under the assumptions:
//   TRIP_COUNT(lengths == T) -> the loop is unrolled to T steps with no masking;
//   RANGE(1 <= lengths <= W) -> device-resident While loop, trip count max(lengths) computed on
//                               the device, masked rows carry their state;
//   TYPE_TAG(tag == TENSOR)  -> the `self.state is None` Switch/Merge is dropped;
//                               without it the predicate is evaluated on the device.
// Every RUNTIME assumption becomes a device AssertOp; the commit is predicated on all of them.
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <string>

#include "gemm_tc.h"
#include "host.h"
#include "imp_kernels.h"
#include "lm_rec.h"
#include "lm_small.h"
#include "step_kernels.h"

namespace jk {

static constexpr int GEMM_PART_TILES = 320;  // split-K scratch: 320 partial 128 x 256 fp32 tiles

static int r8(int x) { return (x + 7) & ~7; }
static size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

static bool slot_of(const Graph &g, int node, int *slot, int64_t dims[4] = nullptr, int *ndim = nullptr) {
  const int o = producer_origin(g, node);
  if (o < 0 || g.ops[o].kind != JOP_STATE_READ) return false;
  *slot = (int)g.ops[o].iattr[0];
  if (dims) for (int k = 0; k < 4; ++k) dims[k] = g.ops[o].iattr[3 + k];
  if (ndim) *ndim = (int)g.ops[o].iattr[2];
  return true;
}

static bool is_arg(const Graph &g, int node, int idx) {
  const int o = producer_origin(g, node);
  return o >= 0 && g.ops[o].kind == JOP_ARG && g.ops[o].iattr[0] == idx;
}

bool lower_lm(Graph &g, std::string &why) {
  LmPlan &p = g.lm;
  p = LmPlan();
  std::vector<int> cells;
  int emb = -1, dec = -1, xent = -1;
  for (int i = 0; i < (int)g.ops.size(); ++i) {
    const janus_op &o = g.ops[i];
    if (o.func != 0) continue;
    if (o.kind == JOP_LSTM_CELL) cells.push_back(i);
    if (o.kind == JOP_EMBEDDING) emb = i;
    if (o.kind == JOP_SOFTMAX_XENT) xent = i;
  }
  if (cells.empty()) { why = "no LSTM_CELL"; return false; }
  p.L = (int)cells.size();
  if (p.L > 4) { why = "more than 4 layers"; return false; }
  int64_t d[4];
  int nd;
  // dropout sites (Zaremba [51]): DROPOUT(x, key, t) with site s on the input of layer s (s < L)
  // and on the decoder input (s = L); every site present, one p and one key argument
  int drop_site_node[5] = {-1, -1, -1, -1, -1};
  auto through_dropout = [&](int node, int port, int site, int *src, int *src_port) -> bool {
    const janus_op &o = g.ops[node];
    if (o.kind != JOP_DROPOUT) { *src = node; *src_port = port; return true; }
    if (o.iattr[0] != site || site > 4) return false;
    const int ko = producer_origin(g, o.in_node[1]);
    if (ko < 0 || g.ops[ko].kind != JOP_ARG) return false;
    const int ka = (int)g.ops[ko].iattr[0];
    if ((p.key_arg >= 0 && p.key_arg != ka) || (p.dropout != 0.f && p.dropout != (float)o.fattr[0])) return false;
    p.key_arg = ka;
    p.dropout = (float)o.fattr[0];
    drop_site_node[site] = node;
    *src = o.in_node[0];
    *src_port = o.in_port[0];
    return true;
  };
  for (int l = 0; l < p.L; ++l) {
    const janus_op &c = g.ops[cells[l]];
    if (!slot_of(g, c.in_node[3], &p.slot_Wih[l], d, &nd) || nd != 2) { why = "W_ih not a state slot"; return false; }
    if (l == 0) { p.H = (int)(d[0] / 4); p.E = (int)d[1]; }
    else if (d[1] != p.H) { why = "layer input width"; return false; }
    if (d[0] != 4 * p.H) { why = "W_ih rows != 4H"; return false; }
    if (!slot_of(g, c.in_node[4], &p.slot_Whh[l], d, &nd) || d[0] != 4 * p.H || d[1] != p.H) { why = "W_hh"; return false; }
    if (!slot_of(g, c.in_node[5], &p.slot_b[l], d, &nd) || d[0] != 4 * p.H) { why = "bias"; return false; }
    if (!slot_of(g, c.in_node[1], &p.slot_h[l], d, &nd) || nd != 2 || d[1] != p.H) { why = "h state"; return false; }
    if (l == 0) p.B = (int)d[0];
    else if (d[0] != p.B) { why = "h batch"; return false; }
    if (!slot_of(g, c.in_node[2], &p.slot_c[l], d, &nd) || d[0] != p.B || d[1] != p.H) { why = "c state"; return false; }
    int xin = -1, xport = 0;
    if (!through_dropout(c.in_node[0], c.in_port[0], l, &xin, &xport)) { why = "dropout site"; return false; }
    if (l == 0) {
      if (xin != emb) { why = "layer-0 input is not the embedding"; return false; }
    } else if (xin != cells[l - 1] || xport != 0) { why = "layer chain"; return false; }
    const janus_op &v = g.ops[c.in_node[6]];
    if (v.kind != JOP_LESS || !is_arg(g, v.in_node[1], 2)) { why = "valid mask"; return false; }
  }
  if (emb < 0) { why = "no EMBEDDING"; return false; }
  {
    const janus_op &e = g.ops[emb];
    if (!slot_of(g, e.in_node[0], &p.slot_E, d, &nd) || nd != 2 || d[1] != p.E) { why = "embedding table"; return false; }
    p.V = (int)d[0];
    const janus_op &col = g.ops[e.in_node[1]];
    if (col.kind != JOP_COLUMN || !is_arg(g, col.in_node[0], 0)) { why = "embedding ids"; return false; }
  }
  if (xent < 0) { why = "no SOFTMAX_XENT"; return false; }
  {
    const janus_op &x = g.ops[xent];
    dec = x.in_node[0];
    const janus_op &lin = g.ops[dec];
    if (lin.kind != JOP_LINEAR || g.ops[lin.in_node[0]].kind != JOP_TA_STACK) { why = "decoder"; return false; }
    for (const auto &o : g.ops)  // what the loop collects for the decoder: h_top or DROPOUT(h_top)
      if (o.func == 0 && o.kind == JOP_TA_WRITE) {
        int src = -1, sp = 0;
        const int vn = o.in_node[2];
        if (!through_dropout(vn, o.in_port[2], p.L, &src, &sp) || src != cells[p.L - 1] || sp != 0) {
          why = "decoder input is not the top layer's h";
          return false;
        }
      }
    if (p.key_arg >= 0)
      for (int s = 0; s <= p.L; ++s)
        if (drop_site_node[s] < 0) { why = "dropout on some but not all non-recurrent connections"; return false; }
    if (!slot_of(g, lin.in_node[1], &p.slot_Wdec, d, &nd) || d[0] != p.V || d[1] != p.H) { why = "W_dec"; return false; }
    if (!slot_of(g, lin.in_node[2], &p.slot_bdec, d, &nd) || d[0] != p.V) { why = "b_dec"; return false; }
    const janus_op &tm = g.ops[x.in_node[1]];
    const janus_op &mk = g.ops[x.in_node[2]];
    if (tm.kind != JOP_TIME_MAJOR || !is_arg(g, tm.in_node[0], 1)) { why = "targets"; return false; }
    if (mk.kind != JOP_SEQ_MASK || !is_arg(g, mk.in_node[0], 2)) { why = "mask"; return false; }
  }
  bool has_output = false;
  for (const auto &o : g.ops) {
    if (o.func != 0) continue;
    if (o.kind == JOP_OUTPUT && o.in_node[0] == xent && o.iattr[0] == 0) has_output = true;
    if (o.kind == JOP_SGD_APPLY) {
      if (o.in_node[0] != xent) {
        // `if training: update` (P:312 train / evaluate branch): SWITCH(loss, training[0]), arm 1
        const janus_op &sw = g.ops[o.in_node[0]];
        if (sw.kind != JOP_SWITCH || sw.in_node[0] != xent || o.in_port[0] != 1) { why = "SGD of another loss"; return false; }
        const janus_op &el = g.ops[sw.in_node[1]];
        const int ao = el.kind == JOP_ELEMENT ? producer_origin(g, el.in_node[0]) : -1;
        const int ko = el.kind == JOP_ELEMENT ? producer_origin(g, el.in_node[1]) : -1;
        if (ao < 0 || g.ops[ao].kind != JOP_ARG || g.ops[ao].iattr[0] != 3 || ko < 0 ||
            g.ops[ko].kind != JOP_CONST || g.ops[ko].fattr[0] != 0.0) {
          why = "update predicate is not training[0] (argument 3)";
          return false;
        }
        p.train_arg = 3;
      }
      const int s = (int)o.iattr[0];
      const float lr = (float)o.fattr[0];
      bool hit = false;
      if (s == p.slot_E) { p.lr_E = lr; hit = true; }
      if (s == p.slot_Wdec) { p.lr_Wdec = lr; hit = true; }
      if (s == p.slot_bdec) { p.lr_bdec = lr; hit = true; }
      for (int l = 0; l < p.L; ++l) {
        if (s == p.slot_Wih[l]) { p.lr_Wih[l] = lr; hit = true; }
        if (s == p.slot_Whh[l]) { p.lr_Whh[l] = lr; hit = true; }
        if (s == p.slot_b[l]) { p.lr_b[l] = lr; hit = true; }
      }
      if (!hit) { why = "SGD on a non-parameter slot"; return false; }
    }
    if (o.kind == JOP_STATE_WRITE) {
      const int s = (int)o.iattr[0];
      const int src = producer_origin(g, o.in_node[0]);
      bool ok = false;
      for (int l = 0; l < p.L; ++l)
        if ((s == p.slot_h[l] || s == p.slot_c[l]) && g.ops[src].kind == JOP_STATE_READ &&
            g.ops[src].iattr[0] == s) ok = true;
      if (ok) p.write_h = true;
      if (!ok && g.ops[src].kind == JOP_CONST && g.ops[src].fattr[0] == 1.0) {
        p.slot_tag = s;
        p.write_tag = true;
        ok = true;
      }
      if (!ok) { why = "unrecognised state write"; return false; }
    }
  }
  if (!has_output) { why = "loss is not output 0"; return false; }
  // the tag Switch: SWITCH(h_0 state, EQ(STATE_READ tag, 1))
  for (const auto &o : g.ops)
    if (o.func == 0 && o.kind == JOP_SWITCH && producer_origin(g, o.in_node[0]) >= 0) {
      int s;
      if (slot_of(g, o.in_node[0], &s) && s == p.slot_h[0] && g.ops[o.in_node[1]].kind == JOP_EQ) {
        int ts;
        if (slot_of(g, g.ops[o.in_node[1]].in_node[0], &ts)) p.slot_tag = ts;
      }
    }
  // assumptions -> specialisation + device guards
  int trip = -1, width = -1;
  for (const auto &a : g.asms)
    if (a.kind == JA_DTYPE_EQ && a.target >= 0 && a.target <= 2) {
      if (a.dtype != JANUS_I32 && a.dtype != JANUS_I64) {
        why = "token / target / length arguments must be int32 or int64";
        return false;
      }
      p.arg_dtype[a.target] = a.dtype;
    }
  for (const auto &a : g.asms) {
    if (a.kind == JA_TRIP_COUNT && a.target == 2) trip = (int)a.value;
    if (a.kind == JA_RANGE && a.target == 2) width = (int)a.hi;
    if (a.kind == JA_SHAPE_MATCH && a.target == 0 && a.ndim == 2) {
      if (a.dims[0] != -1 && a.dims[0] != p.B) { why = "token batch != state batch"; return false; }
      if (a.dims[1] != -1 && width < 0) width = (int)a.dims[1];
    }
    if (a.kind == JA_TYPE_TAG && a.target == p.slot_tag && a.value == 1) p.tag_specialised = true;
    // the training Switch with its value speculated (constant promotion): only the taken
    // arm is kept and the VALUE_EQ AssertOp checks it
    if ((a.kind == JA_VALUE_EQ || a.kind == JA_BRANCH_ARM) && a.mode == JANUS_MODE_RUNTIME && p.train_arg >= 0 &&
        a.target == p.train_arg && a.value != 0)
      p.train_specialised = true;
  }
  for (const auto &a : g.asms)
    if (a.mode == JANUS_MODE_RUNTIME &&
        (a.kind == JA_VALUE_EQ || a.kind == JA_BRANCH_ARM || a.kind == JA_RANGE || a.kind == JA_TRIP_COUNT) &&
        (a.target < 0 || a.target > (p.train_arg >= 0 ? 3 : 2))) {
      why = "runtime assumption on an unknown argument";
      return false;
    }
  if (trip > 0) { p.T = trip; p.while_mode = false; }
  else if (width > 0) { p.T = width; p.while_mode = true; }
  else { why = "no TRIP_COUNT or bounded RANGE assumption on lengths"; return false; }
  if (!p.tag_specialised && p.slot_tag < 0) { why = "state tag slot"; return false; }
  for (const auto &a : g.asms) {
    if (a.mode != JANUS_MODE_RUNTIME) continue;
    LmPlan::RG r{};
    r.id = a.id;
    r.value = a.value; r.lo = a.lo; r.hi = a.hi; r.ref_arg = a.ref_arg; r.ref_dim = a.ref_dim;
    r.arg = a.target; r.slot = -1;
    if (a.kind == JA_TRIP_COUNT) r.kind = G_ALL_EQ;
    else if (a.kind == JA_RANGE) r.kind = G_RANGE;
    else if (a.kind == JA_VALUE_EQ) r.kind = G_FIRST_EQ;
    else if (a.kind == JA_BRANCH_ARM) r.kind = G_FIRST_TRUTH;
    else if (a.kind == JA_TYPE_TAG) { r.kind = G_FIRST_EQ; r.slot = a.target; r.arg = -1; }
    else { why = "unsupported runtime assumption for this graph"; return false; }
    if (g.opts.strip_asserts) continue;
    p.runtime_guards.push_back(r);
  }
  if (g.opts.fail_assert_id >= 0)
    for (const auto &a : g.asms)
      if ((int)a.id == g.opts.fail_assert_id && a.mode == JANUS_MODE_RUNTIME) {
        LmPlan::RG r{};
        r.kind = G_FORCED; r.id = a.id; r.arg = -1; r.slot = -1;
        p.runtime_guards.push_back(r);
      }
  if ((int)p.runtime_guards.size() > MAX_GUARDS) { why = "too many runtime guards"; return false; }
  p.bf16 = g.opts.gemm_dtype != JANUS_F32;
  if (!p.bf16 && p.train_arg >= 0 && !p.train_specialised) {
    why = "fp32 single-CTA path: the training Switch must be speculated (VALUE_EQ)";
    return false;
  }
  if (g.opts.world_size > 1 && !p.bf16) { why = "fp32 path is single-GPU"; return false; }
  if (p.key_arg >= 0 && !p.bf16) { why = "dropout runs on the bf16 tensor-core path"; return false; }
  if (p.key_arg >= 0 && (p.dropout <= 0.f || p.dropout >= 1.f)) { why = "dropout probability outside (0, 1)"; return false; }
  // ------------------------------------------------------------------ workspace layout
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = a256(o + bytes); return r; };
  p.off.status = take(sizeof(DevStatus));
  p.nbar = rec_flag_words(256) * 8;  // per-CTA step flags: 256 CTAs x (L <= 4 layers) x 2 directions
  if ((p.H + 15) / 16 > 256) { why = "hidden size > 4096"; return false; }
  p.off.barriers = take(p.nbar * sizeof(unsigned));
  p.off.stage_args = take((3ull * p.B * p.T + 8) * sizeof(int));  // tokens, targets, lengths, training, key
  const int B = p.B, T = p.T, H = p.H, E = p.E, V = p.V, G4 = 4 * p.H;
  if (!p.bf16) {
    p.off.small_ws = take(small_lm_ws_floats(V, E, H, p.L, B, T) * sizeof(float));
  } else {
    if (B > 128) { why = "batch > 128 (one TMEM tile of batch rows)"; return false; }
    if (H % 2) { why = "odd hidden size"; return false; }
    if (T * B > 8192) { why = "T*B > 8192"; return false; }
    p.Ep = r8(E + 1);
    // h rows are streamed by the recurrent kernels in whole 64-column chunks: pitch >= 64*ceil(H/64)
    p.Hp = std::max(r8(H + 1), 64 * ((H + 63) / 64));
    p.Gz = 64 * ((G4 + 63) / 64);  // dz pitch (chunked the same way)
    const int Vp = r8(V);
    const size_t TB = (size_t)T * B;
    for (int l = 0; l < p.L; ++l) {
      const int Inp = l ? p.Hp : p.Ep;
      p.off.Wih_b[l] = take((size_t)G4 * Inp * 2);
      p.off.Whh_b[l] = take((size_t)G4 * p.Hp * 2);
      p.off.WhhT_b[l] = take((size_t)H * G4 * 2);
      p.off.bil[l] = take((size_t)G4 * 4);
      p.off.Hs[l] = take((TB + B) * p.Hp * 2);
      p.off.Cs[l] = take((TB + B) * p.Hp * 4);
      p.off.G[l] = take(TB * p.Gz * 4);  // gate pitch padded to 64 per recurrent CTA
      p.off.DZ[l] = take(TB * p.Gz * 2);
      p.off.Hsw[l] = take(rec_hsw_bytes(H, B, T));
      p.off.DZsw[l] = take(rec_dzsw_bytes(H, B, T));
      p.off.dX[l] = take(TB * Inp * 4);
      p.off.hT[l] = take((size_t)B * H * 4);
      p.off.cT[l] = take((size_t)B * H * 4);
    }
    if (p.key_arg >= 0)  // dropout: masked bf16 input copies of layers 1 .. L-1 and of the decoder
      for (int s = 1; s <= p.L; ++s) p.off.Xd[s] = take(TB * p.Hp * 2);
    p.off.Wdec_b = take((size_t)V * p.Hp * 2);
    if (p.L == 2) p.off.WihT_b1 = take((size_t)H * G4 * 2);  // W_ih1^T for the backward wavefront
    p.off.X = take(TB * p.Ep * 2);
    p.off.logits = take(TB * Vp * 4);
    p.off.dy = take(TB * Vp * 2);
    p.off.rowloss = take(TB * 4);
    p.off.dHtop = take(TB * p.Hp * 4);
    // gradient arena: one contiguous fp32 block, allreduced in one NCCL call under DP
    p.off.arena_begin = o;
    p.off.gWdec = take((size_t)V * p.Hp * 4);  // first: its allreduce may start during the backward
    p.off.arena_early_end = o;
    for (int l = 0; l < p.L; ++l) {
      const int Inp = l ? p.Hp : p.Ep;
      p.off.gWih[l] = take((size_t)G4 * Inp * 4);
      p.off.gWhh[l] = take((size_t)G4 * p.Hp * 4);
    }
    if (dp_enabled(g)) p.off.dEd = take((size_t)V * E * 4);  // dense embedding gradient
    p.off.arena_end = o;
    p.off.dp_scratch = take(64);
    p.off.seg_word = take(TB * 4);
    p.off.seg_grad = take(TB * p.Ep * 4);
    p.off.nseg = take(16);
    p.off.ehist = take(((size_t)V + 2 * TB + 1) * 4);
    {  // split-K GEMM flags (one region: the step's GEMMs run in stream order)
      const int mx = std::max({(int)TB, V, G4, p.Ep, p.Hp + 1});
      p.off.gflags = take(gemm_flags_count(mx, mx) * 4);
      p.off.gpart = take((size_t)GEMM_PART_TILES * 128 * 256 * 4);
    }
  }
  p.ws_bytes = o;
  char buf[512];
  snprintf(buf, sizeof buf,
           "lstm_lm: L=%d V=%d E=%d H=%d B=%d %s=%d tag=%s train=%s dropout=%g path=%s guards=%zu "
           "phases=[init,%sguards,cast,gather,{gemm_in,rec_fwd}xL,gemm_dec,xent,gemm_dWdec,"
           "gemm_dh,{rec_bwd,gemm_dWhh,gemm_dWih,gemm_dx}xL,embed_grad,finalize,commit]",
           p.L, p.V, p.E, p.H, p.B, p.while_mode ? "while_width" : "unrolled_T", p.T,
           p.tag_specialised ? "specialised" : "device_switch",
           p.train_arg < 0 ? "none" : p.train_specialised ? "specialised" : "device_switch",
           (double)(p.key_arg >= 0 ? p.dropout : 0.f), p.bf16 ? "tcgen05_bf16" : "fp32_single_cta",
           p.runtime_guards.size(), p.while_mode ? "trip," : "");
  g.describe = buf;
  return true;
}

// ---------------------------------------------------------------------------------- run
struct LmPtrs {
  const int *tok, *tgt, *lens;
  int W;
  float *E, *Wih[4], *Whh[4], *b[4], *Wdec, *bdec, *h[4], *c[4];
  int *tag;
};

static bool tensor_ok(const janus_tensor &t, int dtype, int64_t numel) {
  if (!t.data || t.dtype != dtype) return false;
  int64_t n = 1;
  for (int k = 0; k < t.ndim; ++k) n *= t.shape[k];
  return n == numel;
}

static GuardList make_guards(const LmPlan &p, const std::vector<LmPlan::RG> &rgs,
                             const janus_tensor *args, const int *const *argp,
                             const janus_tensor *state) {
  GuardList gl{};
  for (const auto &r : rgs) {
    GuardDesc d{};
    d.kind = r.kind;
    d.id = r.id;
    d.value = r.value; d.lo = r.lo; d.hi = r.hi;
    if (r.kind == G_FORCED) { d.data = nullptr; d.n = 0; }
    else if (r.slot >= 0) { d.data = static_cast<const int *>(state[r.slot].data); d.n = 1; }
    else {
      d.data = argp[r.arg];
      int64_t n = 1;
      for (int k = 0; k < args[r.arg].ndim; ++k) n *= args[r.arg].shape[k];
      d.n = n;
      if (r.kind == G_RANGE && r.ref_arg >= 0)
        d.hi = std::min<int64_t>(d.hi, args[r.ref_arg].shape[r.ref_dim]);
    }
    gl.g[gl.n++] = d;
  }
  (void)p;
  return gl;
}

janus_status finish(Graph &g, DevStatus *dst, const janus_tensor *outs, int n_outs,
                    cudaStream_t st, janus_failure *fail) {
  g.prof.mark("readback", st);
  g.prof.mark(nullptr, st);
  if (!g.h_status && cudaMallocHost(&g.h_status, sizeof(DevStatus)) != cudaSuccess) return JANUS_ERR_CUDA;
  if (n_outs > 0 && outs[0].data && is_device_ptr(outs[0].data))
    if (cudaMemcpyAsync(outs[0].data, &dst->loss, 4, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return JANUS_ERR_CUDA;
  if (cudaMemcpyAsync(g.h_status, dst, sizeof(DevStatus), cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return JANUS_ERR_CUDA;
  cudaError_t e = cudaStreamSynchronize(st);
  g.host_syncs++;
  if (e != cudaSuccess) return JANUS_ERR_CUDA;
  g.prof.collect();
  const DevStatus &h = *g.h_status;
  if (n_outs > 0 && outs[0].data && !is_device_ptr(outs[0].data))
    *static_cast<float *>(outs[0].data) = h.loss;
  if (h.status == JANUS_ASSUMPTION_FAILED) {
    if (fail) {
      fail->assumption_id = (uint32_t)(h.key >> IDX_BITS);
      fail->rank = g.nccl ? h.pad[0] : g.opts.rank;  // DP: the rank that failed (agreement)
      const unsigned long long idx = h.key & ((1ull << IDX_BITS) - 1);
      fail->index = idx == (1ull << IDX_BITS) - 1 ? -1 : (int64_t)idx;
      fail->observed = h.observed;
    }
    return JANUS_ASSUMPTION_FAILED;
  }
  return h.status == 0 ? JANUS_OK : (janus_status)h.status;
}

#define LCHK(name, x)                             \
  do {                                            \
    g.prof.mark(name, st);                        \
    cudaError_t e_ = (x);                         \
    g.launches++;                                 \
    if (e_ != cudaSuccess) return JANUS_ERR_CUDA; \
  } while (0)

// The grouped weight-gradient launch of the 2-layer backward wavefront, shapes only (the same list
// for a step and for its null step, so both reduce the same tiles): [dW_dec | db_dec], dW_hh1,
// [dW_ih1 | db1], dW_hh0, [dW_ih0 | db0] — gradients (c_off = arena byte offset of C) — and the
// embedding dgrad dx0 (not a gradient, when E is trained).
struct WgShape {
  int M, N, K, ldc;
  size_t c_off;
  bool grad;
};
static int lm_wgrad_shapes(const LmPlan &p, bool with_dwdec, WgShape *w) {
  const int TB = p.B * p.T, G4 = 4 * p.H, H = p.H, E = p.E;
  const size_t a0 = p.off.arena_begin;
  int n = 0;
  if (with_dwdec) w[n++] = {p.V, H + 1, TB, p.Hp, p.off.gWdec - a0, true};
  for (int l = 1; l >= 0; --l) {
    w[n++] = {G4, H, TB, p.Hp, p.off.gWhh[l] - a0, true};
    w[n++] = {G4, (l ? H : E) + 1, TB, l ? p.Hp : p.Ep, p.off.gWih[l] - a0, true};
  }
  if (p.lr_E != 0) w[n++] = {TB, E, G4, p.Ep, 0, false};
  return n;
}
// Tile geometry and per-GEMM descriptors of the fused reduction for this step's epoch; returns the
// number of fused tiles (their flags are 0 .. tiles-1 of the flag window).
static int lm_fused_plan(const Graph &g, bool with_dwdec, unsigned epoch, FusedReduce *fr, FusedGeom *geo, int *ng) {
  WgShape w[6];
  const int n = lm_wgrad_shapes(g.lm, with_dwdec, w);
  GemmOp ops[6];
  for (int i = 0; i < n; ++i) { ops[i].M = w[i].M; ops[i].N = w[i].N; ops[i].K = w[i].K; }
  int bn = 0, mb[6], nb[6];
  gemm_group_tiling(ops, n, &bn, mb, nb);
  int tiles = 0, k = 0;
  for (int i = 0; i < n; ++i) {
    if (!w[i].grad) { fr[i] = FusedReduce(); continue; }
    fr[i] = fused_descriptor(g.far, w[i].c_off, (size_t)tiles, epoch);
    geo[k] = FusedGeom{w[i].M, w[i].N, w[i].ldc, mb[i], nb[i], bn};
    ++k;
    tiles += mb[i] * nb[i];
  }
  *ng = k;
  return tiles;
}

janus_status run_lm(Graph &g, const janus_tensor *args, const janus_tensor *state,
                    const janus_tensor *outs, int n_outs, const janus_tensor &ws, cudaStream_t st,
                    janus_failure *fail) {
  const LmPlan &p = g.lm;
  if (!ws.data || (size_t)ws.shape[0] * (ws.dtype == JANUS_U8 ? 1 : 4) < p.ws_bytes) return JANUS_ERR_INVALID;
  uint8_t *W = static_cast<uint8_t *>(ws.data);
  const int B = p.B, H = p.H, E = p.E, V = p.V, G4 = 4 * p.H, L = p.L;
  // ---- arguments (stage host buffers into the workspace: the e2e path)
  const int Wd = (int)args[0].shape[1];
  if (args[0].ndim != 2 || args[0].shape[0] != B || Wd > p.T || (!p.while_mode && Wd != p.T))
    return JANUS_ERR_INVALID;
  const int *argp[4] = {nullptr, nullptr, nullptr, nullptr};
  if (p.train_arg >= 0) {  // training flag i32[1]
    if (!tensor_ok(args[3], JANUS_I32, 1)) return JANUS_ERR_INVALID;
    if (is_device_ptr(args[3].data)) argp[3] = static_cast<const int *>(args[3].data);
    else {
      int *dstp = reinterpret_cast<int *>(W + p.off.stage_args) + (size_t)3 * B * p.T;
      if (cudaMemcpyAsync(dstp, args[3].data, 4, cudaMemcpyHostToDevice, st) != cudaSuccess) return JANUS_ERR_CUDA;
      argp[3] = dstp;
    }
  }
  const int *keyp = nullptr;  // dropout key (Philox), i32[2]
  if (p.key_arg >= 0) {
    if (!tensor_ok(args[p.key_arg], JANUS_I32, 2)) return JANUS_ERR_INVALID;
    if (is_device_ptr(args[p.key_arg].data)) keyp = static_cast<const int *>(args[p.key_arg].data);
    else {
      int *dstp = reinterpret_cast<int *>(W + p.off.stage_args) + (size_t)3 * B * p.T + 4;
      if (cudaMemcpyAsync(dstp, args[p.key_arg].data, 8, cudaMemcpyHostToDevice, st) != cudaSuccess) return JANUS_ERR_CUDA;
      keyp = dstp;
    }
  }
  for (int a = 0; a < 3; ++a) {
    const int64_t n = a < 2 ? (int64_t)B * Wd : B;
    if (!tensor_ok(args[a], p.arg_dtype[a], n)) return JANUS_ERR_INVALID;
    if (p.arg_dtype[a] == JANUS_I64) {
      // type-specialised graph (the cache keys on argument types): narrow on the device
      if (!is_device_ptr(args[a].data)) return JANUS_ERR_INVALID;
      int *dstp = reinterpret_cast<int *>(W + p.off.stage_args) + (size_t)a * B * p.T;
      if (imp::i64_to_i32(dstp, static_cast<const long long *>(args[a].data), n, st) != cudaSuccess)
        return JANUS_ERR_CUDA;
      g.launches++;
      argp[a] = dstp;
    } else if (is_device_ptr(args[a].data)) argp[a] = static_cast<const int *>(args[a].data);
    else {
      int *dstp = reinterpret_cast<int *>(W + p.off.stage_args) + (size_t)a * B * p.T;
      if (cudaMemcpyAsync(dstp, args[a].data, n * 4, cudaMemcpyHostToDevice, st) != cudaSuccess)
        return JANUS_ERR_CUDA;
      argp[a] = dstp;
    }
  }
  // CUDA-graph replay (below) needs every argument at a fixed address: stage device arguments
  // into the workspace slots too (one device-to-device copy each, outside the graph)
  const bool i64_args = p.arg_dtype[0] == JANUS_I64 || p.arg_dtype[1] == JANUS_I64 || p.arg_dtype[2] == JANUS_I64;
  // opt-in (JANUS_STEP_GRAPH=1): measured 72.5k vs 73.5k samples/s for direct launches at C2 —
  // the programmatic-dependent launches already overlap the launch latency, and the replay adds
  // the argument copies
  static const bool graph_on = getenv("JANUS_STEP_GRAPH") && getenv("JANUS_STEP_GRAPH")[0] == '1';
  const bool graphable = graph_on && p.bf16 && !dp_enabled(g) && !g.prof.on && !g.probe && !i64_args &&
                         !getenv("JANUS_NO_GRAPH");
  if (graphable) {
    int *sa = reinterpret_cast<int *>(W + p.off.stage_args);
    int *slot[5] = {sa, sa + (size_t)B * p.T, sa + (size_t)2 * B * p.T, sa + (size_t)3 * B * p.T,
                    sa + (size_t)3 * B * p.T + 4};
    const int64_t cnt[5] = {(int64_t)B * Wd, (int64_t)B * Wd, B, 1, 2};
    for (int a = 0; a < 4; ++a) {
      if (!argp[a] || argp[a] == slot[a]) continue;
      if (cudaMemcpyAsync(slot[a], argp[a], cnt[a] * 4, cudaMemcpyDeviceToDevice, st) != cudaSuccess) return JANUS_ERR_CUDA;
      argp[a] = slot[a];
    }
    if (keyp && keyp != slot[4]) {
      if (cudaMemcpyAsync(slot[4], keyp, 8, cudaMemcpyDeviceToDevice, st) != cudaSuccess) return JANUS_ERR_CUDA;
      keyp = slot[4];
    }
  }
  // ---- state slots
  LmPtrs P{};
  P.tok = argp[0]; P.tgt = argp[1]; P.lens = argp[2]; P.W = Wd;
  auto sf = [&](int slot, int64_t n) -> float * {
    if (slot < 0 || !tensor_ok(state[slot], JANUS_F32, n) || !is_device_ptr(state[slot].data)) return nullptr;
    return static_cast<float *>(state[slot].data);
  };
  if (!(P.E = sf(p.slot_E, (int64_t)V * E))) return JANUS_ERR_INVALID;
  for (int l = 0; l < L; ++l) {
    const int In = l ? H : E;
    if (!(P.Wih[l] = sf(p.slot_Wih[l], (int64_t)G4 * In)) || !(P.Whh[l] = sf(p.slot_Whh[l], (int64_t)G4 * H)) ||
        !(P.b[l] = sf(p.slot_b[l], G4)) || !(P.h[l] = sf(p.slot_h[l], (int64_t)B * H)) ||
        !(P.c[l] = sf(p.slot_c[l], (int64_t)B * H)))
      return JANUS_ERR_INVALID;
  }
  if (!(P.Wdec = sf(p.slot_Wdec, (int64_t)V * H)) || !(P.bdec = sf(p.slot_bdec, V))) return JANUS_ERR_INVALID;
  P.tag = p.slot_tag >= 0 ? static_cast<int *>(state[p.slot_tag].data) : nullptr;
  DevStatus *dst = reinterpret_cast<DevStatus *>(W + p.off.status);
  unsigned *bars = reinterpret_cast<unsigned *>(W + p.off.barriers);
  GuardList gl = make_guards(p, p.runtime_guards, args, argp, state);

  if (!p.bf16) {
    // ------------------------------------------------------------ single-CTA fp32 program
    SmallLmArgs a;
    a.V = V; a.E = E; a.H = H; a.L = L; a.B = B; a.W = Wd; a.T = p.while_mode ? Wd : p.T;
    a.tok = P.tok; a.tgt = P.tgt; a.lens = p.while_mode ? P.lens : nullptr;
    a.Emb = P.E; a.Wdec = P.Wdec; a.bdec = P.bdec; a.tag = p.write_tag ? P.tag : nullptr;
    a.tag_specialised = p.tag_specialised;
    if (!p.tag_specialised) a.tag = P.tag;
    for (int l = 0; l < L; ++l) {
      a.Wih[l] = P.Wih[l]; a.Whh[l] = P.Whh[l]; a.bias[l] = P.b[l]; a.h[l] = P.h[l]; a.c[l] = P.c[l];
      a.upd_Wih[l] = p.lr_Wih[l] != 0; a.upd_Whh[l] = p.lr_Whh[l] != 0; a.upd_b[l] = p.lr_b[l] != 0;
    }
    a.upd_E = p.lr_E != 0; a.upd_Wdec = p.lr_Wdec != 0; a.upd_bdec = p.lr_bdec != 0;
    float lr = 0;
    for (float v : {p.lr_E, p.lr_Wdec, p.lr_bdec, p.lr_Wih[0], p.lr_Whh[0], p.lr_b[0]}) if (v != 0) lr = v;
    a.lr = lr;
    a.gl = gl;
    a.ws = reinterpret_cast<float *>(W + p.off.small_ws);
    a.st = dst;
    LCHK("lm_small_f32", launch_small_lm(a, st));
    return finish(g, dst, outs, n_outs, st, fail);
  }

  // ------------------------------------------------------------ tcgen05 device program
  if (dp_enabled(g)) {
    janus_status r = dp_init(g);
    if (r != JANUS_OK) return r;
  }
  // The step as ONE CUDA graph: the first call with a given (workspace, state, width, stream)
  // runs the launches directly, the second captures them into a graph, later calls replay it
  // (one cudaGraphLaunch instead of 15 launches; the host's dispatch guards and the status readback
  // stay outside). Any capture failure falls back to direct launches for this graph.
  // bf16 operand copies (R1): re-cast from the masters, unless the last commit refreshed them and
  // nothing else wrote state since (host.h copies_epoch); this step's commit refreshes them
  static const bool recast_env = [] { const char *e = getenv("JANUS_RECAST"); return e && e[0] == '1'; }();
  const void *srcs[9] = {};
  for (int l = 0; l < L; ++l) { srcs[2 * l] = P.Wih[l]; srcs[2 * l + 1] = P.Whh[l]; }
  srcs[2 * L] = P.Wdec;
  bool copies_ok = !recast_env && g.copies_in && g.copies_W == W;
  for (int k = 0; k < 9; ++k) copies_ok = copies_ok && g.copies_src[k] == srcs[k];
  const bool refresh = !recast_env;
  g.copies_out = refresh;
  g.copies_W = W;
  for (int k = 0; k < 9; ++k) g.copies_src[k] = srcs[k];
  GraphKey key{};
  key.W = W;
  key.width = Wd;
  key.stream = st;
  key.cast = !copies_ok;
  for (int k = 0; k < g.n_state && k < 64; ++k) key.state[k] = state[k].data;
  if (graphable && g.cg.exec && g.cg.key == key) {
    g.prof.mark("graph", st);
    if (cudaGraphLaunch(static_cast<cudaGraphExec_t>(g.cg.exec), st) != cudaSuccess) return JANUS_ERR_CUDA;
    g.launches += g.cg.kernels;
    return finish(g, dst, outs, n_outs, st, fail);
  }
  const bool capture = graphable && !g.cg.failed && g.cg.seen && g.cg.seen_key == key;
  if (graphable && !capture) { g.cg.seen = true; g.cg.seen_key = key; }
  const uint64_t launches0 = g.launches;
  if (capture && cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
    (void)cudaGetLastError();
    g.cg.failed = true;
  }
  const bool capturing = capture && !g.cg.failed;
  auto enqueue = [&]() -> janus_status {
  // gradient arena: the workspace, or NCCL's symmetric window when reduced in the GEMM epilogue
  auto ar = [&](size_t off) -> float * {
    return g.far.arena ? reinterpret_cast<float *>(static_cast<uint8_t *>(g.far.arena) + (off - p.off.arena_begin))
                       : reinterpret_cast<float *>(W + off);
  };
  const int T = p.T;              // unrolled T or max width W
  const int Tw = p.while_mode ? Wd : T;  // width of this batch
  const int TB = Tw * B;
  const int Vp = r8(V), Ep = p.Ep, Hp = p.Hp;
  const int *Tdev = p.while_mode ? &dst->trip : nullptr;
  auto bf = [&](size_t off) { return reinterpret_cast<__nv_bfloat16 *>(W + off); };
  auto fp = [&](size_t off) { return reinterpret_cast<float *>(W + off); };
  unsigned *gflags = reinterpret_cast<unsigned *>(W + p.off.gflags);
  if (g.gflags_ws != W) {  // counters start at zero; every GEMM launch leaves them at zero
    const int mx = std::max({B * p.T, V, 4 * H, p.Ep, p.Hp + 1});
    if (cudaMemsetAsync(gflags, 0, gemm_flags_count(mx, mx) * 4, st) != cudaSuccess) return JANUS_ERR_CUDA;
    g.gflags_ws = W;
  }
  float *gpart = reinterpret_cast<float *>(W + p.off.gpart);
  auto with_flags = [&](GemmOp o) {
    o.flags = gflags;
    o.partials = gpart;
    o.partials_cap = (size_t)GEMM_PART_TILES * 128 * 256;
    return o;
  };
  if (p.while_mode) {
    LCHK("init", launch_step_init(dst, bars, p.nbar, st, p.bf16 ? rec_flag_words(1) : 1));
    LCHK("trip", launch_trip(P.lens, B, Tw, dst, st));
    if (gl.n) LCHK("guards", launch_guards(gl, dst, st));
  } else {
    LCHK("init", launch_step_init_guards(dst, bars, p.nbar, p.bf16 ? rec_flag_words(1) : 1, gl, st));
  }
  // operand copies (R1): interleaved / transposed bf16 working copies of the fp32 masters, the
  // interleaved biases and the ones columns — one fused launch
  {
    PrepList pl = {};
    auto add = [&](PrepSeg sg) { pl.s[pl.n++] = sg; };
    for (int l = 0; l < L; ++l) {
      const int In = l ? H : E, Inp = l ? Hp : Ep;
      PrepSeg sg = {};
      if (!copies_ok) {
        sg.kind = P_CAST_ROWS; sg.src = P.Wih[l]; sg.dst = bf(p.off.Wih_b[l]); sg.rows = G4; sg.cols = In;
        sg.ld_src = In; sg.ld_dst = Inp; sg.H = H; add(sg);
        sg = {}; sg.kind = P_CAST_ROWS; sg.src = P.Whh[l]; sg.dst = bf(p.off.Whh_b[l]); sg.rows = G4; sg.cols = H;
        sg.ld_src = H; sg.ld_dst = Hp; sg.H = H; add(sg);
        sg = {}; sg.kind = P_CAST_T_IL; sg.src = P.Whh[l]; sg.dst = bf(p.off.WhhT_b[l]); sg.ld_dst = G4; sg.H = H; add(sg);
      }
      sg = {}; sg.kind = P_BIAS_IL; sg.src = P.b[l]; sg.fdst = fp(p.off.bil[l]); sg.H = H; add(sg);
      sg = {}; sg.kind = P_FILL_COL; sg.dst = bf(p.off.Hs[l]); sg.rows = TB + B; sg.cols = H; sg.ld_dst = Hp; add(sg);
    }
    if (L == 2 && !copies_ok) {  // W_ih1^T (interleaved) for the backward wavefront
      PrepSeg sg = {};
      sg.kind = P_CAST_T_IL; sg.src = P.Wih[1]; sg.dst = bf(p.off.WihT_b1); sg.ld_dst = G4; sg.H = H; add(sg);
    }
    if (!copies_ok) {
      PrepSeg sg = {};
      sg.kind = P_CAST_ROWS; sg.src = P.Wdec; sg.dst = bf(p.off.Wdec_b); sg.rows = V; sg.cols = H;
      sg.ld_src = H; sg.ld_dst = Hp; sg.H = 0; add(sg);
    }
    LCHK("cast", launch_prep_gather(pl, P.E, V, E, P.tok, B, Wd, Tw, Tdev, bf(p.off.X), Ep, dst, st));
  }
  const bool drop = p.key_arg >= 0;  // Zaremba dropout: site 0 on the embedding output (in place)
  if (drop) LCHK("dropout", launch_dropout_bf16(bf(p.off.X), bf(p.off.X), TB, E, Ep, keyp, 0, p.dropout, st));
  // input of layer l (l >= 1) and of the decoder: the layer below's h, or its dropped copy
  auto layer_in = [&](int l) -> __nv_bfloat16 * {
    return drop ? bf(p.off.Xd[l]) : bf(p.off.Hs[l - 1]) + (size_t)B * Hp;
  };
  // forward
  // two layers: one wavefront launch (layer 1 one step behind layer 0, its input projection
  // fused into the recurrent MMA) unless disabled or too wide for one CTA per SM
  const bool wavefront = L == 2 && !g.opts.serial_layers && !drop && rec_fwd_wf_grid(H) <= 148;
  // single rank: the embedding-gradient bucketing runs on a side stream beside
  // the forward recurrence (its CTAs leave SMs free); the stream and events are created once
  const bool early_bucket = p.lr_E != 0 && !g.nccl && wavefront && [&] {
    if (g.bk_side) return true;
    return cudaStreamCreateWithFlags(&g.bk_side, cudaStreamNonBlocking) == cudaSuccess &&
           cudaEventCreateWithFlags(&g.ev_bk_fork, cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&g.ev_bk_join, cudaEventDisableTiming) == cudaSuccess;
  }();
  auto rec_args = [&](int l) {
    RecFwdArgs ra;
    ra.B = B; ra.H = H; ra.T = Tw; ra.T_dev = Tdev; ra.lens = p.while_mode ? P.lens : nullptr;
    ra.Hsw = bf(p.off.Hsw[l]);
    ra.G = fp(p.off.G[l]); ra.Hs = bf(p.off.Hs[l]); ra.Cs = fp(p.off.Cs[l]); ra.ldh = Hp;
    ra.h0 = P.h[l]; ra.c0 = P.c[l]; ra.hT = fp(p.off.hT[l]); ra.cT = fp(p.off.cT[l]);
    ra.barrier = bars + rec_flag_words(256) * l; ra.fail = nullptr;
    ra.dbg = (l == 0 || wavefront) ? g.probe : nullptr;  // indexed by the launch's CTA index
    ra.tag = p.tag_specialised ? nullptr : P.tag;
    return ra;
  };
  for (int l = 0; l < L; ++l) {
    const int In = l ? H : E, Inp = l ? Hp : Ep;
    if (wavefront && l == 1) break;
    if (drop && l) LCHK("dropout", launch_dropout_bf16(bf(p.off.Hs[l - 1]) + (size_t)B * Hp, bf(p.off.Xd[l]), TB, H, Hp,
                                                     keyp, l, p.dropout, st));
    GemmOp op;
    op.M = TB; op.N = G4; op.K = In;
    op.A = l ? layer_in(l) : bf(p.off.X); op.lda = Inp;
    op.B = bf(p.off.Wih_b[l]); op.ldb = Inp;
    op.ep.C = fp(p.off.G[l]); op.ep.ldc = p.Gz; op.ep.bias_col = fp(p.off.bil[l]);
    LCHK(l ? "gemm_in1" : "gemm_in0", gemm_bf16(with_flags(op), st));
    if (l == 0 && early_bucket) {
      // the embedding-gradient bucketing depends on the token ids only: one block on a side
      // stream beside the forward recurrence (which leaves SMs free), joined before the sums
      if (cudaEventRecord(g.ev_bk_fork, st) != cudaSuccess || cudaStreamWaitEvent(g.bk_side, g.ev_bk_fork, 0) != cudaSuccess)
        return JANUS_ERR_CUDA;
      if (launch_embed_grad(P.tok, B, Wd, Tw, Tdev, V, nullptr, Ep, E, reinterpret_cast<int *>(W + p.off.seg_word),
                            reinterpret_cast<int *>(W + p.off.ehist), fp(p.off.seg_grad), Ep,
                            reinterpret_cast<int *>(W + p.off.nseg), g.bk_side, 1) != cudaSuccess)
        return JANUS_ERR_CUDA;
      g.launches++;
      if (cudaEventRecord(g.ev_bk_join, g.bk_side) != cudaSuccess) return JANUS_ERR_CUDA;
    }
    if (wavefront) {
      LCHK("rec_fwd01", lstm_rec_fwd_wavefront(rec_args(0), rec_args(1), bf(p.off.Whh_b[0]), bf(p.off.Wih_b[1]),
                                               bf(p.off.Whh_b[1]), Hp, fp(p.off.bil[1]), p.while_mode, st));
    } else {
      LCHK(l ? "rec_fwd1" : "rec_fwd0", lstm_rec_fwd(rec_args(l), bf(p.off.Whh_b[l]), Hp, p.while_mode, st));
    }
  }
  if (drop) LCHK("dropout", launch_dropout_bf16(bf(p.off.Hs[L - 1]) + (size_t)B * Hp, bf(p.off.Xd[L]), TB, H, Hp,
                                               keyp, L, p.dropout, st));
  {
    GemmOp op;  // decoder logits
    op.M = TB; op.N = V; op.K = H;
    op.A = layer_in(L); op.lda = Hp;
    op.B = bf(p.off.Wdec_b); op.ldb = Hp;
    op.ep.C = fp(p.off.logits); op.ep.ldc = Vp; op.ep.bias_col = P.bdec;
    LCHK("gemm_dec", gemm_bf16(with_flags(op), st));
  }
  // two layers, B <= 64: one backward wavefront launch (layer 0 one step behind layer 1, the
  // dgrad of layer 1's input W_ih1^T dz1_t folded into layer 0's recurrent MMA)
  const char *bk_env = getenv("JANUS_REC_BWD");  // dev experiment knob: 'p' = plain (unsplit) kernel
  const bool bwd_wave = g.fused_ar || (L == 2 && B <= 64 && !g.opts.serial_layers && !drop &&
                                        !(bk_env && bk_env[0] == 'p') && rec_bwd_wf_grid(H) <= 148);
  const bool overlap = g.nccl && g.nccl2 && g.side;  // dp_overlap() held at init
  const bool fused = g.fused_ar && g.far.arena && bwd_wave;
  const unsigned fused_epoch = fused ? ++g.far.epoch : 0u;
  int fused_tiles = 0;
  GemmOp dwdec;  // dW_dec | db_dec = dy^T [h_top | 1]
  dwdec.M = V; dwdec.N = H + 1; dwdec.K = TB;
  dwdec.A = bf(p.off.dy); dwdec.lda = Vp; dwdec.a_mn = 1;
  dwdec.B = layer_in(L); dwdec.ldb = Hp; dwdec.b_mn = 1;
  dwdec.ep.C = ar(p.off.gWdec); dwdec.ep.ldc = Hp;
  // dh_top = dy W_dec below: long K (V) over few output tiles — 256-wide tiles on CTA pairs, K
  // halved over twice the CTAs, each half reduce-added into dh_top, which the xent launch zeroes
  // on the side (two addends onto zero: order-independent bits); measured at C2 42 vs 60 us
  const bool dh_split = V >= 4096 && !getenv("JANUS_DH_NOSPLIT");
  LCHK("xent", launch_xent(fp(p.off.logits), V, Vp, TB, P.tgt, B, Wd, p.while_mode ? P.lens : nullptr, Tdev,
                   (float)TB, bf(p.off.dy), Vp, fp(p.off.rowloss), dst, st,
                   dh_split ? reinterpret_cast<float4 *>(fp(p.off.dHtop)) : nullptr,
                   dh_split ? (long long)TB * Hp / 4 : 0));
  {
    if (!bwd_wave || overlap) LCHK("gemm_dWdec", gemm_bf16(with_flags(dwdec), st));  // else grouped below
    if (overlap) {  // allreduce dW_dec on the side stream while the backward recurrence runs
      g.prof.mark("dp_allreduce_early", st);
      if (cudaEventRecord(g.ev_fork, st) != cudaSuccess || cudaStreamWaitEvent(g.side, g.ev_fork, 0) != cudaSuccess)
        return JANUS_ERR_CUDA;
      for (const DpSeg &sg : dp_segments(g))  // the split communicator's segments (dW_dec | db_dec)
        if (sg.comm == 2) {
          janus_status r = dp_allreduce_sum2(g, ar(sg.begin), (sg.end - sg.begin) / 4, g.side);
          if (r != JANUS_OK) return r;
        }
      if (cudaEventRecord(g.ev_join, g.side) != cudaSuccess) return JANUS_ERR_CUDA;
    }
    GemmOp o2;  // dh_top = dy W_dec
    o2.M = TB; o2.N = H; o2.K = V;
    o2.A = bf(p.off.dy); o2.lda = Vp;
    o2.B = bf(p.off.Wdec_b); o2.ldb = Hp; o2.b_mn = 1;
    o2.ep.C = fp(p.off.dHtop); o2.ep.ldc = Hp;
    if (dh_split) { o2.splits = 2; o2.split_add = 1; o2.bn = 256; }  // dh_top zeroed by the xent launch
    LCHK("gemm_dh", gemm_bf16(with_flags(o2), st));
    if (drop) LCHK("dropout", launch_dropout_f32(fp(p.off.dHtop), TB, H, Hp, keyp, L, p.dropout, st));
  }
  auto bwd_args = [&](int l) {
    RecBwdArgs rb;
    rb.B = B; rb.H = H; rb.T = Tw; rb.T_dev = Tdev; rb.lens = p.while_mode ? P.lens : nullptr;
    rb.G = fp(p.off.G[l]); rb.Cs = fp(p.off.Cs[l]); rb.ldh = Hp;
    rb.dHin = l == L - 1 ? fp(p.off.dHtop) : fp(p.off.dX[l + 1]); rb.ldd = Hp;
    rb.DZsw = bf(p.off.DZsw[l]);
    rb.DZ = bf(p.off.DZ[l]); rb.ldz = p.Gz; rb.barrier = bars + rec_flag_words(256) * (L + l);
    rb.dbg = ((l == 0 || bwd_wave) && g.probe) ? g.probe + (size_t)128 * 16 * p.T : nullptr;
    return rb;
  };
  if (bwd_wave) {
    RecBwdArgs r0 = bwd_args(0);
    r0.dHin = nullptr;  // layer 1's input dgrad arrives through the fused MMA
    LCHK("rec_bwd01", lstm_rec_bwd_wavefront(bwd_args(1), r0, bf(p.off.WhhT_b[1]), bf(p.off.WihT_b1),
                                             bf(p.off.WhhT_b[0]), G4, p.while_mode, st));
  }
  auto wgrad_ops = [&](int l, GemmOp &a, GemmOp &b2) {
    const int In = l ? H : E, Inp = l ? Hp : Ep;
    const __nv_bfloat16 *xin = l ? layer_in(l) : bf(p.off.X);
    a = GemmOp();  // dW_hh = dz^T h_{t-1}
    a.M = G4; a.N = H; a.K = TB;
    a.A = bf(p.off.DZ[l]); a.lda = p.Gz; a.a_mn = 1;
    a.B = bf(p.off.Hs[l]); a.ldb = Hp; a.b_mn = 1;
    a.ep.C = ar(p.off.gWhh[l]); a.ep.ldc = Hp;
    b2 = GemmOp();  // dW_ih | db = dz^T [x | 1]
    b2.M = G4; b2.N = In + 1; b2.K = TB;
    b2.A = bf(p.off.DZ[l]); b2.lda = p.Gz; b2.a_mn = 1;
    b2.B = xin; b2.ldb = Inp; b2.b_mn = 1;
    b2.ep.C = ar(p.off.gWih[l]); b2.ep.ldc = Inp;
  };
  if (bwd_wave) {  // every weight gradient + the embedding dgrad in one grouped launch
    GemmOp ops[6];
    int n = 0;
    if (!overlap) ops[n++] = dwdec;
    wgrad_ops(1, ops[n], ops[n + 1]);
    n += 2;
    wgrad_ops(0, ops[n], ops[n + 1]);
    n += 2;
    if (p.lr_E != 0) {
      GemmOp &c2 = ops[n++];  // dx0 = dz0 W_ih0 (embedding gradient rows)
      c2 = GemmOp();
      c2.M = TB; c2.N = E; c2.K = G4;
      c2.A = bf(p.off.DZ[0]); c2.lda = p.Gz;
      c2.B = bf(p.off.Wih_b[0]); c2.ldb = Ep; c2.b_mn = 1;
      c2.ep.C = fp(p.off.dX[0]); c2.ep.ldc = Ep;
    }
    if (fused) {  // NEXT-3: each gradient tile reduced across ranks by the epilogue as it finishes
      FusedReduce fr[6];
      FusedGeom geo[6];
      int ng = 0;
      fused_tiles = lm_fused_plan(g, !overlap, fused_epoch, fr, geo, &ng);
      for (int i = 0; i < n; ++i) ops[i].ep.fr = fr[i];
    }
    LCHK("gemm_wgrad", gemm_bf16_group(ops, n, st));
  }
  for (int l = L - 1; l >= 0; --l) {
    const int In = l ? H : E, Inp = l ? Hp : Ep;
    if (!bwd_wave) {
      LCHK(l ? "rec_bwd1" : "rec_bwd0", lstm_rec_bwd(bwd_args(l), bf(p.off.WhhT_b[l]), G4, p.while_mode, st));
      GemmOp a, b2;
      wgrad_ops(l, a, b2);
      LCHK(l ? "gemm_dWhh1" : "gemm_dWhh0", gemm_bf16(with_flags(a), st));
      LCHK(l ? "gemm_dWih1" : "gemm_dWih0", gemm_bf16(with_flags(b2), st));
    }
    if (!bwd_wave && (l > 0 || p.lr_E != 0)) {
      GemmOp c2;  // dx = dz W_ih
      c2.M = TB; c2.N = In; c2.K = G4;
      c2.A = bf(p.off.DZ[l]); c2.lda = p.Gz;
      c2.B = bf(p.off.Wih_b[l]); c2.ldb = Inp; c2.b_mn = 1;
      c2.ep.C = fp(p.off.dX[l]); c2.ep.ldc = Inp;
      LCHK(l ? "gemm_dx1" : "gemm_dx0", gemm_bf16(with_flags(c2), st));
      // the VJP of the dropout on this layer's input (site l) before the layer below reads it
      if (drop) LCHK("dropout", launch_dropout_f32(fp(p.off.dX[l]), TB, In, Inp, keyp, l, p.dropout, st));
    }
  }
  int *seg_word = reinterpret_cast<int *>(W + p.off.seg_word);
  int *nseg = reinterpret_cast<int *>(W + p.off.nseg);
  if (p.lr_E != 0) {
    if (early_bucket && cudaStreamWaitEvent(st, g.ev_bk_join, 0) != cudaSuccess) return JANUS_ERR_CUDA;
    LCHK("embed_grad", launch_embed_grad(P.tok, B, Wd, Tw, Tdev, V, fp(p.off.dX[0]), Ep, E, seg_word,
                                         reinterpret_cast<int *>(W + p.off.ehist), fp(p.off.seg_grad),
                                         Ep, nseg, st, early_bucket ? 2 : 0));
    if (!early_bucket) g.launches++;  // embed grad is two kernels
  }
  if (g.nccl) {
    // DP: dense embedding gradient, one allreduce(sum) of the whole gradient arena
    if (p.lr_E != 0)
      LCHK("dp_scatter", launch_scatter_rows(fp(p.off.seg_grad), Ep, seg_word, nseg, ar(p.off.dEd), V, E, st));
    g.prof.mark("dp_allreduce", st);
    for (const DpSeg &sg : dp_segments(g))
      if (sg.comm == 1) {
        janus_status r = dp_allreduce_sum(g, ar(sg.begin), (sg.end - sg.begin) / 4, st);
        if (r != JANUS_OK) return r;
      }
    if (overlap && cudaStreamWaitEvent(st, g.ev_join, 0) != cudaSuccess) return JANUS_ERR_CUDA;
  }
  // single rank: the finalize runs as one extra block of the commit launch (below)
  const bool fin_in_commit = !g.nccl && !fused;
  if (!fin_in_commit) LCHK("finalize", launch_finalize(fp(p.off.rowloss), TB, gl, dst, g.opts.world_size, st));
  if (g.nccl) {  // every rank learns the same status before anything commits (reading Q12)
    g.prof.mark("dp_agree", st);
    janus_status r = dp_agree(g, dst, reinterpret_cast<long long *>(W + p.off.dp_scratch), st);
    if (r != JANUS_OK) return r;
  }
  if (fused) {  // every tile of this step reduced (the owners' pushes into this rank landed)
    FusedReduce f0 = fused_descriptor(g.far, 0, 0, fused_epoch);
    LCHK("fused_wait", launch_fused_wait(f0, fused_tiles, st));
  }
  // ---- the all-or-nothing commit (P:164, P:266 (4))
  CommitList cl{};
  auto add = [&](CommitSeg s) { cl.s[cl.n++] = s; };
  const float nr = (float)g.opts.world_size;
  for (int l = 0; l < L; ++l) {
    const int In = l ? H : E, Inp = l ? Hp : Ep;
    CommitSeg s{};
    if (p.lr_Wih[l] != 0) {
      s = {}; s.kind = C_DENSE_IL; s.dst = P.Wih[l]; s.grad = ar(p.off.gWih[l]); s.rows = G4; s.cols = In; s.ldg = Inp; s.H = H; s.lr = p.lr_Wih[l] / nr;
      if (refresh) {
        s.bcopy = bf(p.off.Wih_b[l]); s.ldb = Inp;
        if (l == 1 && L == 2) { s.kind = C_DENSE_IL_T; s.tcopy = bf(p.off.WihT_b1); s.ldt = G4; }
      }
      add(s);
    }
    if (p.lr_b[l] != 0) { s = {}; s.kind = C_BIAS_COL_IL; s.dst = P.b[l]; s.grad = ar(p.off.gWih[l]); s.rows = G4; s.cols = 1; s.ldg = Inp; s.col = In; s.H = H; s.lr = p.lr_b[l] / nr; add(s); }
    if (p.lr_Whh[l] != 0) {
      s = {}; s.kind = C_DENSE_IL; s.dst = P.Whh[l]; s.grad = ar(p.off.gWhh[l]); s.rows = G4; s.cols = H; s.ldg = Hp; s.H = H; s.lr = p.lr_Whh[l] / nr;
      if (refresh) { s.kind = C_DENSE_IL_T; s.bcopy = bf(p.off.Whh_b[l]); s.ldb = Hp; s.tcopy = bf(p.off.WhhT_b[l]); s.ldt = G4; }
      add(s);
    }
    if (p.write_h) {
      s = {}; s.kind = C_COPY; s.dst = P.h[l]; s.grad = fp(p.off.hT[l]); s.rows = B; s.cols = H; add(s);
      s = {}; s.kind = C_COPY; s.dst = P.c[l]; s.grad = fp(p.off.cT[l]); s.rows = B; s.cols = H; add(s);
    }
  }
  {
    CommitSeg s{};
    if (p.lr_Wdec != 0) {
      s = {}; s.kind = C_DENSE; s.dst = P.Wdec; s.grad = ar(p.off.gWdec); s.rows = V; s.cols = H; s.ldg = Hp; s.lr = p.lr_Wdec / nr;
      if (refresh) { s.bcopy = bf(p.off.Wdec_b); s.ldb = Hp; }
      add(s);
    }
    if (p.lr_bdec != 0) { s = {}; s.kind = C_BIAS_COL; s.dst = P.bdec; s.grad = ar(p.off.gWdec); s.rows = V; s.cols = 1; s.ldg = Hp; s.col = H; s.lr = p.lr_bdec / nr; add(s); }
    if (p.lr_E != 0 && !g.nccl) { s = {}; s.kind = C_SPARSE_ROWS; s.dst = P.E; s.grad = fp(p.off.seg_grad); s.cols = E; s.ldg = Ep; s.rows_idx = seg_word; s.nrows = nseg; s.lr = p.lr_E / nr; add(s); }
    if (p.lr_E != 0 && g.nccl) { s = {}; s.kind = C_DENSE; s.dst = P.E; s.grad = ar(p.off.dEd); s.rows = V; s.cols = E; s.ldg = E; s.lr = p.lr_E / nr; add(s); }
    if (p.write_tag && P.tag) { s = {}; s.kind = C_TAG; s.idst = P.tag; s.ival = 1; add(s); }
  }
  if (p.train_arg >= 0 && !p.train_specialised)  // the training Switch evaluated on the device
    for (int k = 0; k < cl.n; ++k)
      if (cl.s[k].kind != C_COPY && cl.s[k].kind != C_TAG) cl.s[k].pred = argp[3];
  if (fin_in_commit) LCHK("commit", launch_commit_finalize(cl, FinalizeArgs{fp(p.off.rowloss), TB, gl}, dst, st));
  else LCHK("commit", launch_commit(cl, dst, st));
  return JANUS_OK;
  };  // enqueue
  const janus_status er = enqueue();
  if (capturing) {
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(st, &graph);
    cudaGraphExec_t exec = nullptr;
    if (er == JANUS_OK && ce == cudaSuccess && graph && cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess) {
      g.cg.reset();
      g.cg.exec = exec;
      g.cg.key = key;
      g.cg.kernels = g.launches - launches0;
      cudaGraphDestroy(graph);
      if (cudaGraphLaunch(exec, st) != cudaSuccess) return JANUS_ERR_CUDA;
    } else {  // not capturable here: launch directly from now on
      (void)cudaGetLastError();
      if (graph) cudaGraphDestroy(graph);
      g.cg.failed = true;
      if (er != JANUS_OK) return er;
      const janus_status r2 = enqueue();
      if (r2 != JANUS_OK) return r2;
    }
  } else if (er != JANUS_OK) {
    return er;
  }
  return finish(g, dst, outs, n_outs, st, fail);
}

}  // namespace jk

namespace jk {

// Null step of a data-parallel rank whose DISPATCH guards failed (P:162 cache miss): it launches no
// compute, but joins the same collective sequence as a normal step so its peers cannot block, and
// publishes its failure through the agreement so every rank aborts (reading Q12).
janus_status run_lm_null(Graph &g, const janus_failure &f, const janus_tensor &ws, cudaStream_t st,
                         janus_failure *fail) {
  const LmPlan &p = g.lm;
  if (!ws.data || !p.bf16 || (size_t)ws.shape[0] * (ws.dtype == JANUS_U8 ? 1 : 4) < p.ws_bytes)
    return JANUS_ERR_INVALID;
  janus_status r = dp_init(g);
  if (r != JANUS_OK) return r;
  uint8_t *W = static_cast<uint8_t *>(ws.data);
  DevStatus *dst = reinterpret_cast<DevStatus *>(W + p.off.status);
  unsigned *bars = reinterpret_cast<unsigned *>(W + p.off.barriers);
  LCHK("init", launch_step_init(dst, bars, p.nbar, st, p.bf16 ? rec_flag_words(1) : 1));
  LCHK("set_failure", launch_set_failure(dst, f.assumption_id, f.index, f.observed, st));
  if (g.fused_ar && g.far.arena) {
    // the fused reduction's part of the step: publish every tile, reduce the tiles this rank
    // owns (stale data: the agreement aborts the step), wait for the owners' pushes
    const unsigned ep = ++g.far.epoch;
    FusedReduce fr[6], frg[6];
    FusedGeom geo[6];
    int ng = 0;
    const int tiles = lm_fused_plan(g, g.nccl2 == nullptr, ep, fr, geo, &ng);
    int k = 0;
    for (int i = 0; i < 6 && k < ng; ++i)
      if (fr[i].win) frg[k++] = fr[i];
    LCHK("fused_null", launch_fused_null(frg, geo, ng, st));
    LCHK("fused_wait", launch_fused_wait(fused_descriptor(g.far, 0, 0, ep), tiles, st));
  }
  // the same per-communicator sequence as a full step (dp_segments in order)
  for (const DpSeg &sg : dp_segments(g)) {
    float *b = g.far.arena ? reinterpret_cast<float *>(static_cast<uint8_t *>(g.far.arena) + (sg.begin - p.off.arena_begin))
                           : reinterpret_cast<float *>(W + sg.begin);
    r = sg.comm == 2 ? dp_allreduce_sum2(g, b, (sg.end - sg.begin) / 4, st)
                     : dp_allreduce_sum(g, b, (sg.end - sg.begin) / 4, st);
    if (r != JANUS_OK) return r;
  }
  r = dp_agree(g, dst, reinterpret_cast<long long *>(W + p.off.dp_scratch), st);
  if (r != JANUS_OK) return r;
  return finish(g, dst, nullptr, 0, st, fail);
}

}  // namespace jk
