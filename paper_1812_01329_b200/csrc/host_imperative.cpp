// host_imperative.cpp — janus_run_imperative: the imperative fallback executor (§3.2,
// Figure 2 (E); the TF-Eager column "Imp." of Table 3). It runs the GENERIC op list (no
// assumptions, no specialisation) the way an imperative framework runs the Python program: the
// host walks the program, every op instance is one kernel launch, and every control decision
// (loop condition, branch predicate, data-dependent index) reads a device value back to the host.
// Gradients come from a device-side tape replayed in reverse (the automatically inserted
// differentiation); effects (STATE_WRITE, SGD_APPLY) are applied at the end unless a
// runtime error occurred.
//
// Interpretation is demand-driven: sinks (OUTPUT, effects) are evaluated in node order; a node
// evaluates its inputs first. A loop frame (Enter/Merge/LoopCond/Switch/NextIteration/Exit)
// runs when one of its Exit nodes is demanded: iteration k re-evaluates the frame's nodes with the
// Merge nodes taking the Enter value (k = 0) or the previous NextIteration value.
#include <math.h>
#include <string.h>

#include <algorithm>
#include <deque>
#include <functional>
#include <map>
#include <string>
#include <vector>

#include "host.h"
#include "imp_kernels.h"

namespace jk {

// bf16 operand copies of the tcgen05 GEMM path (imp_kernels.h set_scratch)
static size_t imp_gemm_scratch_bytes(const Graph &g) {
  const size_t plan = g.kind == "lstm_lm" ? g.lm.ws_bytes : g.kind == "treelstm" ? g.tree.ws_bytes : 0;
  return std::min<size_t>(plan, 256u << 20);
}
size_t imperative_ws_bytes(const Graph &g) {
  const size_t plan = g.kind == "lstm_lm" ? g.lm.ws_bytes : g.kind == "treelstm" ? g.tree.ws_bytes : 0;
  return 3 * plan + (64u << 20) + imp_gemm_scratch_bytes(g);
}

namespace {

enum VK { V_DEAD = 0, V_DEV = 1, V_HOST = 2, V_TA = 3 };

struct IVal {
  int kind = V_DEAD;
  int dtype = JANUS_F32;
  std::vector<int64_t> shape;
  void *ptr = nullptr;
  double hv = 0;
  std::map<int64_t, int> ta;
  bool rg = false;  // requires grad
  int64_t numel() const {
    int64_t n = 1;
    for (auto s : shape) n *= s;
    return n;
  }
};

struct TapeE {
  int kind;
  std::vector<int> in, out;
  std::vector<void *> saved;
  int i0 = 0, i1 = 0, i2 = 0;
};

struct Err {
  janus_status st;
  std::string msg;
};

struct Interp {
  Graph &g;
  const janus_tensor *args;
  int n_args;
  const janus_tensor *state;
  cudaStream_t st;
  bool bf16;
  uint8_t *base;
  size_t cap, used = 0;
  int *err_dev = nullptr;
  std::deque<IVal> vals;  // deque: references stay valid while new values are appended
  std::vector<TapeE> tape;
  std::map<int, int> state_vid;            // slot -> vid of STATE_READ
  std::vector<std::pair<int64_t, std::pair<int, int>>> writes;  // (seq, (slot, vid))
  std::vector<std::pair<int64_t, std::pair<int, float>>> sgds;   // (seq, (slot, lr))
  int out_vid = -1;
  uint64_t launches = 0, syncs = 0;
  bool dp_joined = false;  // this rank has issued the step's data-parallel collective
  // static analysis
  std::vector<std::vector<int>> path;      // frame path per node
  std::vector<std::vector<std::pair<int, int>>> consumers;

  Interp(Graph &gg) : g(gg) {}

  void *alloc(size_t bytes) {
    const size_t o = (used + 255) & ~size_t(255);
    if (o + bytes > cap) throw Err{JANUS_ERR_INVALID, "imperative workspace exhausted"};
    used = o + bytes;
    return base + o;
  }
  void ck(cudaError_t e) {
    launches += 1 + imp::take_extra_launches();
    if (e != cudaSuccess) throw Err{JANUS_ERR_CUDA, cudaGetErrorString(e)};
  }
  int new_val(IVal v) {
    vals.push_back(std::move(v));
    return (int)vals.size() - 1;
  }
  int dev_f(std::vector<int64_t> shape, bool zero = false) {
    IVal v;
    v.kind = V_DEV; v.dtype = JANUS_F32; v.shape = shape;
    v.ptr = alloc(std::max<int64_t>(1, v.numel()) * 4);
    if (zero) ck(imp::fill((float *)v.ptr, 0.f, v.numel(), st));
    return new_val(v);
  }
  int dev_i(std::vector<int64_t> shape) {
    IVal v;
    v.kind = V_DEV; v.dtype = JANUS_I32; v.shape = shape;
    v.ptr = alloc(std::max<int64_t>(1, v.numel()) * 4);
    return new_val(v);
  }
  int host_i(int64_t x) {
    IVal v;
    v.kind = V_HOST; v.dtype = JANUS_I32; v.hv = (double)x;
    return new_val(v);
  }
  // a host integer from a (host or device) int scalar: a device->host read = one host sync
  int64_t as_host_int(int vid) {
    const IVal &v = vals[vid];
    if (v.kind == V_HOST) return (int64_t)v.hv;
    if (v.kind != V_DEV || v.numel() < 1) throw Err{JANUS_ERR_INVALID, "scalar expected"};
    int x = 0;
    float f = 0;
    if (cudaMemcpyAsync(v.dtype == JANUS_I32 ? (void *)&x : (void *)&f, v.ptr, 4, cudaMemcpyDeviceToHost,
                        st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      throw Err{JANUS_ERR_CUDA, "readback"};
    ++syncs;
    const int64_t r = v.dtype == JANUS_I32 ? (int64_t)x : (int64_t)f;
    if (v.numel() == 1) {  // the value is now known on the host: later uses need no sync
      vals[vid].kind = V_HOST;
      vals[vid].hv = (double)r;
    }
    return r;
  }

  // ---------------------------------------------------------------- static analysis
  void analyse() {
    const int n = (int)g.ops.size();
    path.assign(n, {});
    std::vector<bool> known(n, false);
    for (int pass = 0; pass < n + 2; ++pass) {
      bool changed = false;
      for (int i = 0; i < n; ++i) {
        const janus_op &o = g.ops[i];
        std::vector<int> best;
        bool any = o.n_in == 0;
        for (int k = 0; k < o.n_in; ++k) {
          const int p = o.in_node[k];
          if (!known[p]) continue;
          std::vector<int> pp = path[p];
          if (g.ops[p].kind == JOP_ENTER) pp.push_back((int)g.ops[p].iattr[0]);
          else if (g.ops[p].kind == JOP_EXIT && !pp.empty()) pp.pop_back();
          if (!any || pp.size() > best.size()) best = pp;
          any = true;
        }
        if (!any) continue;
        if (!known[i] || path[i] != best) {
          path[i] = best;
          known[i] = true;
          changed = true;
        }
      }
      if (!changed) break;
    }
  }

  // ---------------------------------------------------------------- scopes
  struct Scope {
    std::vector<int> path;
    std::map<int, std::array<int, 2>> memo;  // node -> vids per port (-2 dead)
    Scope *parent = nullptr;
    std::map<int, int> merge_in;             // MERGE node -> vid for this iteration
    int func = 0;
    std::vector<int> fargs;                  // function arguments (func > 0)
  };

  Scope *scope_for(Scope *s, int node) {
    while (s && s->path != path[node]) s = s->parent;
    if (!s) throw Err{JANUS_ERR_INVALID, "node outside its frame"};
    return s;
  }

  int port(Scope *cur, int node, int p) {
    // value of (node, port) seen from scope `cur`
    const janus_op &o = g.ops[node];
    if (o.kind == JOP_ENTER) {  // lives in the parent; its value is the frame input
      Scope *ps = scope_for(cur, node);
      return eval(ps, node)[0];
    }
    if (o.kind == JOP_EXIT) {
      // belongs to the frame path[node]; demanded from the parent scope
      Scope *ps = cur;
      std::vector<int> parent_path = path[node];
      parent_path.pop_back();
      while (ps && ps->path != parent_path) ps = ps->parent;
      if (!ps) throw Err{JANUS_ERR_INVALID, "Exit outside its parent"};
      auto it = ps->memo.find(node);
      if (it == ps->memo.end()) run_loop(ps, path[node].back());
      it = ps->memo.find(node);
      if (it == ps->memo.end()) throw Err{JANUS_ERR_INVALID, "loop produced no exit value"};
      return it->second[p];
    }
    Scope *s = scope_for(cur, node);
    return eval(s, node)[p];
  }

  std::array<int, 2> eval(Scope *s, int node) {
    auto it = s->memo.find(node);
    if (it != s->memo.end()) return it->second;
    const janus_op &o = g.ops[node];
    std::array<int, 2> r{-2, -2};
    if (o.kind == JOP_MERGE) {
      auto mi = s->merge_in.find(node);
      if (mi != s->merge_in.end()) {  // loop merge: value chosen by run_loop
        r = {mi->second, -2};
      } else {                          // if-merge: first live input
        for (int k = 0; k < o.n_in; ++k) {
          const int v = port(s, o.in_node[k], o.in_port[k]);
          if (v >= 0) { r = {v, host_i(k)}; break; }
        }
      }
      s->memo[node] = r;
      return r;
    }
    std::vector<int> in(o.n_in);
    bool dead = false;
    for (int k = 0; k < o.n_in; ++k) {
      in[k] = port(s, o.in_node[k], o.in_port[k]);
      if (in[k] < 0) dead = true;
    }
    if (dead) {
      s->memo[node] = r;
      return r;
    }
    r = exec(s, node, o, in);
    s->memo[node] = r;
    return r;
  }

  // a loop frame F under parent scope ps
  void run_loop(Scope *ps, int F) {
    std::vector<int> fpath = ps->path;
    fpath.push_back(F);
    std::vector<int> fnodes, merges, nis, exits, conds;
    for (int i = 0; i < (int)g.ops.size(); ++i) {
      if (g.ops[i].func != ps->func || path[i] != fpath) continue;
      fnodes.push_back(i);
      const int k = g.ops[i].kind;
      if (k == JOP_MERGE) merges.push_back(i);
      if (k == JOP_NEXT_ITERATION) nis.push_back(i);
      if (k == JOP_EXIT) exits.push_back(i);
      if (k == JOP_LOOP_COND) conds.push_back(i);
    }
    if (conds.size() != 1) throw Err{JANUS_ERR_UNSUPPORTED, "loop frame without one LoopCond"};
    std::map<int, int> ni_prev;
    for (int it = 0;; ++it) {
      Scope fs;
      fs.path = fpath;
      fs.parent = ps;
      fs.func = ps->func;
      fs.fargs = ps->fargs;
      for (int m : merges) {
        const janus_op &o = g.ops[m];
        int chosen = -2;
        for (int k = 0; k < o.n_in; ++k) {
          const int p = o.in_node[k];
          if (g.ops[p].kind == JOP_ENTER && it == 0) chosen = port(&fs, p, o.in_port[k]);
          if (g.ops[p].kind == JOP_NEXT_ITERATION && it > 0) chosen = ni_prev.count(p) ? ni_prev[p] : -2;
        }
        fs.merge_in[m] = chosen;
      }
      const int cv = eval(&fs, conds[0])[0];
      const bool cont = cv >= 0 && as_host_int(cv) != 0;   // LoopCond read back: one host sync
      for (int x : exits) {
        const int v = eval(&fs, x)[0];
        if (v >= 0) ps->memo[x] = {v, -2};
      }
      if (!cont) break;
      std::map<int, int> ni_next;
      for (int n : nis) ni_next[n] = eval(&fs, n)[0];
      ni_prev.swap(ni_next);
      if (it > 1000000) throw Err{JANUS_ERR_RUNTIME, "loop does not terminate"};
    }
    for (int x : exits)
      if (!ps->memo.count(x)) ps->memo[x] = {-2, -2};
  }

  // function body call (InvokeOp): a fresh scope, arguments bound to ARG nodes
  std::vector<int> call(int func, const std::vector<int> &argv) {
    Scope s;
    s.func = func;
    s.fargs = argv;
    int ret = -1;
    for (int i = 0; i < (int)g.ops.size(); ++i)
      if (g.ops[i].func == func && g.ops[i].kind == JOP_RETURN) ret = i;
    if (ret < 0) throw Err{JANUS_ERR_INVALID, "function without RETURN"};
    const janus_op &o = g.ops[ret];
    std::vector<int> out(o.n_in);
    for (int k = 0; k < o.n_in; ++k) out[k] = port(&s, o.in_node[k], o.in_port[k]);
    return out;
  }

  // ---------------------------------------------------------------- op execution
  const IVal &V(int vid) { return vals[vid]; }
  float *fptr(int vid) { return static_cast<float *>(vals[vid].ptr); }
  int *iptr(int vid) { return static_cast<int *>(vals[vid].ptr); }

  // shape mismatch inside a node: a runtime error (S:109 ShapeMismatch), commits nothing
  void need(bool ok) {
    if (!ok) throw Err{JANUS_ERR_RUNTIME, "shape mismatch"};
  }

  // materialise a device float tensor (host scalars become 1-element tensors)
  int as_dev_f(int vid) {
    if (V(vid).kind == V_DEV) return vid;
    const int r = dev_f({});
    ck(imp::fill(fptr(r), (float)V(vid).hv, 1, st));
    return r;
  }
  int as_dev_i(int vid) {
    if (V(vid).kind == V_DEV) return vid;
    const int r = dev_i({});
    ck(imp::fill_i(iptr(r), (int)V(vid).hv, 1, st));
    return r;
  }

  std::array<int, 2> exec(Scope *s, int node, const janus_op &o, const std::vector<int> &in) {
    const bool R = bf16;
    switch (o.kind) {
      case JOP_ARG: {
        const int k = (int)o.iattr[0];
        if (s->func > 0) return {s->fargs.at(k), -2};
        if (k >= n_args) throw Err{JANUS_ERR_INVALID, "missing argument"};
        const janus_tensor &t = args[k];
        IVal v;
        v.kind = V_DEV; v.dtype = t.dtype;
        for (int d = 0; d < t.ndim; ++d) v.shape.push_back(t.shape[d]);
        const int64_t esz = t.dtype == JANUS_I64 ? 8 : 4;
        const int64_t bytes = std::max<int64_t>(1, v.numel()) * esz;
        if (is_device_ptr(t.data)) v.ptr = t.data;
        else {
          v.ptr = alloc(bytes);
          if (cudaMemcpyAsync(v.ptr, t.data, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess)
            throw Err{JANUS_ERR_CUDA, "H2D"};
        }
        if (t.dtype == JANUS_I64) {  // an imperative program takes any integer type (no DtypeEq here)
          void *p32 = alloc(std::max<int64_t>(1, v.numel()) * 4);
          ck(imp::i64_to_i32(static_cast<int *>(p32), static_cast<const long long *>(v.ptr), v.numel(), st));
          v.ptr = p32;
          v.dtype = JANUS_I32;
        } else if (t.dtype != JANUS_I32 && t.dtype != JANUS_F32) {
          throw Err{JANUS_ERR_RUNTIME, "argument dtype"};
        }
        return {new_val(v), -2};
      }
      case JOP_CONST: {
        IVal v;
        v.kind = V_HOST; v.dtype = (int)o.iattr[0]; v.hv = o.fattr[0];
        return {new_val(v), -2};
      }
      case JOP_STATE_READ: {
        const int slot = (int)o.iattr[0];
        const janus_tensor &t = state[slot];
        IVal v;
        v.kind = V_DEV; v.dtype = t.dtype; v.ptr = t.data;
        for (int d = 0; d < t.ndim; ++d) v.shape.push_back(t.shape[d]);
        for (const auto &e : g.ops)
          if (e.kind == JOP_SGD_APPLY && e.iattr[0] == slot) v.rg = true;
        const int vid = new_val(v);
        state_vid[slot] = vid;
        return {vid, -2};
      }
      case JOP_STATE_WRITE:
        writes.push_back({o.iattr[1], {(int)o.iattr[0], in[0]}});
        return {-2, -2};
      case JOP_SGD_APPLY:
        sgds.push_back({o.iattr[1], {(int)o.iattr[0], (float)o.fattr[0]}});
        return {-2, -2};
      case JOP_OUTPUT:
        if (o.iattr[0] == 0) out_vid = in[0];
        return {-2, -2};
      case JOP_IDENTITY: case JOP_LOOP_COND: case JOP_ENTER: case JOP_EXIT: case JOP_NEXT_ITERATION:
        return {in[0], -2};
      case JOP_SWITCH: {
        const bool pred = as_host_int(in[1]) != 0;  // branch decision read back: one host sync
        return pred ? std::array<int, 2>{-2, in[0]} : std::array<int, 2>{in[0], -2};
      }
      case JOP_INVOKE: {
        std::vector<int> r = call((int)o.iattr[0], in);
        return {r.size() > 0 ? r[0] : -2, r.size() > 1 ? r[1] : -2};
      }
      case JOP_ADD: {
        const IVal &a = V(in[0]), &b = V(in[1]);
        if (a.dtype == JANUS_I32 && b.dtype == JANUS_I32)  // Python ints
          return {host_i(as_host_int(in[0]) + as_host_int(in[1])), -2};
        const int x = as_dev_f(in[0]), y = as_dev_f(in[1]);
        const int64_t n = std::max(V(x).numel(), V(y).numel());
        const int big = V(x).numel() >= V(y).numel() ? x : y, sml = big == x ? y : x;
        const int r = dev_f(V(big).shape);
        ck(imp::add_f(fptr(r), fptr(big), fptr(sml), n, V(sml).numel(), st));
        vals[r].rg = V(x).rg || V(y).rg;
        tape.push_back({JOP_ADD, {x, y}, {r}});
        return {r, -2};
      }
      case JOP_LESS: case JOP_EQ: {
        const IVal &a = V(in[0]), &b = V(in[1]);
        const int op = o.kind == JOP_EQ ? 2 : 0;
        if (a.kind == V_HOST && b.kind == V_HOST) {
          const int64_t x = (int64_t)a.hv, y = (int64_t)b.hv;
          return {host_i(op == 2 ? x == y : x < y), -2};
        }
        if (a.kind == V_HOST && b.numel() > 1 && op == 0) {  // scalar < vector
          const int r = dev_i(b.shape);
          ck(imp::less_iv(iptr(r), (int)a.hv, iptr(in[1]), (int)b.numel(), st));
          return {r, -2};
        }
        if (b.kind == V_HOST && a.numel() > 1 && op == 0) {
          const int r = dev_i(a.shape);
          ck(imp::less_vi(iptr(r), iptr(in[0]), (int)b.hv, (int)a.numel(), st));
          return {r, -2};
        }
        if (a.kind == V_DEV && b.kind == V_HOST && a.numel() == 1) {
          const int r = dev_i({});
          ck(imp::cmp_scalar(iptr(r), iptr(in[0]), (int)b.hv, op, st));
          return {r, -2};
        }
        if (b.kind == V_DEV && a.kind == V_HOST && b.numel() == 1) {
          const int r = dev_i({});
          ck(imp::cmp_scalar(iptr(r), iptr(in[1]), (int)a.hv, op == 2 ? 2 : 1, st));
          return {r, -2};
        }
        // device scalar vs device scalar (e.g. t < max(lengths)) -> compare on the host
        const int64_t x = as_host_int(in[0]), y = as_host_int(in[1]);
        return {host_i(op == 2 ? x == y : x < y), -2};
      }
      case JOP_LEN:  // len(x): host metadata, no launch
        need(!V(in[0]).shape.empty());
        return {host_i(V(in[0]).shape[0]), -2};
      case JOP_MAX_REDUCE: {
        const int r = dev_i({});
        ck(imp::max_reduce(iptr(r), iptr(in[0]), (int)V(in[0]).numel(), st));
        return {r, -2};
      }
      case JOP_SUM: {
        const int x = as_dev_f(in[0]);
        const int r = dev_f({});
        ck(imp::sum_all(fptr(r), fptr(x), V(x).numel(), st));
        vals[r].rg = V(x).rg;
        tape.push_back({JOP_SUM, {x}, {r}});
        return {r, -2};
      }
      case JOP_ZEROS_LIKE: {
        const IVal &a = V(in[0]);
        if (a.dtype == JANUS_F32) return {dev_f(a.shape, true), -2};
        const int r = dev_i(a.shape);
        ck(imp::fill_i(iptr(r), 0, a.numel(), st));
        return {r, -2};
      }
      case JOP_COLUMN: {
        const IVal &m = V(in[0]);
        const int t = (int)as_host_int(in[1]);
        const int r = dev_i({m.shape[0]});
        ck(imp::column(iptr(r), iptr(in[0]), (int)m.shape[0], (int)m.shape[1], t, err_dev, st));
        return {r, -2};
      }
      case JOP_ELEMENT: {
        const IVal &v = V(in[0]);
        const int i = (int)as_host_int(in[1]);
        if (v.dtype == JANUS_I32) {
          const int r = dev_i({});
          ck(imp::element_i(iptr(r), iptr(in[0]), (int)v.numel(), i, err_dev, st));
          return {r, -2};
        }
        const int r = dev_f({});
        ck(imp::element_f(fptr(r), fptr(in[0]), (int)v.numel(), i, err_dev, st));
        return {r, -2};
      }
      case JOP_EMBEDDING: {
        const IVal &E = V(in[0]);
        const int ids = as_dev_i(in[1]);
        const int n = (int)std::max<int64_t>(1, V(ids).numel());
        const int r = dev_f({n, E.shape[1]});
        ck(imp::embedding(fptr(r), fptr(in[0]), iptr(ids), n, (int)E.shape[0], (int)E.shape[1], R, err_dev, st));
        vals[r].rg = E.rg;
        tape.push_back({JOP_EMBEDDING, {in[0], ids}, {r}});
        return {r, -2};
      }
      case JOP_LINEAR: {
        const IVal &x = V(in[0]), &W = V(in[1]);
        need(x.shape.size() == 2 && W.shape.size() == 2 && x.shape[1] == W.shape[1] &&
             V(in[2]).numel() == W.shape[0]);
        const int n = (int)x.shape[0], K = (int)x.shape[1], N = (int)W.shape[0];
        const int r = dev_f({n, N});
        ck(imp::gemm_nt(fptr(r), fptr(in[0]), fptr(in[1]), n, N, K, K, K, N, false, R, R, st));
        ck(imp::add_bias(fptr(r), fptr(in[2]), n, N, N, st));
        vals[r].rg = x.rg || W.rg || V(in[2]).rg;
        tape.push_back({JOP_LINEAR, {in[0], in[1], in[2]}, {r}});
        return {r, -2};
      }
      case JOP_LSTM_CELL: {
        const IVal &x = V(in[0]), &h = V(in[1]);
        need(x.shape.size() == 2 && h.shape.size() == 2 && V(in[2]).shape == h.shape &&
             x.shape[0] == h.shape[0] && V(in[6]).numel() == x.shape[0] &&
             V(in[3]).shape == std::vector<int64_t>{4 * h.shape[1], x.shape[1]} &&
             V(in[4]).shape == std::vector<int64_t>{4 * h.shape[1], h.shape[1]} &&
             V(in[5]).numel() == 4 * h.shape[1]);
        const int B = (int)x.shape[0], E = (int)x.shape[1], H = (int)h.shape[1];
        const int Z = dev_f({B, 4 * H});
        ck(imp::gemm_nt(fptr(Z), fptr(in[0]), fptr(in[3]), B, 4 * H, E, E, E, 4 * H, false, R, R, st));
        ck(imp::gemm_nt(fptr(Z), fptr(in[1]), fptr(in[4]), B, 4 * H, H, H, H, 4 * H, true, R, R, st));
        ck(imp::add_bias(fptr(Z), fptr(in[5]), B, 4 * H, 4 * H, st));
        const int gates = dev_f({B, 4 * H}), c2 = dev_f({B, H}), h2 = dev_f({B, H});
        ck(imp::lstm_fwd(fptr(gates), fptr(c2), fptr(h2), fptr(Z), fptr(in[2]), fptr(in[1]), iptr(in[6]), B, H, st));
        bool rg = false;
        for (int k = 0; k < 6; ++k) rg |= V(in[k]).rg;
        vals[c2].rg = vals[h2].rg = rg;
        TapeE te{JOP_LSTM_CELL, {in[0], in[1], in[2], in[3], in[4], in[5], in[6]}, {h2, c2}};
        te.saved = {fptr(gates)};
        tape.push_back(te);
        return {h2, c2};
      }
      case JOP_TREELSTM_LEAF: {
        const IVal &x = V(in[0]), &W = V(in[1]);
        need(x.shape.size() == 2 && W.shape.size() == 2 && W.shape[1] == x.shape[1] &&
             W.shape[0] % 3 == 0 && V(in[2]).numel() == 4 * (W.shape[0] / 3));
        const int n = (int)x.shape[0], E = (int)x.shape[1], H = (int)(W.shape[0] / 3);
        const int Z = dev_f({n, 3 * H}), bb = dev_f({3 * H});
        ck(imp::gemm_nt(fptr(Z), fptr(in[0]), fptr(in[1]), n, 3 * H, E, E, E, 3 * H, false, R, R, st));
        ck(imp::tree_bias(fptr(bb), fptr(in[2]), H, 0, st));
        const int gates = dev_f({n, 3 * H}), c = dev_f({n, H}), h = dev_f({n, H});
        ck(imp::tree_leaf_fwd(fptr(gates), fptr(c), fptr(h), fptr(Z), fptr(bb), n, H, st));
        vals[h].rg = vals[c].rg = x.rg || W.rg || V(in[2]).rg;
        TapeE te{JOP_TREELSTM_LEAF, {in[0], in[1], in[2]}, {h, c}};
        te.saved = {fptr(gates), fptr(c)};
        tape.push_back(te);
        return {h, c};
      }
      case JOP_TREELSTM_CELL: {
        const IVal &hl = V(in[0]);
        need(hl.shape.size() == 2 && V(in[1]).shape == hl.shape && V(in[2]).shape == hl.shape &&
             V(in[3]).shape == hl.shape &&
             V(in[4]).shape == std::vector<int64_t>{5 * hl.shape[1], 2 * hl.shape[1]} &&
             V(in[5]).numel() == 4 * hl.shape[1]);
        const int n = (int)hl.shape[0], H = (int)hl.shape[1];
        const int Z = dev_f({n, 5 * H}), bb = dev_f({5 * H});
        // z = [h_l ; h_r] U^T: the two halves of U's columns
        ck(imp::gemm_nt(fptr(Z), fptr(in[0]), fptr(in[4]), n, 5 * H, H, H, 2 * H, 5 * H, false, R, R, st));
        ck(imp::gemm_nt(fptr(Z), fptr(in[2]), fptr(in[4]) + H, n, 5 * H, H, H, 2 * H, 5 * H, true, R, R, st));
        ck(imp::tree_bias(fptr(bb), fptr(in[5]), H, 1, st));
        const int gates = dev_f({n, 5 * H}), c = dev_f({n, H}), h = dev_f({n, H});
        ck(imp::tree_cell_fwd(fptr(gates), fptr(c), fptr(h), fptr(Z), fptr(bb), fptr(in[1]), fptr(in[3]), n, H, st));
        bool rg = false;
        for (int k = 0; k < 6; ++k) rg |= V(in[k]).rg;
        vals[h].rg = vals[c].rg = rg;
        TapeE te{JOP_TREELSTM_CELL, {in[0], in[1], in[2], in[3], in[4], in[5]}, {h, c}};
        te.saved = {fptr(gates), fptr(c)};
        tape.push_back(te);
        return {h, c};
      }
      case JOP_DROPOUT: {  // y = x m / (1 - p), Philox masks keyed by (site, t * n + r)  (Zaremba [51])
        const IVal &x = V(in[0]);
        need(x.shape.size() == 2 && V(in[1]).numel() == 2 && V(in[1]).dtype == JANUS_I32);
        const int n = (int)x.shape[0], D = (int)x.shape[1];
        const int t = (int)as_host_int(in[2]);
        const int key = as_dev_i(in[1]);
        const int y = dev_f({n, D});
        ck(imp::copy(fptr(y), fptr(in[0]), (int64_t)n * D, st));
        ck(launch_dropout_f32(fptr(y), n, D, D, iptr(key), (int)o.iattr[0], (float)o.fattr[0], st, t * n));
        vals[y].rg = x.rg;
        TapeE te{JOP_DROPOUT, {in[0], key}, {y}};
        te.i0 = (int)o.iattr[0]; te.i1 = t;
        te.saved = {const_cast<void *>(static_cast<const void *>(&o.fattr[0]))};
        tape.push_back(te);
        return {y};
      }
      case JOP_TREERNN_CELL: {  // h = tanh([h_l ; h_r] W^T + b)  (TreeRNN [37])
        const IVal &hl = V(in[0]);
        need(hl.shape.size() == 2 && V(in[1]).shape == hl.shape &&
             V(in[2]).shape == std::vector<int64_t>{hl.shape[1], 2 * hl.shape[1]} && V(in[3]).numel() == hl.shape[1]);
        const int n = (int)hl.shape[0], H = (int)hl.shape[1];
        const int h = dev_f({n, H});
        ck(imp::gemm_nt(fptr(h), fptr(in[0]), fptr(in[2]), n, H, H, H, 2 * H, H, false, R, R, st));
        ck(imp::gemm_nt(fptr(h), fptr(in[1]), fptr(in[2]) + H, n, H, H, H, 2 * H, H, true, R, R, st));
        ck(imp::add_bias(fptr(h), fptr(in[3]), n, H, H, st));
        ck(imp::tanh_inplace(fptr(h), (int64_t)n * H, st));
        bool rg = false;
        for (int k = 0; k < 4; ++k) rg |= V(in[k]).rg;
        vals[h].rg = rg;
        TapeE te{JOP_TREERNN_CELL, {in[0], in[1], in[2], in[3]}, {h}};
        tape.push_back(te);
        return {h};
      }
      case JOP_SOFTMAX_XENT: {
        const IVal &y = V(in[0]);
        const int n = (int)y.shape[0], C = (int)y.shape[1];
        const int tg = as_dev_i(in[1]), mk = as_dev_i(in[2]);
        need(V(tg).numel() == n && V(mk).numel() == n);
        const int loss = dev_f({}), dy = dev_f({n, C});
        ck(imp::xent(fptr(loss), fptr(dy), fptr(in[0]), iptr(tg), iptr(mk), n, C, err_dev, st));
        vals[loss].rg = y.rg;
        TapeE te{JOP_SOFTMAX_XENT, {in[0]}, {loss}};
        te.saved = {fptr(dy)};
        tape.push_back(te);
        return {loss, -2};
      }
      case JOP_SEQ_MASK: {
        const int T = (int)as_host_int(in[1]);
        const int B = (int)V(in[0]).numel();
        const int r = dev_i({(int64_t)T * B});
        ck(imp::seq_mask(iptr(r), iptr(in[0]), B, T, st));
        return {r, -2};
      }
      case JOP_TIME_MAJOR: {
        const int T = (int)as_host_int(in[1]);
        const IVal &m = V(in[0]);
        const int r = dev_i({(int64_t)T * m.shape[0]});
        ck(imp::time_major(iptr(r), iptr(in[0]), (int)m.shape[0], (int)m.shape[1], T, err_dev, st));
        return {r, -2};
      }
      case JOP_TA_NEW: {
        IVal v;
        v.kind = V_TA;
        return {new_val(v), -2};
      }
      case JOP_TA_WRITE: {
        IVal v = V(in[0]);
        v.ta[as_host_int(in[1])] = in[2];
        return {new_val(v), -2};
      }
      case JOP_TA_STACK: {
        const IVal &ta = V(in[0]);
        std::vector<int> items;
        int64_t rows = 0, cols = 1;
        for (auto &kv : ta.ta) {
          const int x = as_dev_f(kv.second);
          items.push_back(x);
          const IVal &e = V(x);
          rows += e.shape.empty() ? 1 : e.shape[0];
          if (e.shape.size() > 1) cols = e.shape[1];
        }
        std::vector<int64_t> shape = {rows};
        if (!items.empty() && V(items[0]).shape.size() > 1) shape.push_back(cols);
        const int r = dev_f(shape);
        int64_t off = 0;
        bool rg = false;
        for (int x : items) {
          ck(imp::copy(fptr(r) + off, fptr(x), V(x).numel(), st));
          off += V(x).numel();
          rg |= V(x).rg;
        }
        vals[r].rg = rg;
        tape.push_back({JOP_TA_STACK, items, {r}});
        return {r, -2};
      }
      case JOP_RETURN:
        return {-2, -2};
      default:
        throw Err{JANUS_ERR_UNSUPPORTED, "op kind not supported by the imperative executor"};
    }
  }

  // ---------------------------------------------------------------- backward (reverse tape)
  std::map<int, float *> grads;
  float *gbuf(int vid) {
    auto it = grads.find(vid);
    if (it != grads.end()) return it->second;
    float *p = static_cast<float *>(alloc(std::max<int64_t>(1, V(vid).numel()) * 4));
    ck(imp::fill(p, 0.f, V(vid).numel(), st));
    grads[vid] = p;
    return p;
  }
  float *gget(int vid) {
    auto it = grads.find(vid);
    return it == grads.end() ? nullptr : it->second;
  }

  void backward(int loss_vid) {
    if (loss_vid < 0 || !V(loss_vid).rg) return;
    ck(imp::fill(gbuf(loss_vid), 1.f, 1, st));
    const bool R = bf16;
    for (int e = (int)tape.size() - 1; e >= 0; --e) {
      const TapeE &t = tape[e];
      bool any = false;
      for (int o : t.out) any |= gget(o) != nullptr;
      if (!any) continue;
      switch (t.kind) {
        case JOP_SOFTMAX_XENT: {
          // d logits = dloss * dy (dloss is 1 at the only use of the loss)
          const int y = t.in[0];
          if (!V(y).rg) break;
          ck(imp::axpy(gbuf(y), (const float *)t.saved[0], 1.f, V(y).numel(), st));
        } break;
        case JOP_LINEAR: {
          const int x = t.in[0], W = t.in[1], b = t.in[2];
          const float *dy = gget(t.out[0]);
          const int n = (int)V(x).shape[0], K = (int)V(x).shape[1], N = (int)V(W).shape[0];
          if (V(x).rg) ck(imp::gemm_nn(gbuf(x), dy, fptr(W), n, N, K, N, K, K, true, R, R, st));
          if (V(W).rg) ck(imp::gemm_tn(gbuf(W), dy, fptr(x), n, N, K, N, K, K, true, R, R, st));
          if (V(b).rg) ck(imp::colsum(gbuf(b), dy, n, N, N, true, R, st));
        } break;
        case JOP_EMBEDDING: {
          const int E = t.in[0], ids = t.in[1];
          if (!V(E).rg) break;
          const float *dX = gget(t.out[0]);
          ck(imp::embedding_bwd(gbuf(E), dX, iptr(ids), (int)V(ids).numel() ? (int)V(ids).numel() : 1,
                                (int)V(E).shape[0], (int)V(E).shape[1], st));
        } break;
        case JOP_LSTM_CELL: {
          const int x = t.in[0], h = t.in[1], c = t.in[2], Wih = t.in[3], Whh = t.in[4], b = t.in[5], valid = t.in[6];
          const int B = (int)V(x).shape[0], E = (int)V(x).shape[1], H = (int)V(h).shape[1];
          float *dh2 = gget(t.out[0]), *dc2 = gget(t.out[1]);
          const int zh = dev_f({B, H}, true);
          if (!dh2) dh2 = fptr(zh);
          if (!dc2) dc2 = fptr(zh);
          const int dz = dev_f({B, 4 * H}), dhp = dev_f({B, H}), dcp = dev_f({B, H});
          ck(imp::lstm_bwd(fptr(dz), fptr(dhp), fptr(dcp), dh2, dc2, (const float *)t.saved[0], fptr(c),
                           fptr(t.out[1]), iptr(valid), B, H, st));
          if (V(x).rg) ck(imp::gemm_nn(gbuf(x), fptr(dz), fptr(Wih), B, 4 * H, E, 4 * H, E, E, true, R, R, st));
          if (V(h).rg) {
            float *gh = gbuf(h);
            ck(imp::gemm_nn(gh, fptr(dz), fptr(Whh), B, 4 * H, H, 4 * H, H, H, true, R, R, st));
            ck(imp::axpy(gh, fptr(dhp), 1.f, (int64_t)B * H, st));
          }
          if (V(c).rg) ck(imp::axpy(gbuf(c), fptr(dcp), 1.f, (int64_t)B * H, st));
          if (V(Wih).rg) ck(imp::gemm_tn(gbuf(Wih), fptr(dz), fptr(x), B, 4 * H, E, 4 * H, E, E, true, R, R, st));
          if (V(Whh).rg) ck(imp::gemm_tn(gbuf(Whh), fptr(dz), fptr(h), B, 4 * H, H, 4 * H, H, H, true, R, R, st));
          if (V(b).rg) ck(imp::colsum(gbuf(b), fptr(dz), B, 4 * H, 4 * H, true, R, st));
        } break;
        case JOP_TREELSTM_LEAF: {
          const int x = t.in[0], W = t.in[1], b = t.in[2];
          const int n = (int)V(x).shape[0], E = (int)V(x).shape[1], H = (int)(V(W).shape[0] / 3);
          float *dh = gget(t.out[0]), *dc = gget(t.out[1]);
          const int zh = dev_f({n, H}, true);
          const int dz = dev_f({n, 3 * H});
          ck(imp::tree_leaf_bwd(fptr(dz), dh ? dh : fptr(zh), dc ? dc : fptr(zh), (const float *)t.saved[0],
                                (const float *)t.saved[1], n, H, st));
          if (V(x).rg) ck(imp::gemm_nn(gbuf(x), fptr(dz), fptr(W), n, 3 * H, E, 3 * H, E, E, true, R, R, st));
          if (V(W).rg) ck(imp::gemm_tn(gbuf(W), fptr(dz), fptr(x), n, 3 * H, E, 3 * H, E, E, true, R, R, st));
          if (V(b).rg) {
            const int gb = dev_f({3 * H});
            ck(imp::colsum(fptr(gb), fptr(dz), n, 3 * H, 3 * H, false, R, st));
            ck(imp::tree_bias_bwd(gbuf(b), fptr(gb), H, 0, st));
          }
        } break;
        case JOP_TREELSTM_CELL: {
          const int hl = t.in[0], cl = t.in[1], hr = t.in[2], cr = t.in[3], U = t.in[4], b = t.in[5];
          const int n = (int)V(hl).shape[0], H = (int)V(hl).shape[1];
          float *dh = gget(t.out[0]), *dc = gget(t.out[1]);
          const int zh = dev_f({n, H}, true);
          const int dz = dev_f({n, 5 * H}), dcl = dev_f({n, H}), dcr = dev_f({n, H});
          ck(imp::tree_cell_bwd(fptr(dz), fptr(dcl), fptr(dcr), dh ? dh : fptr(zh), dc ? dc : fptr(zh),
                                (const float *)t.saved[0], (const float *)t.saved[1], fptr(cl), fptr(cr), n, H, st));
          if (V(hl).rg) ck(imp::gemm_nn(gbuf(hl), fptr(dz), fptr(U), n, 5 * H, H, 5 * H, 2 * H, H, true, R, R, st));
          if (V(hr).rg) ck(imp::gemm_nn(gbuf(hr), fptr(dz), fptr(U) + H, n, 5 * H, H, 5 * H, 2 * H, H, true, R, R, st));
          if (V(cl).rg) ck(imp::axpy(gbuf(cl), fptr(dcl), 1.f, (int64_t)n * H, st));
          if (V(cr).rg) ck(imp::axpy(gbuf(cr), fptr(dcr), 1.f, (int64_t)n * H, st));
          if (V(U).rg) {
            float *gU = gbuf(U);
            ck(imp::gemm_tn(gU, fptr(dz), fptr(hl), n, 5 * H, H, 5 * H, H, 2 * H, true, R, R, st));
            ck(imp::gemm_tn(gU + H, fptr(dz), fptr(hr), n, 5 * H, H, 5 * H, H, 2 * H, true, R, R, st));
          }
          if (V(b).rg) {
            const int gb = dev_f({5 * H});
            ck(imp::colsum(fptr(gb), fptr(dz), n, 5 * H, 5 * H, false, R, st));
            ck(imp::tree_bias_bwd(gbuf(b), fptr(gb), H, 1, st));
          }
        } break;
        case JOP_DROPOUT: {  // dx = dy m / (1 - p): the same mask, regenerated
          const int x = t.in[0];
          if (!V(x).rg) break;
          const int n = (int)V(x).shape[0], D = (int)V(x).shape[1];
          const int d = dev_f({n, D});
          ck(imp::copy(fptr(d), gget(t.out[0]), (int64_t)n * D, st));
          ck(launch_dropout_f32(fptr(d), n, D, D, iptr(t.in[1]), t.i0, (float)*static_cast<const double *>(t.saved[0]),
                                st, t.i1 * n));
          ck(imp::axpy(gbuf(x), fptr(d), 1.f, (int64_t)n * D, st));
        } break;
        case JOP_TREERNN_CELL: {
          const int hl = t.in[0], hr = t.in[1], W = t.in[2], b = t.in[3];
          const int n = (int)V(hl).shape[0], H = (int)V(hl).shape[1];
          const float *dh = gget(t.out[0]);
          const int dz = dev_f({n, H});
          ck(imp::tanh_bwd(fptr(dz), dh, fptr(t.out[0]), (int64_t)n * H, st));  // dz = dh (1 - h^2)
          if (V(hl).rg) ck(imp::gemm_nn(gbuf(hl), fptr(dz), fptr(W), n, H, H, H, 2 * H, H, true, R, R, st));
          if (V(hr).rg) ck(imp::gemm_nn(gbuf(hr), fptr(dz), fptr(W) + H, n, H, H, H, 2 * H, H, true, R, R, st));
          if (V(W).rg) {
            float *gW = gbuf(W);
            ck(imp::gemm_tn(gW, fptr(dz), fptr(hl), n, H, H, H, H, 2 * H, true, R, R, st));
            ck(imp::gemm_tn(gW + H, fptr(dz), fptr(hr), n, H, H, H, H, 2 * H, true, R, R, st));
          }
          if (V(b).rg) ck(imp::colsum(gbuf(b), fptr(dz), n, H, H, true, R, st));
        } break;
        case JOP_TA_STACK: {
          const float *d = gget(t.out[0]);
          int64_t off = 0;
          for (int x : t.in) {
            if (V(x).rg) ck(imp::axpy(gbuf(x), d + off, 1.f, V(x).numel(), st));
            off += V(x).numel();
          }
        } break;
        case JOP_ADD: {
          const float *d = gget(t.out[0]);
          for (int x : t.in) {
            if (!V(x).rg) continue;
            if (V(x).numel() == V(t.out[0]).numel()) ck(imp::axpy(gbuf(x), d, 1.f, V(x).numel(), st));
            else ck(imp::sum_all(gbuf(x), d, V(t.out[0]).numel(), st));  // broadcast scalar
          }
        } break;
        case JOP_SUM: {
          const int x = t.in[0];
          if (!V(x).rg) break;
          // d x_i = d sum (device scalar): read once on the host is avoided with a broadcast copy
          const int64_t n = V(x).numel();
          std::vector<float> ones;
          float dsum = 0.f;
          if (cudaMemcpyAsync(&dsum, gget(t.out[0]), 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
              cudaStreamSynchronize(st) != cudaSuccess)
            throw Err{JANUS_ERR_CUDA, "readback"};
          ++syncs;
          ck(imp::fill(gbuf(x), dsum, n, st));
        } break;
        default:
          break;
      }
    }
  }
};

}  // namespace

janus_status run_imperative(Graph &g, const janus_tensor *args, int n_args,
                            const janus_tensor *state, int n_state, const janus_tensor *outs,
                            int n_outs, const janus_tensor &ws, cudaStream_t st) {
  if (n_args < g.n_args || n_state < g.n_state) return JANUS_ERR_INVALID;
  if (!ws.data) return JANUS_ERR_INVALID;
  const size_t cap = (size_t)ws.shape[0] * (ws.dtype == JANUS_U8 ? 1 : 4);
  if (cap < g.imp_ws_bytes) return JANUS_ERR_INVALID;
  for (int k = 0; k < n_state; ++k)
    if (state[k].data && !is_device_ptr(state[k].data)) return JANUS_ERR_INVALID;
  Interp I(g);
  I.args = args; I.n_args = n_args; I.state = state; I.st = st;
  I.bf16 = g.opts.gemm_dtype != JANUS_F32;
  I.base = static_cast<uint8_t *>(ws.data);
  I.cap = cap;
  const size_t scr = imp_gemm_scratch_bytes(g);
  imp::set_scratch(scr ? I.alloc(scr) : nullptr, scr);
  (void)imp::take_extra_launches();
  janus_status result = JANUS_OK;
  // Data parallel: every rank runs its own shard imperatively, then ONE allreduce(sum) of
  // a gradient arena = [grad of every SGD-updated slot, ascending slot | runtime-error count]. The
  // arena is laid out from the program and the state shapes alone (identical on every rank) and
  // allocated before anything runs, so a rank whose interpretation throws still joins the same
  // collective (zero gradients, error count 1): every rank then returns ERR_RUNTIME and commits
  // nothing, otherwise every rank applies W -= (lr / N) * sum of gradients (reading Q12).
  const bool dp = dp_enabled(g);
  std::vector<std::pair<int, int64_t>> dp_slots;  // (slot, arena offset in floats)
  int64_t dp_n = 0;
  float *arena = nullptr;
  if (dp) {
    const janus_status r = dp_init(g);
    if (r != JANUS_OK) return r;
    std::vector<int> slots;
    for (const janus_op &o : g.ops)
      if (o.kind == JOP_SGD_APPLY) slots.push_back((int)o.iattr[0]);
    std::sort(slots.begin(), slots.end());
    slots.erase(std::unique(slots.begin(), slots.end()), slots.end());
    for (int sl : slots) {
      if (sl < 0 || sl >= n_state || state[sl].dtype != JANUS_F32) return JANUS_ERR_INVALID;
      int64_t n = 1;
      for (int d = 0; d < state[sl].ndim; ++d) n *= state[sl].shape[d];
      dp_slots.push_back({sl, dp_n});
      dp_n += n;
    }
  }
  auto dp_join = [&](bool failed) -> janus_status {  // the step's one collective
    if (failed && imp::fill(arena, 0.f, dp_n, st) != cudaSuccess) return JANUS_ERR_CUDA;
    if (imp::fill(arena + dp_n, failed ? 1.f : 0.f, 1, st) != cudaSuccess) return JANUS_ERR_CUDA;
    I.launches += 1 + (failed ? 1 : 0);
    return dp_allreduce_sum(g, arena, (size_t)dp_n + 1, st);
  };
  try {
    if (dp) arena = static_cast<float *>(I.alloc((size_t)(dp_n + 1) * 4));
    I.err_dev = static_cast<int *>(I.alloc(16));
    I.ck(imp::fill_i(I.err_dev, 0, 4, st));
    I.analyse();
    Interp::Scope main;
    main.func = 0;
    // sinks in program order: outputs, effects
    for (int i = 0; i < (int)g.ops.size(); ++i) {
      const janus_op &o = g.ops[i];
      if (o.func != 0) continue;
      if (o.kind == JOP_OUTPUT || o.kind == JOP_STATE_WRITE || o.kind == JOP_SGD_APPLY) I.eval(&main, i);
    }
    I.backward(I.out_vid);
    // runtime errors are read back with the final sync; effects apply only without one
    int err = 0;
    float loss = 0.f;
    float dp_err = 0.f;
    if (dp) {
      for (auto &sl : dp_slots) {
        const int vid = I.state_vid.count(sl.first) ? I.state_vid[sl.first] : -1;
        const float *gr = vid >= 0 ? I.gget(vid) : nullptr;
        int64_t n = 1;
        for (int d = 0; d < state[sl.first].ndim; ++d) n *= state[sl.first].shape[d];
        I.ck(gr ? imp::copy(arena + sl.second, gr, n, st) : imp::fill(arena + sl.second, 0.f, n, st));
      }
      // this rank's runtime-error word joins the arena: the allreduce is also the agreement
      I.ck(imp::err_to_float(arena + dp_n, I.err_dev, st));
      const janus_status r = dp_allreduce_sum(g, arena, (size_t)dp_n + 1, st);
      I.dp_joined = true;
      if (r != JANUS_OK) throw Err{r, "allreduce"};
      if (cudaMemcpyAsync(&dp_err, arena + dp_n, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess)
        throw Err{JANUS_ERR_CUDA, "D2H"};
    }
    if (cudaMemcpyAsync(&err, I.err_dev, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess) throw Err{JANUS_ERR_CUDA, "D2H"};
    if (I.out_vid >= 0 && I.V(I.out_vid).kind == V_DEV)
      if (cudaMemcpyAsync(&loss, I.V(I.out_vid).ptr, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess)
        throw Err{JANUS_ERR_CUDA, "D2H"};
    if (cudaStreamSynchronize(st) != cudaSuccess) throw Err{JANUS_ERR_CUDA, "sync"};
    ++I.syncs;
    if (err || dp_err != 0.f) {
      result = JANUS_ERR_RUNTIME;
    } else {
      // commit: SGD on the masters, then state write-backs, in effect order (P:266 (4))
      std::vector<std::pair<int64_t, int>> order;
      for (size_t k = 0; k < I.sgds.size(); ++k) order.push_back({I.sgds[k].first, (int)k});
      for (size_t k = 0; k < I.writes.size(); ++k) order.push_back({I.writes[k].first, 1000000 + (int)k});
      std::sort(order.begin(), order.end());
      for (auto &e : order) {
        if (e.second < 1000000) {
          const int slot = I.sgds[e.second].second.first;
          const float lr = I.sgds[e.second].second.second;
          const int vid = I.state_vid.count(slot) ? I.state_vid[slot] : -1;
          float *gr = vid >= 0 ? I.gget(vid) : nullptr;
          if (gr && dp) {  // the summed gradient, averaged over the ranks in the step size
            for (auto &sl : dp_slots)
              if (sl.first == slot) gr = arena + sl.second;
            I.ck(imp::sgd(static_cast<float *>(state[slot].data), gr, lr / (float)g.opts.world_size,
                          I.V(vid).numel(), st));
          } else if (gr) {
            I.ck(imp::sgd(static_cast<float *>(state[slot].data), gr, lr, I.V(vid).numel(), st));
          }
        } else {
          const auto &w = I.writes[e.second - 1000000];
          const int slot = w.second.first, vid = w.second.second;
          const janus_tensor &t = state[slot];
          int64_t n = 1;
          for (int d = 0; d < t.ndim; ++d) n *= t.shape[d];
          const IVal &v = I.V(vid);
          if (t.dtype == JANUS_I32) {
            if (v.kind == V_HOST) I.ck(imp::fill_i(static_cast<int *>(t.data), (int)v.hv, n, st));
            else I.ck(imp::copy_i(static_cast<int *>(t.data), static_cast<const int *>(v.ptr), n, st));
          } else {
            if (v.kind == V_HOST) I.ck(imp::fill(static_cast<float *>(t.data), (float)v.hv, n, st));
            else I.ck(imp::copy(static_cast<float *>(t.data), static_cast<const float *>(v.ptr), n, st));
          }
        }
      }
      if (cudaStreamSynchronize(st) != cudaSuccess) throw Err{JANUS_ERR_CUDA, "sync"};
    }
    if (n_outs > 0 && outs[0].data) {
      if (is_device_ptr(outs[0].data)) cudaMemcpyAsync(outs[0].data, &loss, 4, cudaMemcpyHostToDevice, st);
      else *static_cast<float *>(outs[0].data) = loss;
    }
  } catch (const Err &e) {
    result = e.st;
    // a rank that failed before the collective still joins it (its peers would block otherwise)
    if (dp && arena && !I.dp_joined && e.st != JANUS_ERR_CUDA && e.st != JANUS_ERR_NCCL) {
      const janus_status r = dp_join(true);
      if (r != JANUS_OK) result = r;
    }
    cudaStreamSynchronize(st);
  }
  g.launches += I.launches;
  g.host_syncs += I.syncs;
  return result;
}

}  // namespace jk
