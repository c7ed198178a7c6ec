"""ORACLE — TEST INFRASTRUCTURE ONLY. Serial CPU interpreter of the paper's speculative-graph
semantics. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may import it; it shares no code with the CUDA path.

What it computes:
  1. guard outcomes, exactly: DISPATCH assumptions first (§3.2: checked at graph-cache
     lookup, a failure is a cache miss), then RUNTIME AssertOps (§3.2); the reported
     failure is the minimum failing id (reading Q9) with the first failing element;
  2. when every assumption holds, the result of the *generic* graph under dataflow semantics —
     Switch/Merge demux/mux with deadness, Enter/Exit/NextIteration iteration frames
     (P:222), InvokeOp recursion — which must equal imperative execution;
  3. commit or no change: effects (STATE_WRITE = PySetAttrOp local copies, P:266 (2)-(4);
     SGD_APPLY = deferred parameter update) are logged and applied in sequence order only
     after the run completes (all-or-nothing).
Gradients: reverse-mode over the trace of executed op instances (the automatically inserted
differentiation of P:154). Data parallelism: gradients averaged over ranks.

Parity note: this interpreter is deliberately plain — a fixpoint scan over (node, tag) pairs with
no scheduling cleverness — so it can be checked against the paper by eye.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np

from . import numerics as nm
from .numerics import RuntimeFault

OK, ASSUMPTION_FAILED, ERR_INVALID, ERR_UNSUPPORTED, ERR_RUNTIME = 0, 1, 2, 3, 4
DEAD = "DEAD"
_ids = itertools.count(1)


class Val:
    __slots__ = ("id", "data")

    def __init__(self, data):
        self.id = next(_ids)
        self.data = data


class TA:
    """Tensor array value: immutable map index -> Val (the `outputs += [state]` list, Fig 1)."""

    def __init__(self, items=None):
        self.items = dict(items or {})


@dataclass
class Failure:
    assumption_id: int
    rank: int
    index: int
    observed: int


@dataclass
class Result:
    status: int
    failure: Failure | None = None
    outputs: list = field(default_factory=list)
    state: list = field(default_factory=list)     # new state (copy); unchanged unless OK
    grads: dict = field(default_factory=dict)     # slot -> averaged gradient (OK only)
    trace: dict = field(default_factory=dict)     # diagnostics (trip counts, invokes)


# =============================================================================== guards
_DT = {np.dtype(np.float32): 0, np.dtype(np.int32): 2, np.dtype(np.int64): 3, np.dtype(np.uint8): 4}


def dtype_code(a):
    return _DT.get(np.asarray(a).dtype, -1)


def check_dispatch(prog, args):
    """DISPATCH assumptions in ascending id. Returns a Failure or None.
    Shape match follows Figure 4 / S:244-252: ndim equal and dims[k] in {-1, shape[k]}."""
    for a in sorted(prog.assumptions, key=lambda a: a.id):
        if a.mode != 0:
            continue
        x = args[a.target]
        if a.kind == "DTYPE_EQ":
            if dtype_code(x) != a.dtype:
                return Failure(a.id, 0, -1, dtype_code(x))
        elif a.kind == "SHAPE_MATCH":
            shp = np.shape(x)
            if len(shp) != len(a.dims):
                return Failure(a.id, 0, -1, len(shp))
            for k, (d, s) in enumerate(zip(a.dims, shp)):
                if d != -1 and d != s:
                    return Failure(a.id, 0, k, s)
        else:
            raise ValueError(a.kind)
    return None


def _first_fail(bad, vals):
    bad = np.asarray(bad).reshape(-1)
    if not bad.any():
        return None
    k = int(np.argmax(bad))
    return k, int(np.asarray(vals).reshape(-1)[k])


def tree_binary_violation(kind, left, right, word, off, V, max_nodes):
    """First element violating the TREE_BINARY assumption (janus.h). Elements 0..N-1 are nodes,
    N..N+B are tree_off entries. Returns (index, observed) or None."""
    kind, left, right, word, off = (np.asarray(x, np.int64) for x in (kind, left, right, word, off))
    N, B = len(kind), len(off) - 1
    bad = []
    # tree_off: off[0] = 0, non-decreasing by >= 1 and <= max_nodes, off[B] = N
    for t in range(B + 1):
        ok = True
        if t == 0:
            ok = off[0] == 0
        else:
            sz = off[t] - off[t - 1]
            ok = 1 <= sz <= max_nodes and (t < B or off[B] == N)
        if not ok:
            bad.append((N + t, int(off[t])))
            break
    if bad:
        return bad[0]
    tree_of = np.zeros(N, np.int64)
    for t in range(B):
        tree_of[off[t]:off[t + 1]] = t
    parents = np.zeros(N, np.int64)
    node_bad = np.zeros(N, bool)
    for n in range(N):
        lo = off[tree_of[n]]
        if kind[n] == 0:
            node_bad[n] |= not (0 <= word[n] < V)
        elif kind[n] == 1:
            l, r = left[n], right[n]
            if lo <= l < n and lo <= r < n and l != r:
                parents[l] += 1
                parents[r] += 1
            else:
                node_bad[n] = True
        else:
            node_bad[n] = True
    roots = np.zeros(N, bool)
    roots[off[1:] - 1] = True
    node_bad |= np.where(roots, parents != 0, parents != 1)
    if node_bad.any():
        n = int(np.argmax(node_bad))
        return n, int(kind[n])
    return None


def check_runtime(prog, args, state):
    """RUNTIME assumptions (AssertOps): every one is evaluated over its input data; the
    minimum failing id is reported with its first failing element (reading Q9)."""
    fails = []
    for a in sorted(prog.assumptions, key=lambda a: a.id):
        if a.mode != 1:
            continue
        r = None
        if a.kind == "TRIP_COUNT":
            x = np.asarray(args[a.target])
            r = _first_fail(x != a.value, x)
        elif a.kind == "TYPE_TAG":
            x = np.asarray(state[a.target])
            r = _first_fail(x.reshape(-1)[:1] != a.value, x)
        elif a.kind == "VALUE_EQ":
            x = np.asarray(args[a.target])
            r = _first_fail(x.reshape(-1)[:1] != a.value, x)
        elif a.kind == "BRANCH_ARM":
            # the Switch on args[target][0] (predicate = value != 0, as the SWITCH op reads it)
            # takes arm `value` (P:226-228 single-arm speculation)
            x = np.asarray(args[a.target])
            r = _first_fail((x.reshape(-1)[:1] != 0) != (a.value != 0), x)
        elif a.kind == "RANGE":
            x = np.asarray(args[a.target], np.int64)
            hi = a.hi
            if a.ref_arg >= 0:
                hi = min(hi, np.shape(args[a.ref_arg])[a.ref_dim])
            r = _first_fail((x < a.lo) | (x > hi), x)
        elif a.kind == "TREE_BINARY":
            t = a.target
            r = tree_binary_violation(*args[t:t + 5], a.hi, a.value)
        else:
            raise ValueError(a.kind)
        if r is not None:
            fails.append(Failure(a.id, 0, r[0], r[1]))
    return min(fails, key=lambda f: f.assumption_id) if fails else None


def check_guards(prog, args, state, fail_assert_id=-1, strip_asserts=False):
    f = check_dispatch(prog, args)
    if f is None and fail_assert_id >= 0:
        forced = [a for a in prog.assumptions if a.id == fail_assert_id and a.mode == 0]
        if forced:
            f = Failure(fail_assert_id, 0, -1, -1)
    if f is not None:
        return f
    f = None if strip_asserts else check_runtime(prog, args, state)
    if fail_assert_id >= 0 and any(a.id == fail_assert_id and a.mode == 1 for a in prog.assumptions):
        forced = Failure(fail_assert_id, 0, -1, -1)
        if f is None or forced.assumption_id < f.assumption_id:
            f = forced
    return f


def _frozen(a):
    """The step's view of a state slot: read-only (nothing in a step mutates its inputs; Prec
    may then round a parameter once per step)."""
    a.flags.writeable = False
    return a


# =============================================================================== tape autodiff
class Tape:
    """Trace of executed differentiable op instances; reverse pass = the inserted autodiff
    (P:154). Control-flow ops alias Vals and need no entry."""

    def __init__(self, P):
        self.P = P
        self.entries = []

    def add(self, kind, ins, outs, saved=None, attrs=None):
        self.entries.append((kind, ins, outs, saved, attrs))

    def backward(self, loss_val, skip=()):
        """skip: ids of leaf Vals whose gradient is not wanted (state slots without an SGD
        effect, e.g. C3's frozen word vectors): their VJP is not formed (nothing flows on)."""
        P = self.P
        g = {loss_val.id: np.float64(1.0)}

        def acc(v, d):
            if v is None or d is None:
                return
            g[v.id] = g[v.id] + d if v.id in g else np.array(d, dtype=np.float64)

        for kind, ins, outs, saved, attrs in reversed(self.entries):
            douts = [g.get(o.id) if o is not None else None for o in outs]
            if all(d is None for d in douts):
                continue
            if kind == "SOFTMAX_XENT":
                logits = ins[0]
                acc(logits, nm.xent_vjp(logits.data, saved, douts[0]))
            elif kind == "LINEAR":
                x, W, b = ins
                dx, dW, db = nm.linear_vjp(P, x.data, W.data, douts[0])
                acc(x, dx); acc(W, dW); acc(b, db)
            elif kind == "EMBEDDING":
                E, ids = ins
                if E.id not in skip:
                    acc(E, nm.embedding_vjp(E.data.shape, ids.data, douts[0]))
            elif kind == "LSTM_CELL":
                x, h, c, W_ih, W_hh, b = ins
                dh2 = douts[0] if douts[0] is not None else np.zeros_like(h.data, dtype=np.float64)
                dc2 = douts[1] if douts[1] is not None else np.zeros_like(c.data, dtype=np.float64)
                dx, dh, dc, dWih, dWhh, db = nm.lstm_vjp(P, saved, x.data, h.data, W_ih.data,
                                                         W_hh.data, dh2, dc2)
                acc(x, dx); acc(h, dh); acc(c, dc); acc(W_ih, dWih); acc(W_hh, dWhh); acc(b, db)
            elif kind == "TREELSTM_LEAF":
                x, W, b = ins
                dh = douts[0] if douts[0] is not None else 0.0
                dc = douts[1] if douts[1] is not None else 0.0
                H = W.data.shape[0] // 3
                dh = np.broadcast_to(dh, (x.data.shape[0], H))
                dc = np.broadcast_to(dc, (x.data.shape[0], H))
                dx, dW, db = nm.tree_leaf_vjp(P, saved, x.data, W.data, dh, dc)
                acc(x, dx); acc(W, dW); acc(b, db)
            elif kind == "TREELSTM_CELL":
                hl, cl, hr, cr, U, b = ins
                H = hl.data.shape[1]
                dh = douts[0] if douts[0] is not None else np.zeros((1, H))
                dc = douts[1] if douts[1] is not None else np.zeros((1, H))
                dhl, dcl, dhr, dcr, dU, db = nm.tree_cell_vjp(P, saved, U.data, dh, dc)
                acc(hl, dhl); acc(cl, dcl); acc(hr, dhr); acc(cr, dcr); acc(U, dU); acc(b, db)
            elif kind == "DROPOUT":
                acc(ins[0], nm.dropout_vjp(saved, douts[0]))
            elif kind == "TREERNN_CELL":
                hl, hr, W, b = ins
                dh = douts[0] if douts[0] is not None else np.zeros((1, hl.data.shape[1]))
                dhl, dhr, dW, db = nm.tree_rnn_vjp(P, saved, W.data, dh)
                acc(hl, dhl); acc(hr, dhr); acc(W, dW); acc(b, db)
            elif kind == "TA_STACK":
                # ins = element Vals in index order; each contributed `rows` rows
                d = douts[0]
                r = 0
                for v in ins:
                    k = v.data.shape[0] if np.ndim(v.data) > 0 else 1
                    acc(v, d[r:r + k].reshape(np.shape(v.data)))
                    r += k
            elif kind == "ADD":
                a, b = ins
                d = douts[0]
                for v in (a, b):
                    if v is not None:
                        acc(v, np.sum(d) if np.ndim(v.data) < np.ndim(d) else d)
            elif kind == "SUM":
                (a,) = ins
                acc(a, np.full(np.shape(a.data), douts[0]))
            else:
                raise ValueError(kind)
        return g


# =============================================================================== graph executor
def _is_float(v):
    return isinstance(v, np.ndarray) and v.dtype.kind == "f"


class GraphExec:
    """Tagged-token dataflow interpreter of one program (all function bodies)."""

    def __init__(self, prog, args, state, P, local=None):
        self.prog = prog
        self.ops = prog.ops
        self.args = args
        self.state = state
        self.P = P
        self.tape = Tape(P)
        self.local = {} if local is None else local  # local copies of state
        self.effects = []                              # (seq, kind, slot, Val, lr)
        self.outputs = {}
        self.state_vals = {}                           # slot -> Val produced by STATE_READ
        self.n_invokes = 0
        self.trip_counts = []
        self.bodies = {}
        for f in sorted({op.func for op in self.ops}):
            self.bodies[f] = self._analyse(f)

    # -- static analysis: node frame paths (which loop frames a node lives in)
    def _analyse(self, func):
        nodes = [k for k, op in enumerate(self.ops) if op.func == func]
        path = {}
        for _ in range(len(nodes) + 2):
            changed = False
            for n in nodes:
                op = self.ops[n]
                cands = []
                for (p, _port) in op.ins:
                    if p not in path:
                        continue
                    po = self.ops[p]
                    pp = path[p]
                    if po.kind == "ENTER":
                        pp = pp + (po.i[0],)
                    elif po.kind == "EXIT":
                        pp = pp[:-1]
                    cands.append(pp)
                if not op.ins:
                    cands.append(())
                if not cands:
                    continue
                best = max(cands, key=len)
                if path.get(n) != best:
                    path[n] = best
                    changed = True
            if not changed:
                break
        return nodes, path

    def run_body(self, func, inputs):
        nodes, path = self.bodies[func]
        ops = self.ops
        tok = {}          # (node, port, tag) -> Val | DEAD
        fired = set()
        tags = [()]
        ret = None

        def put(n, port, tag, v):
            tok[(n, port, tag)] = v
            if tag not in tags:
                tags.append(tag)

        def get(p, port, tag):
            po = ops[p]
            if po.kind == "ENTER" and po.i[1] == 1:      # loop-invariant Enter
                if not tag or tag[-1][0] != po.i[0]:
                    return None
                return tok.get((p, port, tag[:-1]))
            return tok.get((p, port, tag))

        def tag_ok(n, tag):
            return tuple(f for f, _ in tag) == path.get(n, None)

        progress = True
        while progress:
            progress = False
            for tag in list(tags):
                for n in nodes:
                    if (n, tag) in fired or not tag_ok(n, tag):
                        continue
                    op = ops[n]
                    vals = [get(p, port, tag) for (p, port) in op.ins]
                    if op.kind == "MERGE":
                        live = [(k, v) for k, v in enumerate(vals) if v is not None and v is not DEAD]
                        if live:
                            k, v = live[0]
                            put(n, 0, tag, v)
                            put(n, 1, tag, Val(np.array(k, np.int64)))
                        elif all(v is DEAD for v in vals):
                            put(n, 0, tag, DEAD); put(n, 1, tag, DEAD)
                        else:
                            continue
                        fired.add((n, tag)); progress = True
                        continue
                    if any(v is None for v in vals):
                        continue
                    fired.add((n, tag)); progress = True
                    if any(v is DEAD for v in vals):
                        if op.kind in ("NEXT_ITERATION", "EXIT", "OUTPUT", "STATE_WRITE",
                                       "SGD_APPLY", "RETURN"):
                            continue           # dead tokens are not forwarded out of frames
                        nports = 2 if op.kind in ("SWITCH", "LSTM_CELL", "TREELSTM_LEAF",
                                                  "TREELSTM_CELL", "INVOKE") else 1
                        for p_ in range(nports):
                            put(n, p_, tag, DEAD)
                        continue
                    r = self._fire(n, op, vals, tag, inputs, put)
                    if op.kind == "RETURN":
                        ret = r
        return ret

    def _fire(self, n, op, vals, tag, inputs, put):
        P, k = self.P, op.kind
        d = [v.data for v in vals]
        if k == "ARG":
            put(n, 0, tag, inputs[op.i[0]] if op.func > 0 else Val(np.asarray(self.args[op.i[0]])))
        elif k == "CONST":
            dt = np.int64 if op.i[0] == 2 else np.float64
            put(n, 0, tag, Val(np.array(op.f[0], dt)))
        elif k == "STATE_READ":
            slot = op.i[0]
            if slot in self.local:
                v = self.local[slot]
            else:
                raw = np.asarray(self.state[slot])
                v = Val(_frozen(raw.astype(np.float64) if raw.dtype.kind == "f" else raw.astype(np.int64)))
            self.state_vals[slot] = v
            put(n, 0, tag, v)
        elif k == "STATE_WRITE":
            self.local[op.i[0]] = vals[0]
            self.effects.append((op.i[1], "write", op.i[0], vals[0], 0.0))
        elif k == "SGD_APPLY":
            self.effects.append((op.i[1], "sgd", op.i[0], vals[0], op.f[0]))
        elif k == "OUTPUT":
            self.outputs[op.i[0]] = vals[0]
        elif k in ("ADD", "LESS", "EQ"):
            a, b = d
            if k == "ADD":
                out = Val(a + b)
                if _is_float(out.data):
                    self.tape.add("ADD", [v if _is_float(v.data) else None for v in vals], [out])
            elif k == "LESS":
                out = Val((a < b).astype(np.int64))
            else:
                out = Val((a == b).astype(np.int64))
            put(n, 0, tag, out)
        elif k == "LEN":                               # whitelisted len
            put(n, 0, tag, Val(np.array(len(d[0]), np.int64)))
        elif k == "MAX_REDUCE":
            put(n, 0, tag, Val(np.array(np.max(d[0]), np.int64)))
        elif k == "SUM":
            out = Val(np.array(np.sum(d[0]), np.float64))
            self.tape.add("SUM", [vals[0]], [out])
            put(n, 0, tag, out)
        elif k == "ZEROS_LIKE":
            put(n, 0, tag, Val(np.zeros_like(d[0])))
        elif k == "COLUMN":
            t = int(d[1])
            if not 0 <= t < d[0].shape[1]:
                raise RuntimeFault("column index out of range")
            put(n, 0, tag, Val(np.ascontiguousarray(d[0][:, t])))
        elif k == "ELEMENT":
            i = int(d[1])
            if not 0 <= i < len(d[0]):
                raise RuntimeFault(f"element index {i} out of range")
            put(n, 0, tag, Val(np.array(d[0][i])))
        elif k == "EMBEDDING":
            out = Val(nm.embedding_fwd(P, d[0], d[1]))
            self.tape.add("EMBEDDING", [vals[0], vals[1]], [out])
            put(n, 0, tag, out)
        elif k == "LINEAR":
            out = Val(nm.linear_fwd(P, *d))
            self.tape.add("LINEAR", vals, [out])
            put(n, 0, tag, out)
        elif k == "LSTM_CELL":
            h2, c2, saved = nm.lstm_fwd(P, *d)
            oh, oc = Val(h2), Val(c2)
            self.tape.add("LSTM_CELL", vals[:6], [oh, oc], saved)
            put(n, 0, tag, oh); put(n, 1, tag, oc)
        elif k == "TREELSTM_LEAF":
            h, c, saved = nm.tree_leaf_fwd(P, *d)
            oh, oc = Val(h), Val(c)
            self.tape.add("TREELSTM_LEAF", vals, [oh, oc], saved)
            put(n, 0, tag, oh); put(n, 1, tag, oc)
        elif k == "TREELSTM_CELL":
            h, c, saved = nm.tree_cell_fwd(P, *d)
            oh, oc = Val(h), Val(c)
            self.tape.add("TREELSTM_CELL", vals, [oh, oc], saved)
            put(n, 0, tag, oh); put(n, 1, tag, oc)
        elif k == "DROPOUT":  # in0 x [B, D], in1 key i32[2], in2 step t; rows t * B + b
            x, key, t = d[0], d[1], int(d[2])
            rows = t * x.shape[0] + np.arange(x.shape[0])
            y, saved = nm.dropout_fwd(x, key, op.i[0], rows, op.f[0])
            out = Val(y)
            self.tape.add("DROPOUT", [vals[0]], [out], saved)
            put(n, 0, tag, out)
        elif k == "TREERNN_CELL":
            h, saved = nm.tree_rnn_fwd(P, *d)
            oh = Val(h)
            self.tape.add("TREERNN_CELL", vals, [oh], saved)
            put(n, 0, tag, oh)
        elif k == "SOFTMAX_XENT":
            loss, saved = nm.xent_fwd(*d)
            out = Val(np.array(loss))
            self.tape.add("SOFTMAX_XENT", vals, [out], saved)
            put(n, 0, tag, out)
        elif k == "SEQ_MASK":
            lens, T = d[0], int(d[1])
            put(n, 0, tag, Val((np.arange(T)[:, None] < lens[None, :]).astype(np.int64).reshape(-1)))
        elif k == "TIME_MAJOR":
            m, T = d[0], int(d[1])
            if T > m.shape[1]:
                raise RuntimeFault("TIME_MAJOR beyond width")
            put(n, 0, tag, Val(np.ascontiguousarray(m[:, :T].T).reshape(-1).astype(np.int64)))
        elif k == "TA_NEW":
            put(n, 0, tag, Val(TA()))
        elif k == "TA_WRITE":
            ta = TA(d[0].items)
            ta.items[int(d[1])] = vals[2]
            put(n, 0, tag, Val(ta))
        elif k == "TA_STACK":
            items = [d[0].items[i] for i in sorted(d[0].items)]
            data = (np.concatenate([np.atleast_1d(v.data) for v in items], axis=0) if items
                    else np.zeros((0,), np.float64))
            out = Val(data)
            self.tape.add("TA_STACK", items, [out])
            put(n, 0, tag, out)
        elif k == "SWITCH":
            pred = int(np.asarray(d[1]).reshape(-1)[0]) != 0
            put(n, 1 if pred else 0, tag, vals[0])
            put(n, 0 if pred else 1, tag, DEAD)
        elif k == "ENTER":
            F = op.i[0]
            if op.i[1] == 1:
                put(n, 0, tag, vals[0])
            else:
                put(n, 0, tag + ((F, 0),), vals[0])
        elif k == "EXIT":
            put(n, 0, tag[:-1], vals[0])
            self.trip_counts.append(tag[-1][1])
        elif k == "NEXT_ITERATION":
            F, it = tag[-1]
            put(n, 0, tag[:-1] + ((F, it + 1),), vals[0])
        elif k in ("LOOP_COND", "IDENTITY"):
            put(n, 0, tag, vals[0])
        elif k == "INVOKE":
            self.n_invokes += 1
            outs = self.run_body(op.i[0], vals)
            for p_, v in enumerate(outs):
                put(n, p_, tag, v)
        elif k == "RETURN":
            return vals
        else:
            raise ValueError(k)
        return None


# =============================================================================== commit
def clip_scale(prog, effects, grads, n_ranks):
    """Global gradient-norm clipping (reading R15: Zaremba et al. [51], the LM P:312 follows,
    clip the gradient's global L2 norm; janus_build_opts.clip_norm = c, 0 = off): with G the
    rank-averaged gradient of every parameter the step updates, the update uses
    g * min(1, c / ||G||_2) — i.e. c / ||G|| when ||G|| > c, else the gradient unchanged."""
    c = float(prog.meta.get("clip_norm", 0.0) or 0.0)
    slots = sorted({e[2] for e in effects if e[1] == "sgd"})
    if c <= 0 or not slots:
        return 1.0
    sq = sum(float(np.sum((np.asarray(grads[k], np.float64) / n_ranks) ** 2)) for k in slots)
    norm = np.sqrt(sq)
    return c / norm if norm > c else 1.0


def _commit(prog, state, effects, grads, n_ranks):
    """Apply the effect log in sequence order (P:266 (4)): SGD on the fp32 master with the
    rank-averaged gradient (reading Q13), scaled by the global-norm clip (R15), then state
    write-backs."""
    new = [np.array(s, copy=True) for s in state]
    scale = clip_scale(prog, effects, grads, n_ranks)
    for seq, kind, slot, v, lr in sorted(effects, key=lambda e: e[0]):
        if kind == "sgd":
            g = grads[slot] / n_ranks
            new[slot] = (new[slot].astype(np.float64) - (lr * scale) * g).astype(new[slot].dtype)
        else:
            new[slot] = np.asarray(v.data).astype(new[slot].dtype).reshape(new[slot].shape)
    return new


def _forward_backward(prog, args, state, P):
    ex = GraphExec(prog, args, state, P)
    ex.run_body(0, None)
    loss_val = ex.outputs.get(0)
    grads = {}
    sgd_slots = [e[2] for e in ex.effects if e[1] == "sgd"]
    if sgd_slots:
        g = ex.tape.backward(loss_val, {v.id for s, v in ex.state_vals.items() if s not in sgd_slots})
        for s in sgd_slots:
            v = ex.state_vals.get(s)
            gd = g.get(v.id) if v is not None else None
            grads[s] = np.zeros(np.shape(state[s])) if gd is None else np.asarray(gd).reshape(np.shape(state[s]))
    return ex, grads


def run_graph_step(prog, args, state, mode="bf16", fail_assert_id=-1, strip_asserts=False):
    """One step of the speculative graph (janus_run semantics) on one rank."""
    return run_dp_step(prog, [args], [state], mode, fail_assert_id, strip_asserts)[0]


def run_dp_step(prog, shard_args, shard_states, mode="bf16", fail_assert_id=-1, strip_asserts=False):
    """DP emulation (reading Q12/Q13): every rank checks its guards; any failure aborts every
    rank (minimum (id, rank)); otherwise gradients are summed over ranks, divided by N, and each
    rank commits. Returns one Result per rank."""
    P = nm.Prec(mode)
    N = len(shard_args)
    fails = []
    for r, (a, s) in enumerate(zip(shard_args, shard_states)):
        f = check_guards(prog, a, s, fail_assert_id, strip_asserts)
        if f is not None:
            f.rank = r
            fails.append(f)
    if fails:
        f = min(fails, key=lambda f: (f.assumption_id, f.rank))
        return [Result(ASSUMPTION_FAILED, f, [], [np.array(x, copy=True) for x in s])
                for s in shard_states]
    try:
        runs = [_forward_backward(prog, a, s, P) for a, s in zip(shard_args, shard_states)]
    except RuntimeFault as e:
        return [Result(ERR_RUNTIME, None, [], [np.array(x, copy=True) for x in s],
                       trace={"error": str(e)}) for s in shard_states]
    tot = {}
    for _, g in runs:
        for s, v in g.items():
            tot[s] = tot[s] + v if s in tot else v.copy()
    out = []
    for (ex, _), s in zip(runs, shard_states):
        new = _commit(prog, s, ex.effects, tot, N)
        outs = [np.asarray(ex.outputs[k].data) for k in sorted(ex.outputs)]
        out.append(Result(OK, None, outs, new, {k: v / N for k, v in tot.items()},
                          {"trip_counts": ex.trip_counts, "invokes": ex.n_invokes}))
    return out


# =============================================================================== imperative
def run_imperative_step(prog, args, state, mode="bf16"):
    """The imperative program the graph was generated from, run directly with Python control flow
    (TF-Eager analogue; O5): no assumptions, effects applied at the end, gradients
    from the same reverse pass. Implemented for the programs of workloads.programs."""
    P = nm.Prec(mode)
    model = prog.meta["model"]
    tape = Tape(P)
    sv = {k: Val(_frozen(np.asarray(s).astype(np.float64) if np.asarray(s).dtype.kind == "f"
                         else np.asarray(s).astype(np.int64))) for k, s in enumerate(state)}
    sid = {s.name: k for k, s in enumerate(prog.slots)}
    writes = {}
    update = True
    try:
        if model == "lstm_lm":
            loss = _imp_lstm_lm(prog, args, sv, sid, tape, P, writes)
            if prog.meta.get("training_flag"):          # `if training:` around the update
                update = int(np.asarray(args[3]).reshape(-1)[0]) != 0
        elif model == "treelstm":
            loss = _imp_treelstm(prog, args, sv, sid, tape, P)
        elif model == "treernn":
            loss = _imp_treernn(prog, args, sv, sid, tape, P)
        elif model == "running_sum":
            seq = np.asarray(args[0], np.float64)
            s = sv[0]
            outs = []
            for item in seq:
                s2 = Val(s.data + item)
                tape.add("ADD", [s, None], [s2])
                s = s2
                outs.append(s)
            st = Val(np.concatenate([np.atleast_1d(v.data) for v in outs]) if outs else np.zeros(0))
            tape.add("TA_STACK", outs, [st])
            loss = Val(np.array(np.sum(st.data)))
            tape.add("SUM", [st], [loss])
            writes[0] = s
        else:
            raise ValueError(model)
    except RuntimeFault as e:
        return Result(ERR_RUNTIME, None, [], [np.array(x, copy=True) for x in state],
                      trace={"error": str(e)})
    effects = []
    grads = {}
    params = [k for k, s in enumerate(prog.slots) if s.param] if update else []
    if params:
        g = tape.backward(loss, {sv[k].id for k in sv if k not in params})
        for k in params:
            gd = g.get(sv[k].id)
            grads[k] = np.zeros(np.shape(state[k])) if gd is None else np.asarray(gd).reshape(np.shape(state[k]))
            effects.append((k, "sgd", k, None, prog.lr))
    for k, v in writes.items():
        effects.append((1000 + k, "write", k, v, 0.0))
    new = _commit(prog, state, effects, grads, 1)
    return Result(OK, None, [np.asarray(loss.data)], new, grads)


def _imp_lstm_lm(prog, args, sv, sid, tape, P, writes):
    m = prog.meta
    L = m["L"]
    tok, tgt, lens = (np.asarray(a, np.int64) for a in args[:3])
    is_tensor = int(sv[sid["tag"]].data.reshape(-1)[0]) == 1
    h = [sv[sid[f"h{l}"]] if is_tensor else Val(np.zeros_like(sv[sid[f"h{l}"]].data)) for l in range(L)]
    c = [sv[sid[f"c{l}"]] if is_tensor else Val(np.zeros_like(sv[sid[f"c{l}"]].data)) for l in range(L)]
    T = int(lens.max())
    outs = []
    E = sv[sid["E"]]
    pdrop = m.get("dropout", 0.0)
    key = np.asarray(args[m["key_arg"]]).reshape(-1) if pdrop else None
    B = tok.shape[0]

    def drop(x, site, t):  # x = dropout(x) on a non-recurrent connection (Zaremba [51])
        if not pdrop:
            return x
        y, saved = nm.dropout_fwd(x.data, key, site, t * B + np.arange(B), pdrop)
        out = Val(y)
        tape.add("DROPOUT", [x], [out], saved)
        return out

    for t in range(T):
        ids = Val(tok[:, t])
        x = Val(nm.embedding_fwd(P, E.data, ids.data))
        tape.add("EMBEDDING", [E, ids], [x])
        x = drop(x, 0, t)
        valid = (t < lens).astype(np.int64)
        for l in range(L):
            W_ih, W_hh, b = sv[sid[f"W_ih{l}"]], sv[sid[f"W_hh{l}"]], sv[sid[f"b{l}"]]
            h2, c2, saved = nm.lstm_fwd(P, x.data, h[l].data, c[l].data, W_ih.data, W_hh.data, b.data, valid)
            oh, oc = Val(h2), Val(c2)
            tape.add("LSTM_CELL", [x, h[l], c[l], W_ih, W_hh, b], [oh, oc], saved)
            h[l], c[l] = oh, oc
            x = drop(oh, l + 1, t)
        outs.append(x)
    st = Val(np.concatenate([v.data for v in outs], axis=0))
    tape.add("TA_STACK", outs, [st])
    W, b = sv[sid["W_dec"]], sv[sid["b_dec"]]
    logits = Val(nm.linear_fwd(P, st.data, W.data, b.data))
    tape.add("LINEAR", [st, W, b], [logits])
    mask = (np.arange(T)[:, None] < lens[None, :]).reshape(-1)
    tgt_tm = tgt[:, :T].T.reshape(-1)
    lv, saved = nm.xent_fwd(logits.data, tgt_tm, mask)
    loss = Val(np.array(lv))
    tape.add("SOFTMAX_XENT", [logits, None, None], [loss], saved)
    for l in range(L):
        writes[sid[f"h{l}"]] = h[l]
        writes[sid[f"c{l}"]] = c[l]
    writes[sid["tag"]] = Val(np.array([1]))
    return loss


def _imp_treelstm(prog, args, sv, sid, tape, P):
    kind, left, right, word, off, label = (np.asarray(a, np.int64) for a in args)
    E, W_leaf, U, b = (sv[sid[k]] for k in ("E", "W_leaf", "U", "b"))

    def node(n):                                  # recursion = InvokeOp
        if not 0 <= n < len(kind):
            raise RuntimeFault("node id out of range")
        if kind[n] == 0:
            ids = Val(np.array([word[n]]))
            x = Val(nm.embedding_fwd(P, E.data, ids.data))
            tape.add("EMBEDDING", [E, ids], [x])
            h, c, saved = nm.tree_leaf_fwd(P, x.data, W_leaf.data, b.data)
            oh, oc = Val(h), Val(c)
            tape.add("TREELSTM_LEAF", [x, W_leaf, b], [oh, oc], saved)
            return oh, oc
        hl, cl = node(int(left[n]))
        hr, cr = node(int(right[n]))
        h, c, saved = nm.tree_cell_fwd(P, hl.data, cl.data, hr.data, cr.data, U.data, b.data)
        oh, oc = Val(h), Val(c)
        tape.add("TREELSTM_CELL", [hl, cl, hr, cr, U, b], [oh, oc], saved)
        return oh, oc

    roots = [node(int(off[i + 1]) - 1)[0] for i in range(len(off) - 1)]
    st = Val(np.concatenate([v.data for v in roots], axis=0))
    tape.add("TA_STACK", roots, [st])
    W, bc = sv[sid["W_c"]], sv[sid["b_c"]]
    logits = Val(nm.linear_fwd(P, st.data, W.data, bc.data))
    tape.add("LINEAR", [st, W, bc], [logits])
    lv, saved = nm.xent_fwd(logits.data, label, np.ones(len(label)))
    loss = Val(np.array(lv))
    tape.add("SOFTMAX_XENT", [logits, None, None], [loss], saved)
    return loss


def _imp_treernn(prog, args, sv, sid, tape, P):
    kind, left, right, word, off, label = (np.asarray(a, np.int64) for a in args)
    E, W, b = (sv[sid[k]] for k in ("E", "W", "b"))

    def node(n):                                  # recursion = InvokeOp
        if not 0 <= n < len(kind):
            raise RuntimeFault("node id out of range")
        if kind[n] == 0:                          # a leaf is its word vector
            ids = Val(np.array([word[n]]))
            x = Val(nm.embedding_fwd(P, E.data, ids.data))
            tape.add("EMBEDDING", [E, ids], [x])
            return x
        hl = node(int(left[n]))
        hr = node(int(right[n]))
        h, saved = nm.tree_rnn_fwd(P, hl.data, hr.data, W.data, b.data)
        oh = Val(h)
        tape.add("TREERNN_CELL", [hl, hr, W, b], [oh], saved)
        return oh

    roots = [node(int(off[i + 1]) - 1) for i in range(len(off) - 1)]
    st = Val(np.concatenate([v.data for v in roots], axis=0))
    tape.add("TA_STACK", roots, [st])
    Wc, bc = sv[sid["W_c"]], sv[sid["b_c"]]
    logits = Val(nm.linear_fwd(P, st.data, Wc.data, bc.data))
    tape.add("LINEAR", [st, Wc, bc], [logits])
    lv, saved = nm.xent_fwd(logits.data, label, np.ones(len(label)))
    loss = Val(np.array(lv))
    tape.add("SOFTMAX_XENT", [logits, None, None], [loss], saved)
    return loss


# =============================================================================== tree schedule
def tree_schedule(kind, left, right, off):
    """Level schedule of a forest (reading Q8): height = 0 for leaves, 1 + max(children) for
    internal nodes (computed by recursion); order = stable sort of node ids by height;
    level_offset[l] = #nodes with height < l; pos = index in order - level_offset[height];
    internal rank = rank among internal nodes in the same order; parent slot of a non-root node =
    (internal rank of its parent, side 0 = left / 1 = right). Root slots are (-1, -1)."""
    kind, left, right, off = (np.asarray(x, np.int64) for x in (kind, left, right, off))
    N = len(kind)
    height = np.full(N, -1, np.int64)

    def hgt(n):
        if height[n] < 0:
            height[n] = 0 if kind[n] == 0 else 1 + max(hgt(left[n]), hgt(right[n]))
        return height[n]

    for t in range(len(off) - 1):
        hgt(int(off[t + 1]) - 1)
    order = np.array(sorted(range(N), key=lambda n: (height[n], n)), np.int64)
    Lmax = int(height.max()) if N else 0
    level_offset = np.array([int((height < l).sum()) for l in range(Lmax + 2)], np.int64)
    pos = np.zeros(N, np.int64)
    for k, n in enumerate(order):
        pos[n] = k - level_offset[height[n]]
    internal = [n for n in order if kind[n] == 1]
    irank = np.full(N, -1, np.int64)
    for k, n in enumerate(internal):
        irank[n] = k
    pslot = np.full((N, 2), -1, np.int64)
    for n in range(N):
        if kind[n] == 1:
            pslot[left[n]] = (irank[n], 0)
            pslot[right[n]] = (irank[n], 1)
    return dict(height=height, order=order, level_offset=level_offset, pos=pos, irank=irank,
                parent_slot=pslot)
