"""Op-list constructors for the imperative programs the paper converts (inputs, not arithmetic).

Each constructor returns a `Program`: the *generic* symbolic graph of one training step, written
with the paper's conversion rules (§4.1 basics; §4.2.1 Switch/Merge, loop
frames, InvokeOp; §4.2.3 state read/write; §3.1 inserted parameter updates), plus
the speculative assumptions under which the graph path may specialise it.

This module holds no arithmetic of the method. Both the oracle (`oracle/`) and the CUDA path (via
the C ABI, `paper_1812_01329_b200.janus`) consume the same Program objects, like the seeded data
from `workloads.gen`.
"""
from __future__ import annotations

from dataclasses import dataclass, field

# dtype codes (janus.h janus_dtype)
F32, BF16, I32, I64, U8 = 0, 1, 2, 3, 4
DTYPE_NAMES = {F32: "f32", BF16: "bf16", I32: "i32", I64: "i64", U8: "u8"}

OP_KINDS = [
    "ARG", "CONST", "STATE_READ", "STATE_WRITE", "OUTPUT",
    "ADD", "LESS", "EQ", "MAX_REDUCE", "SUM", "ZEROS_LIKE",
    "COLUMN", "ELEMENT",
    "EMBEDDING", "LINEAR", "LSTM_CELL", "TREELSTM_LEAF",
    "TREELSTM_CELL", "SOFTMAX_XENT", "SEQ_MASK", "TIME_MAJOR",
    "TA_NEW", "TA_WRITE", "TA_STACK",
    "SWITCH", "MERGE", "ENTER", "EXIT", "NEXT_ITERATION",
    "LOOP_COND", "IDENTITY", "INVOKE", "RETURN",
    "SGD_APPLY", "LEN", "TREERNN_CELL", "DROPOUT",
]
OP_CODE = {k: i for i, k in enumerate(OP_KINDS)}

ASM_KINDS = ["DTYPE_EQ", "SHAPE_MATCH", "TRIP_COUNT", "TYPE_TAG", "RANGE", "TREE_BINARY", "VALUE_EQ",
             "BRANCH_ARM"]
ASM_CODE = {k: i for i, k in enumerate(ASM_KINDS)}
DISPATCH, RUNTIME = 0, 1

TAG_NONE, TAG_TENSOR = 0, 1  # type tag of a state slot (objects vs tensors)


@dataclass
class Op:
    kind: str
    ins: list = field(default_factory=list)  # [(node, port)]
    i: list = field(default_factory=list)    # integer attributes
    f: list = field(default_factory=list)    # float attributes
    func: int = 0


@dataclass
class Assumption:
    id: int
    kind: str
    mode: int
    target: int
    dtype: int = 0
    dims: tuple = ()
    lo: int = 0
    hi: int = 0
    value: int = 0
    ref_arg: int = -1
    ref_dim: int = -1


@dataclass
class Slot:
    name: str
    dtype: int
    shape: tuple
    param: bool = False  # updated by SGD_APPLY


@dataclass
class Program:
    name: str
    ops: list
    assumptions: list
    slots: list          # state slots, index = slot id
    args: list           # [(name, dtype, shape or None)]
    n_outputs: int
    lr: float
    meta: dict = field(default_factory=dict)

    def slot_index(self, name):
        return [s.name for s in self.slots].index(name)


class _G:
    """Tiny graph builder: node ids are positions in `ops`."""

    def __init__(self):
        self.ops: list[Op] = []
        self.func = 0
        self.seq = 0

    def op(self, kind, ins=(), i=(), f=()):
        ins = [x if isinstance(x, tuple) else (x, 0) for x in ins]
        self.ops.append(Op(kind, list(ins), list(i), list(f), self.func))
        return len(self.ops) - 1

    def effect_seq(self):
        self.seq += 1
        return self.seq

    def patch_input(self, node, k, src):
        self.ops[node].ins[k] = src if isinstance(src, tuple) else (src, 0)


def _state_read(g, slot_id, slot):
    dims = list(slot.shape) + [0] * (4 - len(slot.shape))
    return g.op("STATE_READ", i=[slot_id, slot.dtype, len(slot.shape)] + dims)


# ------------------------------------------------------------------------------------------------
# LSTM language model — the Figure 1 program with the PTB LSTM of Table 2.
# ------------------------------------------------------------------------------------------------
def lstm_lm_slots(V, E, H, L, B):
    slots = [Slot("E", F32, (V, E), True)]
    for l in range(L):
        In = E if l == 0 else H
        slots += [Slot(f"W_ih{l}", F32, (4 * H, In), True), Slot(f"W_hh{l}", F32, (4 * H, H), True),
                  Slot(f"b{l}", F32, (4 * H,), True)]
    slots += [Slot("W_dec", F32, (V, H), True), Slot("b_dec", F32, (V,), True)]
    for l in range(L):
        slots += [Slot(f"h{l}", F32, (B, H)), Slot(f"c{l}", F32, (B, H))]
    slots += [Slot("tag", I32, (1,))]
    return slots


def lstm_lm_program(V, E, H, L, B, T, lr, *, speculate="unroll", gemm="bf16", max_T=None,
                    training_flag=False, dropout=0.0, flag_speculation="value", clip_norm=0.0):
    """Generic graph of one truncated-BPTT step of the Figure 1 RNN model:

        state = self.state (zeros if it is still None)          # attribute read, P:266 (1)
        for t < max(lengths):                                   # loop frame
            x = embedding(tokens[:, t]); for l: h_l, c_l = lstm_cell(...)  (rows t >= len keep h,c)
            outputs += [h_L]
        self.state = state                                      # deferred write, P:266 (2),(4)
        loss = compute_loss(outputs); optimizer update           # P:154 inserted updates

    Arguments: 0 tokens i32[B,W], 1 targets i32[B,W], 2 lengths i32[B]; with training_flag also
    3 training i32[1]: the optimizer update runs only `if training:` (the train / evaluate branch
    of P:312), speculated on its profiled value (constant promotion) by a RUNTIME VALUE_EQ
    assumption (id 8): the single taken arm is kept and asserted; with
    flag_speculation="branch" the assumption is BRANCH_ARM instead — the Switch takes its true arm
    (any non-zero flag), the control-flow speculation itself rather than the value.
    dropout = p > 0: the Zaremba et al. [51] regularised model (PTB medium: H = 650, p =
    0.5): dropout on every non-recurrent connection — the embedding output, each layer's output
    into the next layer and the top layer's output into the decoder (DROPOUT sites 0 .. L) — with
    masks drawn by Philox4x32-10 from a per-step key argument i32[2] (the last argument).
    speculate: "unroll" — fixed trip count T (C1/C2: TRIP_COUNT assumption, unrolled graph);
               "while"  — variable trip count (C4: device-resident While, RANGE assumption);
               "none"   — no RUNTIME assumptions (imperative path only).
    """
    slots = lstm_lm_slots(V, E, H, L, B)
    sid = {s.name: k for k, s in enumerate(slots)}
    g = _G()
    tok = g.op("ARG", i=[0])
    tgt = g.op("ARG", i=[1])
    lens = g.op("ARG", i=[2])
    rd = {s.name: _state_read(g, k, s) for k, s in enumerate(slots)}
    zero = g.op("CONST", i=[I32], f=[0.0])
    one = g.op("CONST", i=[I32], f=[1.0])
    tag_tensor = g.op("CONST", i=[I32], f=[float(TAG_TENSOR)])
    is_tensor = g.op("EQ", [rd["tag"], tag_tensor])
    init = {}
    for l in range(L):
        for nm in (f"h{l}", f"c{l}"):
            sw = g.op("SWITCH", [rd[nm], is_tensor])
            z = g.op("ZEROS_LIKE", [(sw, 0)])
            init[nm] = g.op("MERGE", [(sw, 1), z])
    T_b = g.op("MAX_REDUCE", [lens])
    acc0 = g.op("TA_NEW")
    FR = 1
    # loop frame: Enter / Merge / LoopCond / Switch / body / NextIteration / Exit
    e_t = g.op("ENTER", [zero], i=[FR, 0])
    e_state = {nm: g.op("ENTER", [init[nm]], i=[FR, 0]) for nm in init}
    e_acc = g.op("ENTER", [acc0], i=[FR, 0])
    inv = {}
    key_arg = 4 if training_flag else 3
    extra = [("key", g.op("ARG", i=[key_arg]))] if dropout else []
    for nm, src in [("T_b", T_b), ("tok", tok), ("lens", lens), ("one", one), ("E", rd["E"])] + extra + \
            [(f"{p}{l}", rd[f"{p}{l}"]) for l in range(L) for p in ("W_ih", "W_hh", "b")]:
        inv[nm] = g.op("ENTER", [src], i=[FR, 1])

    def drop(x, site):  # dropout on a non-recurrent connection, masks keyed by (site, t * B + b)
        return (g.op("DROPOUT", [x, inv["key"], t], i=[site], f=[dropout]), 0) if dropout else x
    m_t = g.op("MERGE", [e_t, e_t])  # second input patched to the NextIteration below
    m_state = {nm: g.op("MERGE", [e_state[nm], e_state[nm]]) for nm in init}
    m_acc = g.op("MERGE", [e_acc, e_acc])
    cond = g.op("LESS", [m_t, inv["T_b"]])
    lc = g.op("LOOP_COND", [cond])
    s_t = g.op("SWITCH", [m_t, lc])
    s_state = {nm: g.op("SWITCH", [m_state[nm], lc]) for nm in init}
    s_acc = g.op("SWITCH", [m_acc, lc])
    t = (s_t, 1)
    tok_t = g.op("COLUMN", [inv["tok"], t])
    valid = g.op("LESS", [t, inv["lens"]])
    x = drop((g.op("EMBEDDING", [inv["E"], tok_t]), 0), 0)
    new_state = {}
    for l in range(L):
        cell = g.op("LSTM_CELL", [x, (s_state[f"h{l}"], 1), (s_state[f"c{l}"], 1), inv[f"W_ih{l}"],
                                  inv[f"W_hh{l}"], inv[f"b{l}"], valid])
        new_state[f"h{l}"], new_state[f"c{l}"] = (cell, 0), (cell, 1)
        x = drop((cell, 0), l + 1)
    acc1 = g.op("TA_WRITE", [(s_acc, 1), t, x])
    t1 = g.op("ADD", [t, inv["one"]])
    ni_t = g.op("NEXT_ITERATION", [t1])
    g.patch_input(m_t, 1, ni_t)
    for nm in init:
        ni = g.op("NEXT_ITERATION", [new_state[nm]])
        g.patch_input(m_state[nm], 1, ni)
    ni_acc = g.op("NEXT_ITERATION", [acc1])
    g.patch_input(m_acc, 1, ni_acc)
    x_state = {nm: g.op("EXIT", [(s_state[nm], 0)]) for nm in init}
    x_acc = g.op("EXIT", [(s_acc, 0)])
    outs = g.op("TA_STACK", [x_acc])
    mask = g.op("SEQ_MASK", [lens, T_b])
    tgt_tm = g.op("TIME_MAJOR", [tgt, T_b])
    logits = g.op("LINEAR", [outs, rd["W_dec"], rd["b_dec"]])
    loss = g.op("SOFTMAX_XENT", [logits, tgt_tm, mask])
    g.op("OUTPUT", [loss], i=[0])
    upd = loss
    if training_flag:                        # if training: optimizer.apply(...)  (Switch)
        train = g.op("ARG", i=[3])
        pred = g.op("ELEMENT", [train, zero])
        upd = (g.op("SWITCH", [loss, pred]), 1)
    for s in slots:
        if s.param:
            g.op("SGD_APPLY", [upd], i=[sid[s.name], g.effect_seq()], f=[lr])
    for nm in init:
        g.op("STATE_WRITE", [x_state[nm]], i=[sid[nm], g.effect_seq()])
    g.op("STATE_WRITE", [tag_tensor], i=[sid["tag"], g.effect_seq()])

    W = T if max_T is None else max_T
    asms = [Assumption(0, "DTYPE_EQ", DISPATCH, 0, dtype=I32),
            Assumption(1, "DTYPE_EQ", DISPATCH, 2, dtype=I32)]
    if speculate == "unroll":
        asms += [Assumption(2, "TRIP_COUNT", RUNTIME, 2, value=T),
                 Assumption(3, "TYPE_TAG", RUNTIME, sid["tag"], value=TAG_TENSOR),
                 Assumption(4, "SHAPE_MATCH", DISPATCH, 0, dims=(B, T)),
                 Assumption(5, "SHAPE_MATCH", DISPATCH, 1, dims=(B, T)),
                 Assumption(6, "SHAPE_MATCH", DISPATCH, 2, dims=(B,)),
                 Assumption(7, "DTYPE_EQ", DISPATCH, 1, dtype=I32)]
    elif speculate == "while":
        asms += [Assumption(2, "RANGE", RUNTIME, 2, lo=1, hi=W, ref_arg=0, ref_dim=1),
                 Assumption(3, "TYPE_TAG", RUNTIME, sid["tag"], value=TAG_TENSOR),
                 Assumption(4, "SHAPE_MATCH", DISPATCH, 0, dims=(B, -1)),
                 Assumption(5, "SHAPE_MATCH", DISPATCH, 1, dims=(B, -1)),
                 Assumption(6, "SHAPE_MATCH", DISPATCH, 2, dims=(B,)),
                 Assumption(7, "DTYPE_EQ", DISPATCH, 1, dtype=I32)]
    elif speculate != "none":
        raise ValueError(speculate)
    args = [("tokens", I32, (B, T)), ("targets", I32, (B, T)), ("lengths", I32, (B,))]
    if training_flag:
        args.append(("training", I32, (1,)))
        if speculate != "none":
            asms += [Assumption(8, "VALUE_EQ" if flag_speculation == "value" else "BRANCH_ARM", RUNTIME, 3,
                                value=1),
                     Assumption(9, "DTYPE_EQ", DISPATCH, 3, dtype=I32)]
    if dropout:
        args.append(("dropout_key", I32, (2,)))
        if speculate != "none":
            asms += [Assumption(10, "DTYPE_EQ", DISPATCH, key_arg, dtype=I32),
                     Assumption(11, "SHAPE_MATCH", DISPATCH, key_arg, dims=(2,))]
    return Program(f"lstm_lm_L{L}_H{H}" + (f"_drop{dropout:g}" if dropout else ""), g.ops, asms, slots, args, 1, lr,
                   meta=dict(model="lstm_lm", V=V, E=E, H=H, L=L, B=B, T=T, W=W, gemm=gemm,
                             speculate=speculate, training_flag=training_flag, dropout=dropout,
                             key_arg=key_arg if dropout else -1, clip_norm=clip_norm))


# ------------------------------------------------------------------------------------------------
# TreeLSTM — recursive TreeNN of Table 2, recursion through InvokeOp (P:224, P:316 fn6).
# ------------------------------------------------------------------------------------------------
def treernn_slots(V, H, C):
    return [Slot("E", F32, (V, H), False),          # frozen word vectors (leaves; E = H)
            Slot("W", F32, (H, 2 * H), True),
            Slot("b", F32, (H,), True),
            Slot("W_c", F32, (C, H), True),
            Slot("b_c", F32, (C,), True)]


def treernn_program(V, H, C, B, lr, *, max_nodes=127, speculate="levels", gemm="bf16", clip_norm=0.0):
    """Generic graph of one TreeRNN training step (Socher et al. [37]; Table 2):

        def node(n):                                    # function 1, recursive (InvokeOp)
            if kind[n] == LEAF: return embedding(word[n])               # Switch/Merge
            else: return tanh([node(left[n]); node(right[n])] W^T + b)  # TREERNN_CELL
        for i < len(label): roots += [node(tree_off[i+1]-1)]           # loop frame
        loss = xent(linear(roots), labels); optimizer update

    Same arguments, assumptions and level lowering as treelstm_program; one output port per node.
    """
    slots = treernn_slots(V, H, C)
    sid = {s.name: k for k, s in enumerate(slots)}
    g = _G()
    # ---- function 1: node(n, kind, left, right, word, E, W, b) -> h ----
    g.func = 1
    a = [g.op("ARG", i=[k]) for k in range(8)]
    n, kind, left, right, word, Emb, W, b = a
    k0 = g.op("CONST", i=[I32], f=[0.0])
    kn = g.op("ELEMENT", [kind, n])
    is_leaf = g.op("EQ", [kn, k0])
    sw = g.op("SWITCH", [n, is_leaf])
    w = g.op("ELEMENT", [word, (sw, 1)])             # leaf arm (port 1): the word vector
    x = g.op("EMBEDDING", [Emb, w])
    ln = g.op("ELEMENT", [left, (sw, 0)])            # internal arm (port 0)
    rn = g.op("ELEMENT", [right, (sw, 0)])
    rest = [kind, left, right, word, Emb, W, b]
    hl = g.op("INVOKE", [ln] + rest, i=[1])
    hr = g.op("INVOKE", [rn] + rest, i=[1])
    cell = g.op("TREERNN_CELL", [(hl, 0), (hr, 0), W, b])
    mh = g.op("MERGE", [x, cell])
    g.op("RETURN", [mh])
    # ---- main ----
    g.func = 0
    kind, left, right, word, off, label = [g.op("ARG", i=[k]) for k in range(6)]
    rd = {s.name: _state_read(g, k, s) for k, s in enumerate(slots)}
    zero = g.op("CONST", i=[I32], f=[0.0])
    one = g.op("CONST", i=[I32], f=[1.0])
    nB = g.op("LEN", [label])
    acc0 = g.op("TA_NEW")
    FR = 1
    e_i = g.op("ENTER", [zero], i=[FR, 0])
    e_acc = g.op("ENTER", [acc0], i=[FR, 0])
    inv = {nm: g.op("ENTER", [src], i=[FR, 1]) for nm, src in
           [("nB", nB), ("one", one), ("kind", kind), ("left", left), ("right", right),
            ("word", word), ("off", off), ("E", rd["E"]), ("W", rd["W"]), ("b", rd["b"])]}
    m_i = g.op("MERGE", [e_i, e_i])
    m_acc = g.op("MERGE", [e_acc, e_acc])
    cond = g.op("LESS", [m_i, inv["nB"]])
    lc = g.op("LOOP_COND", [cond])
    s_i = g.op("SWITCH", [m_i, lc])
    s_acc = g.op("SWITCH", [m_acc, lc])
    i1 = g.op("ADD", [(s_i, 1), inv["one"]])
    end = g.op("ELEMENT", [inv["off"], i1])
    root = g.op("ADD", [end, g.op("ENTER", [g.op("CONST", i=[I32], f=[-1.0])], i=[FR, 1])])
    hroot = g.op("INVOKE", [root, inv["kind"], inv["left"], inv["right"], inv["word"], inv["E"],
                            inv["W"], inv["b"]], i=[1])
    acc1 = g.op("TA_WRITE", [(s_acc, 1), (s_i, 1), (hroot, 0)])
    g.patch_input(m_i, 1, g.op("NEXT_ITERATION", [i1]))
    g.patch_input(m_acc, 1, g.op("NEXT_ITERATION", [acc1]))
    x_acc = g.op("EXIT", [(s_acc, 0)])
    roots = g.op("TA_STACK", [x_acc])
    logits = g.op("LINEAR", [roots, rd["W_c"], rd["b_c"]])
    ones_mask = g.op("LESS", [g.op("CONST", i=[I32], f=[-1.0]), label])
    loss = g.op("SOFTMAX_XENT", [logits, label, ones_mask])
    g.op("OUTPUT", [loss], i=[0])
    for s in slots:
        if s.param:
            g.op("SGD_APPLY", [loss], i=[sid[s.name], g.effect_seq()], f=[lr])
    asms = [Assumption(a, "DTYPE_EQ", DISPATCH, a, dtype=I32) for a in range(6)]
    asms += [Assumption(6, "SHAPE_MATCH", DISPATCH, 4, dims=(B + 1,)),
             Assumption(7, "SHAPE_MATCH", DISPATCH, 5, dims=(B,))]
    if speculate == "levels":
        asms += [Assumption(8, "TREE_BINARY", RUNTIME, 0, hi=V, value=max_nodes)]
    args = [("kind", I32, None), ("left", I32, None), ("right", I32, None), ("word", I32, None),
            ("tree_off", I32, (B + 1,)), ("label", I32, (B,))]
    return Program(f"treernn_H{H}", g.ops, asms, slots, args, 1, lr,
                   meta=dict(model="treernn", V=V, E=H, H=H, C=C, B=B, gemm=gemm, clip_norm=clip_norm,
                             max_nodes=max_nodes, speculate=speculate))


def treelstm_slots(V, E, H, C):
    return [Slot("E", F32, (V, E), False),          # frozen word vectors
            Slot("W_leaf", F32, (3 * H, E), True),
            Slot("U", F32, (5 * H, 2 * H), True),
            Slot("b", F32, (4 * H,), True),
            Slot("W_c", F32, (C, H), True),
            Slot("b_c", F32, (C,), True)]


def treelstm_program(V, E, H, C, B, lr, *, max_nodes=127, speculate="levels", gemm="bf16", clip_norm=0.0):
    """Generic graph of one TreeLSTM training step:

        def node(n):                                    # function 1, recursive (InvokeOp)
            if kind[n] == LEAF: return leaf(embedding(word[n]))        # Switch/Merge
            else: return cell(node(left[n]), node(right[n]))
        for i < len(label): roots += [node(tree_off[i+1]-1)]           # loop frame
        loss = xent(linear(roots), labels); optimizer update

    Arguments: 0 kind i32[N], 1 left i32[N], 2 right i32[N], 3 word i32[N], 4 tree_off i32[B+1],
    5 label i32[B]. speculate="levels": TREE_BINARY assumption, lowered to level batches.
    """
    slots = treelstm_slots(V, E, H, C)
    sid = {s.name: k for k, s in enumerate(slots)}
    g = _G()
    # ---- function 1: node(n, kind, left, right, word, E, W_leaf, U, b) -> (h, c) ----
    g.func = 1
    a = [g.op("ARG", i=[k]) for k in range(9)]
    n, kind, left, right, word, Emb, W_leaf, U, b = a
    k0 = g.op("CONST", i=[I32], f=[0.0])
    kn = g.op("ELEMENT", [kind, n])
    is_leaf = g.op("EQ", [kn, k0])
    sw = g.op("SWITCH", [n, is_leaf])
    # leaf arm (port 1)
    w = g.op("ELEMENT", [word, (sw, 1)])
    x = g.op("EMBEDDING", [Emb, w])
    leaf = g.op("TREELSTM_LEAF", [x, W_leaf, b])
    # internal arm (port 0)
    ln = g.op("ELEMENT", [left, (sw, 0)])
    rn = g.op("ELEMENT", [right, (sw, 0)])
    rest = [kind, left, right, word, Emb, W_leaf, U, b]
    hl = g.op("INVOKE", [ln] + rest, i=[1])
    hr = g.op("INVOKE", [rn] + rest, i=[1])
    cell = g.op("TREELSTM_CELL", [(hl, 0), (hl, 1), (hr, 0), (hr, 1), U, b])
    mh = g.op("MERGE", [(leaf, 0), (cell, 0)])
    mc = g.op("MERGE", [(leaf, 1), (cell, 1)])
    g.op("RETURN", [mh, mc])
    # ---- main ----
    g.func = 0
    kind, left, right, word, off, label = [g.op("ARG", i=[k]) for k in range(6)]
    rd = {s.name: _state_read(g, k, s) for k, s in enumerate(slots)}
    zero = g.op("CONST", i=[I32], f=[0.0])
    one = g.op("CONST", i=[I32], f=[1.0])
    nB = g.op("LEN", [label])                        # for i < len(labels): the batch of trees
    acc0 = g.op("TA_NEW")
    FR = 1
    e_i = g.op("ENTER", [zero], i=[FR, 0])
    e_acc = g.op("ENTER", [acc0], i=[FR, 0])
    inv = {nm: g.op("ENTER", [src], i=[FR, 1]) for nm, src in
           [("nB", nB), ("one", one), ("kind", kind), ("left", left), ("right", right),
            ("word", word), ("off", off), ("E", rd["E"]), ("W_leaf", rd["W_leaf"]), ("U", rd["U"]),
            ("b", rd["b"])]}
    m_i = g.op("MERGE", [e_i, e_i])
    m_acc = g.op("MERGE", [e_acc, e_acc])
    cond = g.op("LESS", [m_i, inv["nB"]])
    lc = g.op("LOOP_COND", [cond])
    s_i = g.op("SWITCH", [m_i, lc])
    s_acc = g.op("SWITCH", [m_acc, lc])
    i1 = g.op("ADD", [(s_i, 1), inv["one"]])
    end = g.op("ELEMENT", [inv["off"], i1])
    root = g.op("ADD", [end, g.op("ENTER", [g.op("CONST", i=[I32], f=[-1.0])], i=[FR, 1])])
    hroot = g.op("INVOKE", [root, inv["kind"], inv["left"], inv["right"], inv["word"], inv["E"],
                            inv["W_leaf"], inv["U"], inv["b"]], i=[1])
    acc1 = g.op("TA_WRITE", [(s_acc, 1), (s_i, 1), (hroot, 0)])
    g.patch_input(m_i, 1, g.op("NEXT_ITERATION", [i1]))
    g.patch_input(m_acc, 1, g.op("NEXT_ITERATION", [acc1]))
    x_acc = g.op("EXIT", [(s_acc, 0)])
    roots = g.op("TA_STACK", [x_acc])
    logits = g.op("LINEAR", [roots, rd["W_c"], rd["b_c"]])
    ones_mask = g.op("LESS", [g.op("CONST", i=[I32], f=[-1.0]), label])  # label > -1: all rows
    loss = g.op("SOFTMAX_XENT", [logits, label, ones_mask])
    g.op("OUTPUT", [loss], i=[0])
    for s in slots:
        if s.param:
            g.op("SGD_APPLY", [loss], i=[sid[s.name], g.effect_seq()], f=[lr])
    asms = [Assumption(a, "DTYPE_EQ", DISPATCH, a, dtype=I32) for a in range(6)]
    asms += [Assumption(6, "SHAPE_MATCH", DISPATCH, 4, dims=(B + 1,)),
             Assumption(7, "SHAPE_MATCH", DISPATCH, 5, dims=(B,))]
    if speculate == "levels":
        asms += [Assumption(8, "TREE_BINARY", RUNTIME, 0, hi=V, value=max_nodes)]
    args = [("kind", I32, None), ("left", I32, None), ("right", I32, None), ("word", I32, None),
            ("tree_off", I32, (B + 1,)), ("label", I32, (B,))]
    return Program(f"treelstm_H{H}", g.ops, asms, slots, args, 1, lr,
                   meta=dict(model="treelstm", V=V, E=E, H=H, C=C, B=B, gemm=gemm, clip_norm=clip_norm,
                             max_nodes=max_nodes, speculate=speculate))


# ------------------------------------------------------------------------------------------------
# SPEC P2: Figure 1 with the cell `s = s + item`; used to pin graph semantics.
# ------------------------------------------------------------------------------------------------
def running_sum_program(n):
    """step(seq): s = self.state; outs = []; for item in seq: s = s + item; outs += [s];
    self.state = s; return sum(outs).   Arg 0: f32[n]. State slot 0: f32 scalar-like [1]."""
    slots = [Slot("state", F32, (1,))]
    g = _G()
    seq = g.op("ARG", i=[0])
    st = _state_read(g, 0, slots[0])
    zero = g.op("CONST", i=[I32], f=[0.0])
    one = g.op("CONST", i=[I32], f=[1.0])
    nn = g.op("CONST", i=[I32], f=[float(n)])
    acc0 = g.op("TA_NEW")
    FR = 1
    e_i = g.op("ENTER", [zero], i=[FR, 0])
    e_s = g.op("ENTER", [st], i=[FR, 0])
    e_acc = g.op("ENTER", [acc0], i=[FR, 0])
    inv = {nm: g.op("ENTER", [src], i=[FR, 1]) for nm, src in [("n", nn), ("one", one), ("seq", seq)]}
    m_i, m_s, m_acc = (g.op("MERGE", [e, e]) for e in (e_i, e_s, e_acc))
    lc = g.op("LOOP_COND", [g.op("LESS", [m_i, inv["n"]])])
    s_i, s_s, s_acc = (g.op("SWITCH", [m, lc]) for m in (m_i, m_s, m_acc))
    item = g.op("ELEMENT", [inv["seq"], (s_i, 1)])
    s1 = g.op("ADD", [(s_s, 1), item])
    acc1 = g.op("TA_WRITE", [(s_acc, 1), (s_i, 1), s1])
    g.patch_input(m_i, 1, g.op("NEXT_ITERATION", [g.op("ADD", [(s_i, 1), inv["one"]])]))
    g.patch_input(m_s, 1, g.op("NEXT_ITERATION", [s1]))
    g.patch_input(m_acc, 1, g.op("NEXT_ITERATION", [acc1]))
    x_s = g.op("EXIT", [(s_s, 0)])
    x_acc = g.op("EXIT", [(s_acc, 0)])
    total = g.op("SUM", [g.op("TA_STACK", [x_acc])])
    g.op("OUTPUT", [total], i=[0])
    g.op("STATE_WRITE", [x_s], i=[0, g.effect_seq()])
    asms = [Assumption(0, "SHAPE_MATCH", DISPATCH, 0, dims=(n,))]
    return Program("running_sum", g.ops, asms, slots, [("seq", F32, (n,))], 1, 0.0,
                   meta=dict(model="running_sum", n=n))
