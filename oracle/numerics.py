"""ORACLE — TEST INFRASTRUCTURE ONLY. Op numerics (forward + vector-Jacobian products) of the
whitelisted framework functions the graph may contain (§4.3.1: "matmul", ...).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may import
this package. It shares no code with the CUDA path.

Arithmetic: float64 throughout. Precision mode "f32" computes in fp64 with no rounding (the paper's
fp32 models; C1 is compared at 1e-5). Mode "bf16" additionally rounds, round-to-nearest-even,
at the three points of DESIGN.md reading R (SURVEY §8(c) rounding points):
  R1  GEMM operand copies of weight matrices (W_ih, W_hh, W_dec, W_leaf, U, E) = rb(master)
  R2  every h / x that feeds a GEMM = rb(h)
  R3  dz and dy are rounded before the dgrad / wgrad GEMMs; bias gradients are sums of the
      rounded rows (the bias gradient is the wgrad of a ones column)
The cell equations follow the cited models because the paper gives none (P:312 cites [51] LSTM and
[40] TreeLSTM): readings Q1 and Q5 of DESIGN.md, written out in the docstrings below.
"""
from __future__ import annotations

import numpy as np


class RuntimeFault(Exception):
    """A runtime error inside a pure node (bad index) — reported distinctly from an assumption
    failure and commits nothing."""


def rb(x):
    """Round float64 values to the nearest bfloat16 (ties to even), returned as float64.
    Goes through fp32 first, as a GPU rounds its fp32 registers."""
    a = np.asarray(x, dtype=np.float64).astype(np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) & 0xFFFF0000
    out = u.astype(np.uint32).view(np.float32).astype(np.float64)
    nan = np.isnan(a)
    if nan.any():
        out = np.where(nan, np.nan, out)
    return out


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


class Prec:
    """Precision mode: `g(x)` applies the GEMM operand rounding (R1/R2/R3) in bf16 mode."""

    def __init__(self, mode):
        assert mode in ("f32", "bf16")
        self.mode = mode
        self._memo = {}  # id(array) -> (array, rb(array)): rb is a pure function of the values

    def g(self, x):
        if self.mode != "bf16":
            return np.asarray(x, np.float64)
        if isinstance(x, np.ndarray) and x.size >= 4096 and not x.flags.writeable:
            # large read-only arrays (the step's parameters, frozen by the executor) are rounded
            # once per step instead of once per use: the same values (R1: one bf16 working copy)
            hit = self._memo.get(id(x))
            if hit is not None and hit[0] is x:
                return hit[1]
            r = rb(x)
            self._memo[id(x)] = (x, r)
            return r
        return rb(x)


# ------------------------------------------------------------------------ embedding (KP3)
def embedding_fwd(P, E, ids):
    """X[r] = E[id_r]; ids outside [0, V) are a runtime error."""
    ids = np.asarray(ids, np.int64).reshape(-1)
    V = E.shape[0]
    bad = (ids < 0) | (ids >= V)
    if bad.any():
        raise RuntimeFault(f"embedding id out of range at {int(np.argmax(bad))}")
    return P.g(E[ids])  # rb is elementwise: rounding the gathered rows == gathering rounded rows


def embedding_vjp(E_shape, ids, dX):
    """dE[w] = sum over rows r with id_r = w of dX[r], in ascending r (segmented sum)."""
    ids = np.asarray(ids, np.int64).reshape(-1)
    dE = np.zeros(E_shape)
    for r, w in enumerate(ids):
        dE[w] += dX[r]
    return dE


# ------------------------------------------------------------------------ linear (KP1)
def linear_fwd(P, x, W, b):
    """y = x W^T + b with bf16-rounded operands in bf16 mode (R1, R2)."""
    return P.g(x) @ P.g(W).T + b


def linear_vjp(P, x, W, dy):
    """dx = rb(dy) W, dW = rb(dy)^T x, db = sum_rows rb(dy)   (R3)."""
    d = P.g(dy)
    return d @ P.g(W), d.T @ P.g(x), d.sum(axis=0)


# ------------------------------------------------------------------------ LSTM cell (Fig 1 rnn_cell)
def lstm_fwd(P, x, h, c, W_ih, W_hh, b, valid):
    """Zaremba/torch.nn.LSTM cell (reading Q1; gate blocks i, f, g, o; one folded bias):
        z = x W_ih^T + h W_hh^T + b;  i, f, o = sigmoid;  g = tanh
        c' = f * c + i * g;  h' = o * tanh(c')
    Rows with valid == 0 carry (h, c) unchanged (masked step, reading Q18 / C4)."""
    H = h.shape[1]
    z = P.g(x) @ P.g(W_ih).T + P.g(h) @ P.g(W_hh).T + b
    i = sigmoid(z[:, 0:H]); f = sigmoid(z[:, H:2 * H])
    g = np.tanh(z[:, 2 * H:3 * H]); o = sigmoid(z[:, 3 * H:4 * H])
    c2 = f * c + i * g
    h2 = o * np.tanh(c2)
    v = (np.asarray(valid).reshape(-1, 1) != 0)
    h2 = np.where(v, h2, h)
    c2 = np.where(v, c2, c)
    return h2, c2, (i, f, g, o, c, c2, v)


def lstm_vjp(P, saved, x, h, W_ih, W_hh, dh2, dc2):
    """Backward of lstm_fwd (SURVEY §8(c) "LSTM bwd"):
        tc = tanh(c');  do = dh tc;  dc = dc' + dh o (1 - tc^2)
        di = dc g;  dg = dc i;  df = dc c;  dc_prev = dc f
        dz = [di i(1-i), df f(1-f), dg (1-g^2), do o(1-o)]
        dx = rb(dz) W_ih;  dh_prev = rb(dz) W_hh;  dW_ih = rb(dz)^T x;  dW_hh = rb(dz)^T h;
        db = sum_rows rb(dz).   Masked rows pass dh, dc through and contribute no dz."""
    i, f, g, o, c, c2, v = saved
    tc = np.tanh(c2)
    do = dh2 * tc
    dc = dc2 + dh2 * o * (1.0 - tc * tc)
    di, dg, df = dc * g, dc * i, dc * c
    dz = np.concatenate([di * i * (1 - i), df * f * (1 - f), dg * (1 - g * g), do * o * (1 - o)], axis=1)
    dz = np.where(v, dz, 0.0)
    d = P.g(dz)
    dx = d @ P.g(W_ih)
    dh_prev = np.where(v, d @ P.g(W_hh), dh2)
    dc_prev = np.where(v, dc * f, dc2)
    return dx, dh_prev, dc_prev, d.T @ P.g(x), d.T @ P.g(h), d.sum(axis=0)


# ------------------------------------------------------------------------ TreeLSTM (Tai et al. [40])
def tree_leaf_fwd(P, x, W_leaf, b):
    """Leaf (reading Q5): z = x W_leaf^T + [b_i; b_o; b_u]; i, o = sigmoid, u = tanh;
    c = i u; h = o tanh(c).  b has blocks (i, f, o, u)."""
    H = W_leaf.shape[0] // 3
    bb = np.concatenate([b[0:H], b[2 * H:3 * H], b[3 * H:4 * H]])
    z = P.g(x) @ P.g(W_leaf).T + bb
    i = sigmoid(z[:, 0:H]); o = sigmoid(z[:, H:2 * H]); u = np.tanh(z[:, 2 * H:3 * H])
    c = i * u
    h = o * np.tanh(c)
    return h, c, (i, o, u, c)


def tree_leaf_vjp(P, saved, x, W_leaf, dh, dc_in):
    """tc = tanh c; do = dh tc; dc = dc_in + dh o (1 - tc^2); di = dc u; du = dc i;
    dz = [di i(1-i), do o(1-o), du (1-u^2)]; dW_leaf = rb(dz)^T x; db_{i,o,u} = sum rb(dz);
    dx = rb(dz) W_leaf."""
    i, o, u, c = saved
    H = i.shape[1]
    tc = np.tanh(c)
    do = dh * tc
    dc = dc_in + dh * o * (1 - tc * tc)
    dz = np.concatenate([dc * u * i * (1 - i), do * o * (1 - o), dc * i * (1 - u * u)], axis=1)
    d = P.g(dz)
    s = d.sum(axis=0)
    db = np.concatenate([s[0:H], np.zeros(H), s[H:2 * H], s[2 * H:3 * H]])
    return d @ P.g(W_leaf), d.T @ P.g(x), db


def tree_cell_fwd(P, hl, cl, hr, cr, U, b):
    """Binary N-ary TreeLSTM cell (reading Q5): z = [h_l; h_r] U^T + [b_i; b_f; b_f; b_o; b_u];
    i, f_l, f_r, o = sigmoid, u = tanh; c = i u + f_l c_l + f_r c_r; h = o tanh(c)."""
    H = hl.shape[1]
    bb = np.concatenate([b[0:H], b[H:2 * H], b[H:2 * H], b[2 * H:3 * H], b[3 * H:4 * H]])
    hh = np.concatenate([hl, hr], axis=1)
    z = P.g(hh) @ P.g(U).T + bb
    i = sigmoid(z[:, 0:H]); fl = sigmoid(z[:, H:2 * H]); fr = sigmoid(z[:, 2 * H:3 * H])
    o = sigmoid(z[:, 3 * H:4 * H]); u = np.tanh(z[:, 4 * H:5 * H])
    c = i * u + fl * cl + fr * cr
    h = o * np.tanh(c)
    return h, c, (i, fl, fr, o, u, cl, cr, c, hh)


def tree_cell_vjp(P, saved, U, dh, dc_in):
    """tc = tanh c; do = dh tc; dc = dc_in + dh o (1-tc^2); di = dc u; du = dc i;
    df_l = dc c_l; df_r = dc c_r; dz = [di i(1-i), df_l f_l(1-f_l), df_r f_r(1-f_r), do o(1-o),
    du (1-u^2)]; [dh_l; dh_r] = rb(dz) U; dc_l = dc f_l; dc_r = dc f_r; dU = rb(dz)^T [h_l; h_r];
    db_i, db_o, db_u = sums of rb(dz) blocks; db_f = sum of the rb(dz_fl) + rb(dz_fr) blocks."""
    i, fl, fr, o, u, cl, cr, c, hh = saved
    H = i.shape[1]
    tc = np.tanh(c)
    do = dh * tc
    dc = dc_in + dh * o * (1 - tc * tc)
    dz = np.concatenate([dc * u * i * (1 - i), dc * cl * fl * (1 - fl), dc * cr * fr * (1 - fr),
                         do * o * (1 - o), dc * i * (1 - u * u)], axis=1)
    d = P.g(dz)
    dhh = d @ P.g(U)
    s = d.sum(axis=0)
    db = np.concatenate([s[0:H], s[H:2 * H] + s[2 * H:3 * H], s[3 * H:4 * H], s[4 * H:5 * H]])
    return dhh[:, :H], dc * fl, dhh[:, H:], dc * fr, d.T @ P.g(hh), db


def tree_rnn_fwd(P, hl, hr, W, b):
    """TreeRNN cell (Socher et al. [37]; Table 2 TreeRNN on SST; reading R13): the parent of
    two children is h = tanh([h_l; h_r] W^T + b), W [H, 2H], b [H]. Leaves are the word vectors."""
    hh = np.concatenate([hl, hr], axis=1)
    h = np.tanh(P.g(hh) @ P.g(W).T + b)
    return h, (h, hh)


def tree_rnn_vjp(P, saved, W, dh):
    """dz = dh (1 - h^2); [dh_l; dh_r] = rb(dz) W; dW = rb(dz)^T rb([h_l; h_r]); db = sum rb(dz)
    (R3 / R4 as for every affine op)."""
    h, hh = saved
    H = h.shape[1]
    d = P.g(dh * (1.0 - h * h))
    dhh = d @ P.g(W)
    return dhh[:, :H], dhh[:, H:], d.T @ P.g(hh), d.sum(axis=0)


# ------------------------------------------------------------------------ dropout (NEXT-4)
_PHILOX_M0, _PHILOX_M1 = 0xD2511F53, 0xCD9E8D57
_PHILOX_W0, _PHILOX_W1 = 0x9E3779B9, 0xBB67AE85


def philox4x32_10(ctr, key):
    """Philox4x32-10 (Salmon et al., SC'11), the counter-based generator the dropout masks are
    drawn from: ctr uint32 [..., 4], key uint32 [..., 2] -> uint32 [..., 4]. Ten rounds; round i
    uses the key bumped i times by (W0, W1); a round is
    (hi0, lo0) = M0 * c0, (hi1, lo1) = M1 * c2, c <- (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)."""
    c = np.asarray(ctr, np.uint64) & 0xFFFFFFFF
    k = np.asarray(key, np.uint64) & 0xFFFFFFFF
    c0, c1, c2, c3 = (c[..., i] for i in range(4))
    k0, k1 = k[..., 0], k[..., 1]
    for r in range(10):
        if r:
            k0 = (k0 + _PHILOX_W0) & 0xFFFFFFFF
            k1 = (k1 + _PHILOX_W1) & 0xFFFFFFFF
        p0 = c0 * _PHILOX_M0
        p1 = c2 * _PHILOX_M1
        hi0, lo0 = p0 >> 32, p0 & 0xFFFFFFFF
        hi1, lo1 = p1 >> 32, p1 & 0xFFFFFFFF
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return np.stack([c0, c1, c2, c3], axis=-1).astype(np.uint32)


def dropout_mask(key, site, rows, cols, p):
    """Keep mask of dropout site `site` (reading R14): element (r, j) draws word j mod 4 of
    Philox4x32-10(counter = (j div 4, r, site, 0), key) and is kept iff word >= floor(p * 2^32).
    rows: global row indices (time-major t * B + b)."""
    rows = np.asarray(rows, np.uint64).reshape(-1)
    j = np.arange(cols, dtype=np.uint64)
    ctr = np.zeros((len(rows), cols, 4), np.uint64)
    ctr[..., 0] = j[None, :] >> 2
    ctr[..., 1] = rows[:, None]
    ctr[..., 2] = site
    k = np.broadcast_to(np.asarray(key, np.uint64).reshape(2), ctr.shape[:-1] + (2,))
    words = philox4x32_10(ctr, k)
    w = np.take_along_axis(words, (j & 3).astype(np.int64)[None, :, None].repeat(len(rows), 0), axis=-1)[..., 0]
    thr = np.uint64(min(int(p * 4294967296.0), 4294967295))
    return (w.astype(np.uint64) >= thr).astype(np.float64)


def dropout_fwd(x, key, site, rows, p):
    """Inverted dropout of the non-recurrent connections (Zaremba et al. [51]): y = x m / (1 - p)."""
    m = dropout_mask(key, site, rows, x.shape[1], p) / (1.0 - p)
    return x * m, m


def dropout_vjp(saved, dy):
    return dy * saved


# ------------------------------------------------------------------------ loss (KP4)
def xent_fwd(logits, tgt, mask):
    """loss = sum_r mask_r (logsumexp(y_r) - y_r[tgt_r]) / max(1, sum_r mask_r)  (reading Q3).
    Targets of masked rows outside [0, C) are a runtime error."""
    tgt = np.asarray(tgt, np.int64).reshape(-1)
    m = np.asarray(mask).reshape(-1) != 0
    C = logits.shape[1]
    bad = m & ((tgt < 0) | (tgt >= C))
    if bad.any():
        raise RuntimeFault(f"target out of range at {int(np.argmax(bad))}")
    n = max(1, int(m.sum()))
    mx = logits.max(axis=1, keepdims=True)
    lse = (mx + np.log(np.exp(logits - mx).sum(axis=1, keepdims=True)))[:, 0]
    t = np.clip(tgt, 0, C - 1)
    lr = lse - logits[np.arange(len(t)), t]
    loss = float(np.where(m, lr, 0.0).sum() / n)
    return loss, (lse, t, m, n)


def xent_vjp(logits, saved, dloss):
    """dy = mask (softmax(y) - onehot(tgt)) / n_valid * dloss."""
    lse, t, m, n = saved
    p = np.exp(logits - lse[:, None])
    p[np.arange(len(t)), t] -= 1.0
    return np.where(m[:, None], p, 0.0) * (dloss / n)
