"""Seeded synthetic inputs; shared by the oracle tests, the GPU tests and bench.py.

Holds no arithmetic of the method: only numpy PCG64 draws shaped like the paper's workloads
(PTB-shaped token streams for the LSTM of Table 2, SST-shaped binary parse trees for the
TreeLSTM of Table 2). Both backends consume the same arrays; neither regenerates them.
"""
from __future__ import annotations

import numpy as np

SEED_C1, SEED_C2, SEED_C3, SEED_C4, SEED_C5 = 1812, 1813, 1814, 1815, 1816


def rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


# ----------------------------------------------------------------------------- parameters
def uniform_params(program, seed, scale):
    """fp32 U(-scale, scale) for every parameter slot, zeros for carried state, tag = TENSOR."""
    r = rng(seed)
    out = []
    for s in program.slots:
        if s.name == "tag":
            out.append(np.ones(s.shape, np.int32))
        elif s.param or s.name == "E":
            out.append(r.uniform(-scale, scale, size=s.shape).astype(np.float32))
        else:
            out.append(np.zeros(s.shape, np.float32))
    return out


# ----------------------------------------------------------------------------- LSTM LM
def zipf_stream(seed, n, V):
    """i.i.d. tokens with p(k) ∝ 1/(k+1) over V words (PTB-like long tail)."""
    p = 1.0 / np.arange(1, V + 1, dtype=np.float64)
    p /= p.sum()
    return rng(seed).choice(V, size=n, p=p).astype(np.int32)


def lm_batches(seed, B, T, V, n_steps, ranks=1):
    """Zaremba batching: one stream reshaped to [ranks*B, n_steps*T+1]; rank r owns rows
    [rB, (r+1)B). Yields (tokens, targets, lengths) per step for the global batch."""
    stream = zipf_stream(seed, ranks * B * (n_steps * T + 1), V).reshape(ranks * B, n_steps * T + 1)
    for s in range(n_steps):
        tok = np.ascontiguousarray(stream[:, s * T:(s + 1) * T])
        tgt = np.ascontiguousarray(stream[:, s * T + 1:(s + 1) * T + 1])
        yield tok, tgt, np.full(ranks * B, T, np.int32)


def c1_batches(n_steps=10, B=4, T=8, V=32):
    """C1 toy: seed 1812; step 3 carries lengths [8,8,7,8] (the hand-worked RUNTIME failure)."""
    out = []
    for s, (tok, tgt, ln) in enumerate(lm_batches(SEED_C1, B, T, V, n_steps)):
        if s == 3:
            ln = ln.copy()
            ln[2] = T - 1
        out.append((tok, tgt, ln))
    return out


def c4_batch(seed, step, B, V, W_max=64, W_min=5):
    """Variable-length batch: W ~ U{W_min..W_max}; lengths ~ U{1..W} with row (step mod B) = W."""
    r = rng(seed * 1000003 + step)
    W = int(r.integers(W_min, W_max + 1))
    lens = r.integers(1, W + 1, size=B).astype(np.int32)
    lens[step % B] = W
    p = 1.0 / np.arange(1, V + 1, dtype=np.float64)
    p /= p.sum()
    tok = r.choice(V, size=(B, W), p=p).astype(np.int32)
    tgt = r.choice(V, size=(B, W), p=p).astype(np.int32)
    return tok, tgt, lens


# ----------------------------------------------------------------------------- trees
def _split(r, n):
    """Random binary shape over n leaves: left leaf count k ~ U{1..n-1}. Returns nested tuples,
    a leaf is None."""
    if n == 1:
        return None
    k = int(r.integers(1, n))
    return (_split(r, k), _split(r, n - k))


def _chain(n):
    """Right-branching chain over n leaves: (leaf, (leaf, (... leaf)))."""
    t = None
    for _ in range(n - 1):
        t = (None, t)
    return t


def forest_from_shapes(shapes, words):
    """Post-order encoding of a list of shapes (None = leaf). Returns kind, left, right, word,
    tree_off (int32). Children ids are global; a leaf's left/right are -1; internal word = -1."""
    kind, left, right, word, off = [], [], [], [], [0]
    wi = iter(words)

    def emit(s):
        if s is None:
            kind.append(0); left.append(-1); right.append(-1); word.append(int(next(wi)))
            return len(kind) - 1
        a = emit(s[0]); b = emit(s[1])
        kind.append(1); left.append(a); right.append(b); word.append(-1)
        return len(kind) - 1

    for s in shapes:
        emit(s)
        off.append(len(kind))
    f = lambda x: np.asarray(x, np.int32)
    return f(kind), f(left), f(right), f(word), f(off)


def n_leaves(s):
    return 1 if s is None else n_leaves(s[0]) + n_leaves(s[1])


def sst_forest(seed, step, B, V, max_leaves=64, chain=False):
    """SST-shaped synthetic batch: leaves n = clamp(round(LogNormal(ln 17, 0.55)), 1, 64),
    random splits (or right-branching chains), words U{0..V-1}, labels Bernoulli(0.5)."""
    r = rng(seed * 1000003 + step)
    ns = np.clip(np.rint(r.lognormal(np.log(17.0), 0.55, size=B)), 1, max_leaves).astype(int)
    shapes = [_chain(int(n)) if chain else _split(r, int(n)) for n in ns]
    words = r.integers(0, V, size=int(ns.sum()))
    kind, left, right, word, off = forest_from_shapes(shapes, words)
    label = r.integers(0, 2, size=B).astype(np.int32)
    return kind, left, right, word, off, label


def all_shapes(n):
    """Every binary tree shape with n leaves (Catalan(n-1) of them)."""
    if n == 1:
        return [None]
    out = []
    for k in range(1, n):
        for a in all_shapes(k):
            for b in all_shapes(n - k):
                out.append((a, b))
    return out
