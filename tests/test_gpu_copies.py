"""The bf16 operand copies refreshed by the commit (R1, "copy refresh"): a step skips the
re-cast of W_ih / W_hh / W_hh^T / W_ih1^T / W_dec when the last commit of the same graph wrote them
and nothing else wrote state since. The trajectory must equal re-casting every step (JANUS_RECAST=1,
read once per process: that arm runs in a subprocess) bit for bit, through every event that must
invalidate the copies: an in-place write by the caller (torch version counter -> janus_state_changed),
another graph committing into the same state, the imperative executor, fresh state tensors, and an
AssertOp abort (nothing committed: the copies stay valid). The TreeLSTM / TreeRNN steps likewise."""
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from workloads import gen, programs as pg  # noqa: E402
from tests.helpers import to_dev, to_host  # noqa: E402


def _trajectory(L, dropout):
    from paper_1812_01329_b200 import janus
    B, T, V = 8, 6, 64
    kw = dict(V=V, E=40, H=48, L=L, B=B, T=T, lr=0.5, dropout=dropout)
    A = janus.Graph(pg.lstm_lm_program(**kw))
    W = janus.Graph(pg.lstm_lm_program(speculate="while", **kw))
    assert A.device_path and W.device_path, (A.build_message, W.build_message)
    wa, ww = A.new_workspace(), W.new_workspace()
    sid = {s.name: k for k, s in enumerate(A.program.slots)}
    dev = to_dev(gen.uniform_params(A.program, 5, 0.1))
    batches = list(gen.lm_batches(gen.SEED_C2, B, T, V, 12))
    key = [np.array([7, k], np.int32) for k in range(12)]
    loss = torch.zeros(1, device="cuda")
    trace = []

    def step(g, ws, k, lens=None, imperative=False):
        tk, tg, ln = batches[k]
        args = [tk, tg, ln if lens is None else lens] + ([key[k]] if dropout else [])
        if imperative:
            st = g.run_imperative(to_dev(args), dev, ws, outs=[loss])
        else:
            st, _ = g.run(to_dev(args), dev, ws, outs=[loss])
        trace.append((st, loss.item()))

    step(A, wa, 0)
    step(A, wa, 1)                                  # copies from the commit of step 0
    step(A, wa, 2)
    with torch.no_grad():
        dev[sid["W_hh0"]].mul_(0.9)                 # caller writes a master in place
        dev[sid["W_dec"]][3].add_(0.25)
    step(A, wa, 3)
    step(W, ww, 4, lens=gen.rng(44).integers(1, T + 1, B).astype(np.int32))  # another graph commits
    step(A, wa, 5)
    bad = np.full(B, T, np.int32)
    bad[2] = T - 1
    step(A, wa, 6, lens=bad)                        # TRIP_COUNT miss: nothing runs, nothing commits
    step(A, wa, 7)
    step(A, wa, 8, imperative=True)                 # the imperative executor commits
    step(A, wa, 9)
    dev = [t.clone() for t in dev]                  # fresh state tensors
    step(A, wa, 10)
    step(A, wa, 11)
    return trace, [t.tobytes() for t in to_host(dev)]


def _tree_trajectory(rnn):
    """The tree programs keep W_leaf / U (TreeRNN: W) copies the same way: row copies and the
    transposed U the backward streams."""
    from paper_1812_01329_b200 import janus
    V, B, H = 500, 6, 24
    prog = (pg.treernn_program(V=V, H=H, C=2, B=B, lr=0.3) if rnn else
            pg.treelstm_program(V=V, E=20, H=H, C=2, B=B, lr=0.3))
    A, A2 = janus.Graph(prog), janus.Graph(prog)
    wa, wb = A.new_workspace(), A2.new_workspace()
    sid = {s.name: k for k, s in enumerate(prog.slots)}
    dev = to_dev(gen.uniform_params(prog, 3, 0.2))
    loss = torch.zeros(1, device="cuda")
    trace = []

    def step(g, ws, k, imperative=False):
        f = to_dev(gen.sst_forest(gen.SEED_C3, k, B, V))
        if imperative:
            st = g.run_imperative(f, dev, ws, outs=[loss])
        else:
            st, _ = g.run(f, dev, ws, outs=[loss])
        trace.append((st, loss.item()))

    for k in range(3):
        step(A, wa, k)
    with torch.no_grad():
        dev[sid["W" if rnn else "U"]].mul_(0.9)
    step(A, wa, 3)
    step(A2, wb, 4)
    step(A, wa, 5)
    step(A, wa, 6, imperative=True)
    step(A, wa, 7)
    step(A, wa, 8)
    return trace, [t.tobytes() for t in to_host(dev)]


CASES = [(2, 0.0), (2, 0.3), (1, 0.0), (3, 0.0)]
TREE_CASES = [False, True]


def _dump(path):
    np.save(path, np.array([_trajectory(L, p) for L, p in CASES] + [_tree_trajectory(r) for r in TREE_CASES],
                           dtype=object), allow_pickle=True)


def test_copy_refresh_equals_recast_every_step():
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "recast.npy")
        env = dict(os.environ, JANUS_RECAST="1")
        r = subprocess.run([sys.executable, "-c", f"import tests.test_gpu_copies as t; t._dump({path!r})"],
                           env=env, capture_output=True, text=True, timeout=600,
                           cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
        ref = np.load(path, allow_pickle=True)
    for (L, p), (rtrace, rstate) in zip(CASES, ref[:len(CASES)]):
        trace, state = _trajectory(L, p)
        assert [s for s, _ in trace] == [s for s, _ in rtrace], (L, p, trace)
        assert trace == rtrace, (L, p, trace, rtrace)
        assert all(a == b for a, b in zip(state, rstate)), (L, p)
        assert trace[6][0] != 0 and all(s == 0 for k, (s, _) in enumerate(trace) if k != 6), trace
    for rnn, (rtrace, rstate) in zip(TREE_CASES, ref[len(CASES):]):
        trace, state = _tree_trajectory(rnn)
        assert all(s == 0 for s, _ in trace), trace
        assert trace == rtrace, (rnn, trace, rtrace)
        assert all(a == b for a, b in zip(state, rstate)), rnn
