"""Data-parallel collective paths on one GPU (1-rank NCCL communicator, JANUS_FORCE_DP=1) and
whole-step determinism. P:298 §5 (gradients averaged over workers through collectives in the
graph); reading Q12 (one failing rank aborts every rank). On one rank the allreduce is the
identity, so each DP step must equal the single-GPU step bit for bit, and the collective path
(arena allreduce, agreement, null step) must run without blocking."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import interp as I  # noqa: E402
from workloads import gen, programs as pg  # noqa: E402
from tests.helpers import to_dev, to_host  # noqa: E402


def J():
    from paper_1812_01329_b200 import janus
    return janus


def _graph(prog, monkeypatch, dp):
    return J().Graph(prog, force_dp=dp)


def _same(a, b):
    return all(x.tobytes() == y.tobytes() for x, y in zip(a, b))


def test_tree_dp_collective_path_single_gpu(monkeypatch):
    """TreeLSTM (C3 program): the DP step (arena allreduce + agreement) equals the plain step bit
    for bit; a dispatch miss (a partial last minibatch against B-tree shapes) runs the tree null
    step and reports the failing assumption without touching state."""
    V, B = 60, 6
    prog = pg.treelstm_program(V=V, E=24, H=32, C=2, B=B, lr=0.2)
    g1, g2 = _graph(prog, monkeypatch, False), _graph(prog, monkeypatch, True)
    assert g1.device_path and g2.device_path
    state = gen.uniform_params(prog, 3, 0.3)
    d1, d2 = to_dev(state), to_dev(state)
    w1, w2 = g1.new_workspace(), g2.new_workspace()
    for k in range(2):
        args = list(gen.sst_forest(gen.SEED_C3, 20 + k, B, V, max_leaves=16))
        l1, l2 = torch.zeros(1, device="cuda"), torch.zeros(1, device="cuda")
        s1, _ = g1.run(to_dev(args), d1, w1, outs=[l1])
        s2, _ = g2.run(to_dev(args), d2, w2, outs=[l2])
        assert s1 == s2 == I.OK and l1.item() == l2.item()
        assert _same(to_host(d1), to_host(d2))
    # partial last minibatch: B-1 trees -> SHAPE_MATCH (id 6, tree_off) misses at dispatch
    kind, left, right, word, off, label = gen.sst_forest(gen.SEED_C3, 30, B - 1, V, max_leaves=16)
    before = to_host(d2)
    st, fail = g2.run(to_dev([kind, left, right, word, off, label]), d2, w2)
    assert st == I.ASSUMPTION_FAILED and fail["assumption_id"] == 6 and fail["observed"] == B
    assert _same(to_host(d2), before)
    # the next full batch runs normally after the null step
    args = list(gen.sst_forest(gen.SEED_C3, 31, B, V, max_leaves=16))
    s1, _ = g1.run(to_dev(args), d1, w1)
    s2, _ = g2.run(to_dev(args), d2, w2)
    assert s1 == s2 == I.OK and _same(to_host(d1), to_host(d2))


def test_imperative_dp_collective_path_single_gpu(monkeypatch):
    """janus_run_imperative at world_size > 1 semantics on a 1-rank communicator: one arena
    allreduce (gradients of every SGD slot + the runtime-error count) and the lr / N commit equal
    the single-GPU imperative step bit for bit; a runtime error (token >= V) still joins the
    collective and commits nothing."""
    B, T, V = 4, 5, 40
    prog = pg.lstm_lm_program(V=V, E=16, H=24, L=2, B=B, T=T, lr=0.3)
    g1, g2 = _graph(prog, monkeypatch, False), _graph(prog, monkeypatch, True)
    state = gen.uniform_params(prog, 11, 0.1)
    d1, d2 = to_dev(state), to_dev(state)
    w1, w2 = g1.new_workspace(), g2.new_workspace()
    r = gen.rng(5)
    tok = r.integers(0, V, (B, T)).astype(np.int32)
    tgt = r.integers(0, V, (B, T)).astype(np.int32)
    ln = np.full(B, T, np.int32)
    l1, l2 = torch.zeros(1, device="cuda"), torch.zeros(1, device="cuda")
    s1 = g1.run_imperative(to_dev([tok, tgt, ln]), d1, w1, outs=[l1])
    s2 = g2.run_imperative(to_dev([tok, tgt, ln]), d2, w2, outs=[l2])
    assert s1 == s2 == I.OK and l1.item() == l2.item()
    assert _same(to_host(d1), to_host(d2))
    ora = I.run_imperative_step(prog, [tok, tgt, ln], state, mode="bf16")
    assert abs(l2.item() - float(ora.outputs[0])) <= 2e-2 * abs(float(ora.outputs[0]))
    bad = tok.copy(); bad[2, 3] = V
    before = to_host(d2)
    st = g2.run_imperative(to_dev([bad, tgt, ln]), d2, w2)
    assert st == I.ERR_RUNTIME and _same(to_host(d2), before)
    s1 = g1.run_imperative(to_dev([tgt, tok, ln]), d1, w1)
    s2 = g2.run_imperative(to_dev([tgt, tok, ln]), d2, w2)
    assert s1 == s2 == I.OK and _same(to_host(d1), to_host(d2))


@pytest.mark.parametrize("B", [25, 256])
def test_tree_whole_step_deterministic(B):
    """Identical inputs give identical output bits (SURVEY §8(b) determinism): two C3-shaped
    steps from the same state produce byte-identical parameters, loss and schedule."""
    V = 2000
    prog = pg.treelstm_program(V=V, E=300, H=300, C=2, B=B, lr=0.05)
    g = J().Graph(prog)
    state = gen.uniform_params(prog, 4, 0.05)
    args = list(gen.sst_forest(gen.SEED_C3, 40, B, V))
    outs = []
    for _ in range(2):
        ws = g.new_workspace()
        dev = to_dev(state)
        loss = torch.zeros(1, device="cuda")
        st, _ = g.run(to_dev(args), dev, ws, outs=[loss])
        assert st == I.OK
        outs.append((loss.item(), to_host(dev)))
    assert outs[0][0] == outs[1][0] and _same(outs[0][1], outs[1][1])


def test_lm_whole_step_deterministic():
    """C2-shaped LM step (fixed grid): two runs from the same state are bit-identical."""
    B, T, V = 64, 35, 10000
    prog = pg.lstm_lm_program(V=V, E=650, H=650, L=2, B=B, T=T, lr=1.0)
    g = J().Graph(prog)
    state = gen.uniform_params(prog, 7, 0.05)
    args = list(gen.lm_batches(gen.SEED_C2, B, T, V, 1))[0]
    outs = []
    for _ in range(2):
        ws = g.new_workspace()
        dev = to_dev(state)
        loss = torch.zeros(1, device="cuda")
        st, _ = g.run(to_dev(list(args)), dev, ws, outs=[loss])
        assert st == I.OK
        outs.append((loss.item(), to_host(dev)))
    assert outs[0][0] == outs[1][0] and _same(outs[0][1], outs[1][1])


@pytest.mark.parametrize("size,pull", [("small", False), ("small", True), ("c2", True)])
def test_fused_gradient_reduction_single_rank(size, pull, monkeypatch):
    """NEXT-3 on a 1-rank communicator: the weight gradients live in NCCL symmetric windows and
    are reduced tile by tile in the weight-gradient GEMM's epilogue (publish, owner sum in rank
    order, push, per-tile epoch flags) instead of an NCCL allreduce. With one rank the sum is the
    tile itself, so the step must equal the NCCL path bit for bit (same grouped launch: no early
    dW_dec allreduce on either side), across steps (epochs) and around a null step. pull=True
    (JANUS_FUSED_FORCE_PULL) runs the owner's pull / sum / push data path, which one rank skips."""
    if pull:
        monkeypatch.setenv("JANUS_FUSED_FORCE_PULL", "1")
    if size == "small":
        B, T, V, E, H = 8, 6, 64, 40, 48
    else:
        B, T, V, E, H = 64, 35, 10000, 650, 650
    prog = pg.lstm_lm_program(V=V, E=E, H=H, L=2, B=B, T=T, lr=0.5)
    janus = J()
    g1 = janus.Graph(prog, force_dp=True, no_dp_overlap=True)
    g2 = janus.Graph(prog, force_dp=True, no_dp_overlap=True, fused_allreduce=True)
    state = gen.uniform_params(prog, 9, 0.05)
    batches = list(gen.lm_batches(gen.SEED_C2, B, T, V, 3))
    d1, d2 = to_dev(state), to_dev(state)
    w1, w2 = g1.new_workspace(), g2.new_workspace()
    for k, args in enumerate(batches):
        l1, l2 = torch.zeros(1, device="cuda"), torch.zeros(1, device="cuda")
        s1, _ = g1.run(to_dev(list(args)), d1, w1, outs=[l1])
        s2, _ = g2.run(to_dev(list(args)), d2, w2, outs=[l2])
        assert s1 == s2 == I.OK and l1.item() == l2.item()
        assert _same(to_host(d1), to_host(d2)), f"step {k}"
        if k == 0:  # a null step (dispatch miss: B-1 rows) on both, then the next step as usual
            tok, tgt, ln = args
            a = [tok[:B - 1], tgt[:B - 1], ln[:B - 1]]
            s1, f1 = g1.run(to_dev(a), d1, w1)
            s2, f2 = g2.run(to_dev(a), d2, w2)
            assert s1 == s2 == I.ASSUMPTION_FAILED and f1 == f2
    if size == "small":
        ora = I.run_graph_step(prog, list(batches[0]), state, mode="bf16")
        assert ora.status == I.OK
