"""janus_run_imperative (the per-op GPU fallback, P:160 / Table 3 "Imp.") vs the oracle's
imperative execution of the same generic programs."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import interp as I  # noqa: E402
from workloads import gen, programs as pg  # noqa: E402
from tests.helpers import assert_state_parity, rel_err, to_dev, to_host  # noqa: E402


def J():
    from paper_1812_01329_b200 import janus
    return janus


def _imp(g, ws, args, dev):
    loss = torch.zeros(1, device="cuda")
    st = g.run_imperative(to_dev(args), dev, ws, outs=[loss])
    return st, float(loss.item())


def test_spec_p2_running_sum_imperative():
    """S:112-113 through the GPU imperative executor: 10.0 / 6.0, then 24.0 / 9.0."""
    janus = J()
    dev = to_dev([np.array([0.0], np.float32)])
    for seq, ret, after in (([1.0, 2.0, 3.0], 10.0, 6.0), ([1.0, 1.0, 1.0], 24.0, 9.0)):
        prog = pg.running_sum_program(3)
        g = janus.Graph(prog)
        assert not g.device_path       # no device lowering: only the imperative path runs it
        st, loss = _imp(g, g.new_workspace(), [np.array(seq, np.float32)], dev)
        assert st == I.OK and loss == ret and float(dev[0].item()) == after


def test_c1_imperative_fp32_and_control_syncs():
    prog = pg.lstm_lm_program(V=32, E=16, H=16, L=1, B=4, T=8, lr=0.1, gemm="f32")
    janus = J()
    g = janus.Graph(prog)
    ws = g.new_workspace()
    state = gen.uniform_params(prog, gen.SEED_C1, 0.1)
    for k, args in enumerate(gen.c1_batches()[:4]):
        dev = to_dev(state)
        c0 = g.counters()
        st, loss = _imp(g, ws, args, dev)
        c1 = g.counters()
        ora = I.run_imperative_step(prog, list(args), state, mode="f32")
        assert st == I.OK == ora.status        # never ASSUMPTION_FAILED (also at step 3)
        assert rel_err(loss, ora.outputs[0]) <= 1e-5
        assert_state_parity(prog, state, to_host(dev), ora.state, 1e-5, what=f"imp step {k}")
        T = int(args[2].max())
        launches, syncs = c1["launches"] - c0["launches"], c1["host_syncs"] - c0["host_syncs"]
        assert launches > 10 * T                # one launch per op instance
        assert syncs >= T + 1                   # every LoopCond is read back by the host
        state = ora.state


def test_lm_imperative_bf16_and_while_lengths():
    B, W, V = 8, 7, 64
    prog = pg.lstm_lm_program(V=V, E=40, H=48, L=2, B=B, T=W, lr=0.5, speculate="none")
    janus = J()
    g = janus.Graph(prog)
    ws = g.new_workspace()
    state = gen.uniform_params(prog, 9, 0.1)
    r = gen.rng(5)
    lens = r.integers(1, W + 1, B).astype(np.int32)
    args = (r.integers(0, V, (B, W)).astype(np.int32), r.integers(0, V, (B, W)).astype(np.int32), lens)
    dev = to_dev(state)
    st, loss = _imp(g, ws, args, dev)
    ora = I.run_imperative_step(prog, list(args), state, mode="bf16")
    assert st == I.OK
    assert rel_err(loss, ora.outputs[0]) <= 2e-2
    assert_state_parity(prog, state, to_host(dev), ora.state, 2e-2, what="imp bf16")


def test_tree_imperative_recursion():
    V, B = 30, 3
    prog = pg.treelstm_program(V=V, E=16, H=24, C=2, B=B, lr=0.2, speculate="none")
    janus = J()
    g = janus.Graph(prog)
    ws = g.new_workspace()
    state = gen.uniform_params(prog, 4, 0.3)
    f = list(gen.sst_forest(gen.SEED_C3, 2, B, V, max_leaves=6))
    dev = to_dev(state)
    c0 = g.counters()
    st, loss = _imp(g, ws, f, dev)
    c1 = g.counters()
    ora = I.run_imperative_step(prog, f, state, mode="bf16")
    assert st == I.OK
    assert rel_err(loss, ora.outputs[0]) <= 2e-2
    assert_state_parity(prog, state, to_host(dev), ora.state, 2e-2, what="imp tree")
    assert c1["host_syncs"] - c0["host_syncs"] >= len(f[0])   # a branch decision per node


def test_fallback_after_assumption_failure_and_runtime_error():
    """the graph path aborts with nothing mutated, the imperative path then produces the
    imperative result, committed exactly once. A bad token id is ERR_RUNTIME on both paths."""
    B, T, V = 8, 6, 64
    prog = pg.lstm_lm_program(V=V, E=40, H=48, L=2, B=B, T=T, lr=0.5)
    janus = J()
    g = janus.Graph(prog)
    ws = g.new_workspace()
    state = gen.uniform_params(prog, 9, 0.1)
    tok, tgt, ln = list(gen.lm_batches(gen.SEED_C2, B, T, V, 1))[0]
    ln = ln.copy(); ln[2] = T - 1
    dev = to_dev(state)
    st, fail = g.run(to_dev([tok, tgt, ln]), dev, ws)
    assert st == I.ASSUMPTION_FAILED and fail["assumption_id"] == 2
    assert all(a.tobytes() == b.tobytes() for a, b in zip(to_host(dev), state))
    st, loss = _imp(g, ws, [tok, tgt, ln], dev)
    ora = I.run_imperative_step(prog, [tok, tgt, ln], state, mode="bf16")
    assert st == I.OK and rel_err(loss, ora.outputs[0]) <= 2e-2
    assert_state_parity(prog, state, to_host(dev), ora.state, 2e-2, what="fallback")
    bad = tok.copy(); bad[0, 0] = V + 3
    before = to_host(dev)
    st, _ = _imp(g, ws, [bad, tgt, ln], dev)
    assert st == I.ERR_RUNTIME
    assert all(a.tobytes() == b.tobytes() for a, b in zip(to_host(dev), before))
