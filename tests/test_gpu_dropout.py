"""Dropout LM (NEXT-4: the Zaremba et al. [51] model of P:312, dropout on every non-recurrent
connection, Philox4x32-10 masks keyed per step) through the C ABI on the GPU vs the oracle: the
device regenerates the masks the oracle draws (same counter layout, reading R14), forward and
backward, on the graph path and on the imperative executor."""
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


def _steps(prog, batches, seed=5, scale=0.1, tol=2e-2, imperative=False):
    janus = J()
    g = janus.Graph(prog)
    assert g.device_path, g.build_message
    assert "dropout=0.5" in g.describe()
    ws = g.new_workspace()
    state = gen.uniform_params(prog, seed, scale)
    for k, args in enumerate(batches):
        dev = to_dev(state)
        loss = torch.zeros(1, device="cuda")
        if imperative:
            st = g.run_imperative(to_dev(list(args)), dev, ws, outs=[loss])
            ora = I.run_imperative_step(prog, list(args), state, mode="bf16")
        else:
            st, fail = g.run(to_dev(list(args)), dev, ws, outs=[loss])
            ora = I.run_graph_step(prog, list(args), state, mode="bf16")
        assert st == ora.status == I.OK
        assert rel_err(loss.item(), ora.outputs[0]) <= tol, (loss.item(), ora.outputs[0])
        assert_state_parity(prog, state, to_host(dev), ora.state, tol, what=f"dropout step {k}")
        state = ora.state


def _batches(B, T, V, n, ragged=False):
    out = []
    for k, (tok, tgt, ln) in enumerate(gen.lm_batches(gen.SEED_C2, B, T, V, n)):
        if ragged:
            ln = gen.rng(40 + k).integers(1, T + 1, B).astype(np.int32)
            ln[0] = T
        out.append((tok, tgt, ln, np.array([1000 + k, 77 * k + 3], np.int32)))
    return out


def test_dropout_lm_small_unrolled():
    B, T, V = 8, 6, 64
    prog = pg.lstm_lm_program(V=V, E=40, H=48, L=2, B=B, T=T, lr=0.5, dropout=0.5)
    _steps(prog, _batches(B, T, V, 3))


def test_dropout_lm_ragged_while_three_layers():
    B, T, V = 13, 9, 120
    prog = pg.lstm_lm_program(V=V, E=72, H=100, L=3, B=B, T=T, lr=0.5, dropout=0.5, speculate="while")
    _steps(prog, _batches(B, T, V, 2, ragged=True), scale=0.2)


def test_dropout_lm_c2_full_size():
    """The Zaremba medium model at the C2 shape: 2 x 650, V = 10000, T = 35, B = 64, p = 0.5."""
    B, T, V = 64, 35, 10000
    prog = pg.lstm_lm_program(V=V, E=650, H=650, L=2, B=B, T=T, lr=1.0, dropout=0.5)
    _steps(prog, _batches(B, T, V, 1), scale=0.05)


def test_dropout_lm_imperative_executor():
    B, T, V = 4, 5, 40
    prog = pg.lstm_lm_program(V=V, E=16, H=24, L=2, B=B, T=T, lr=0.3, dropout=0.5)
    _steps(prog, _batches(B, T, V, 2), imperative=True)


def test_dropout_key_changes_the_step():
    B, T, V = 8, 6, 64
    prog = pg.lstm_lm_program(V=V, E=40, H=48, L=2, B=B, T=T, lr=0.5, dropout=0.5)
    janus = J()
    g = janus.Graph(prog)
    ws = g.new_workspace()
    state = gen.uniform_params(prog, 5, 0.1)
    tok, tgt, ln, _ = _batches(B, T, V, 1)[0]
    losses = []
    for key in ([1, 2], [1, 2], [3, 2]):
        loss = torch.zeros(1, device="cuda")
        st, _ = g.run(to_dev([tok, tgt, ln, np.array(key, np.int32)]), to_dev(state), ws, outs=[loss])
        assert st == I.OK
        losses.append(loss.item())
    assert losses[0] == losses[1] and losses[0] != losses[2]
