"""Round-2 GPU parity cases (VERDICT r1 "What's weak" 2): the device RANGE and VALUE_EQ AssertOps
bit-exact against the oracle, the `training` Switch (speculated and device-evaluated), C4 at the
full C2 model size, C3 at B=256 with H=E=300, and 5-step bf16 drift runs of C2 and C3."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import interp as I  # noqa: E402
from workloads import gen, programs as pg  # noqa: E402
from tests.helpers import assert_state_parity, rel_err, to_dev, to_host  # noqa: E402
from tests.test_gpu_lm import _run_parity, _step  # noqa: E402
from tests.test_gpu_tree import _check  # noqa: E402


def J():
    from paper_1812_01329_b200 import janus
    return janus


def _fail_tuple(fail):
    return fail["assumption_id"], fail["index"], fail["observed"]


def _ora_tuple(r):
    return r.failure.assumption_id, r.failure.index, r.failure.observed


# ----------------------------------------------------------------------------- RANGE (C4 guard)
def test_range_guard_failures_bit_exact():
    """RANGE(id 2, 1 <= len <= min(W, width)) on the device: the hand-worked cases of
    test_oracle_pins_r2 (length 0, length > W, length > this batch's width) give the oracle's
    {id, index, observed}; the state is byte-identical afterwards; a passing batch commits."""
    B, W, V = 8, 12, 64
    prog = pg.lstm_lm_program(V=V, E=24, H=32, L=2, B=B, T=W, lr=0.5, speculate="while")
    janus = J()
    g = janus.Graph(prog)
    assert g.device_path and "while_width" in g.describe(), g.build_message
    ws = g.new_workspace()
    state = gen.uniform_params(prog, 4, 0.2)
    r = gen.rng(11)
    tok = r.integers(0, V, (B, W)).astype(np.int32)
    cases = [(tok, [5, 3, 0, 7, 0, 2, 1, 1]),          # zeros at 2 and 4: index 2 reported
             (tok, [12, 12, 13, 12, 1, 1, 1, 1]),      # 13 > W
             (tok[:, :6].copy(), [6, 6, 6, 7, 6, 1, 2, 3]),  # 7 > width 6
             (tok[:, :6].copy(), [6, 6, 6, 6, 6, 1, 2, 3])]  # passes
    for t_, lens in cases:
        args = [t_, t_.copy(), np.array(lens, np.int32)]
        ora = I.run_graph_step(prog, args, state, mode="bf16")
        dev = to_dev(state)
        st, fail, loss = _step(g, ws, args, dev)
        assert st == ora.status
        if st == I.ASSUMPTION_FAILED:
            assert _fail_tuple(fail) == _ora_tuple(ora)
            assert all(a.tobytes() == b.tobytes() for a, b in zip(to_host(dev), state))
        else:
            assert rel_err(loss, ora.outputs[0]) <= 2e-2
            assert_state_parity(prog, state, to_host(dev), ora.state, 2e-2, what="range pass")


# ----------------------------------------------------------------------------- training Switch
def test_training_switch_speculated_value_eq():
    """The C2 program with `if training: update`: VALUE_EQ(training == 1) (id 8) specialised away
    on the device; training = 0 / 3 fails bit-exactly with nothing committed, then the imperative
    fallback gives the oracle's evaluate step (parameters unchanged, carried state advanced)."""
    B, T, V = 8, 6, 64
    prog = pg.lstm_lm_program(V=V, E=40, H=48, L=2, B=B, T=T, lr=0.5, training_flag=True)
    janus = J()
    g = janus.Graph(prog)
    assert g.device_path and "train=specialised" in g.describe(), g.build_message
    tok, tgt, ln = list(gen.lm_batches(gen.SEED_C2, B, T, V, 1))[0]
    _run_parity(prog, "bf16", 2e-2, [(tok, tgt, ln, np.array([1], np.int32))])
    ws = g.new_workspace()
    state = gen.uniform_params(prog, 5, 0.1)
    for flag in (0, 3):
        args = [tok, tgt, ln, np.array([flag], np.int32)]
        ora = I.run_graph_step(prog, args, state, mode="bf16")
        dev = to_dev(state)
        st, fail, _ = _step(g, ws, args, dev)
        assert st == ora.status == I.ASSUMPTION_FAILED
        assert _fail_tuple(fail) == _ora_tuple(ora) == (8, 0, flag)
        assert all(a.tobytes() == b.tobytes() for a, b in zip(to_host(dev), state))
    args = [tok, tgt, ln, np.array([0], np.int32)]
    dev = to_dev(state)
    loss = torch.zeros(1, device="cuda")
    assert g.run_imperative(to_dev(args), dev, ws, outs=[loss]) == I.OK
    imp = I.run_imperative_step(prog, args, state, mode="bf16")
    got = to_host(dev)
    for k, s in enumerate(prog.slots):
        if s.param:
            assert got[k].tobytes() == state[k].tobytes(), s.name
    assert_state_parity(prog, state, got, imp.state, 2e-2, what="eval fallback")


def test_training_switch_speculated_branch_arm():
    """The same Switch speculated by BRANCH_ARM (the control-flow assumption): every
    non-zero flag takes the true arm (training = 1 and 5 both commit the update, parity with the
    oracle); training = 0 fails bit-exactly as {8, 0, 0} with nothing committed."""
    B, T, V = 8, 6, 64
    prog = pg.lstm_lm_program(V=V, E=40, H=48, L=2, B=B, T=T, lr=0.5, training_flag=True,
                              flag_speculation="branch")
    janus = J()
    g = janus.Graph(prog)
    assert g.device_path and "train=specialised" in g.describe(), g.build_message
    tok, tgt, ln = list(gen.lm_batches(gen.SEED_C2, B, T, V, 1))[0]
    _run_parity(prog, "bf16", 2e-2, [(tok, tgt, ln, np.array([1], np.int32)),
                                     (tok, tgt, ln, np.array([5], np.int32))])
    ws = g.new_workspace()
    state = gen.uniform_params(prog, 5, 0.1)
    args = [tok, tgt, ln, np.array([0], np.int32)]
    ora = I.run_graph_step(prog, args, state, mode="bf16")
    dev = to_dev(state)
    st, fail, _ = _step(g, ws, args, dev)
    assert st == ora.status == I.ASSUMPTION_FAILED
    assert _fail_tuple(fail) == _ora_tuple(ora) == (8, 0, 0)
    assert all(a.tobytes() == b.tobytes() for a, b in zip(to_host(dev), state))


def test_training_switch_on_the_device():
    """Without the VALUE_EQ assumption (what janus_relax leaves after it breaks) the Switch is
    evaluated on the device: the commit kernel reads training[0]; both arms match the oracle."""
    B, T, V = 8, 6, 64
    prog = pg.lstm_lm_program(V=V, E=40, H=48, L=2, B=B, T=T, lr=0.5, training_flag=True)
    prog.assumptions = [a for a in prog.assumptions if a.kind != "VALUE_EQ"]
    janus = J()
    g = janus.Graph(prog)
    assert g.device_path and "train=device_switch" in g.describe(), g.build_message
    tok, tgt, ln = list(gen.lm_batches(gen.SEED_C2, B, T, V, 1))[0]
    _run_parity(prog, "bf16", 2e-2, [(tok, tgt, ln, np.array([f], np.int32)) for f in (0, 1, 0, 2)])
    ws = g.new_workspace()
    state = gen.uniform_params(prog, 6, 0.1)
    dev = to_dev(state)
    st, _, _ = _step(g, ws, [tok, tgt, ln, np.array([0], np.int32)], dev)
    got = to_host(dev)
    assert st == I.OK
    for k, s in enumerate(prog.slots):
        if s.param:
            assert got[k].tobytes() == state[k].tobytes(), s.name
    # host-resident flag (the e2e path stages it through the workspace)
    dev = to_dev(state)
    host = [torch.tensor(a).pin_memory() for a in (tok, tgt, ln, np.array([1], np.int32))]
    st, _ = g.run(host, dev, ws, outs=[torch.zeros(1, device="cuda")])
    ora = I.run_graph_step(prog, [tok, tgt, ln, np.array([1], np.int32)], state, mode="bf16")
    assert st == I.OK
    assert_state_parity(prog, state, to_host(dev), ora.state, 2e-2, what="host flag")


# ----------------------------------------------------------------------------- C4 at C2 size
def test_c4_full_size_device_while():
    """C4: the C2 model (2x650, V=10000, B=64) with per-batch width W ~ U{5..64} and
    ragged lengths, lowered to the device While (RANGE guard); every output against the oracle."""
    B, V = 64, 10000
    prog = pg.lstm_lm_program(V=V, E=650, H=650, L=2, B=B, T=64, lr=1.0, speculate="while")
    batches = [gen.c4_batch(gen.SEED_C4, k, B, V) for k in range(2)]
    assert len({b[0].shape[1] for b in batches}) == 2
    _run_parity(prog, "bf16", 2e-2, batches, scale=0.05)


# ----------------------------------------------------------------------------- C3 at B=256
def test_tree_c3_b256_full_size():
    """C3 B=256, H=E=300, V=20000 (the bench's second TreeLSTM line): schedule bit-exact,
    numerics within the bf16 tolerance."""
    V, B = 20000, 256
    prog = pg.treelstm_program(V=V, E=300, H=300, C=2, B=B, lr=0.05)
    _check(prog, [gen.sst_forest(gen.SEED_C3, 0, B, V)], scale=0.05)


# ----------------------------------------------------------------------------- 5-step drift
def _drift(prog, batches, seed, scale, tol=2e-2):
    """Both sides keep their own trajectory for len(batches) steps (no re-sync): the loss of every
    step and the final carried state must stay within the bf16 tolerance."""
    janus = J()
    g = janus.Graph(prog)
    ws = g.new_workspace()
    state = gen.uniform_params(prog, seed, scale)
    ora_state = state
    dev = to_dev(state)
    losses = []
    for args in batches:
        loss = torch.zeros(1, device="cuda")
        st, fail = g.run(to_dev(list(args)), dev, ws, outs=[loss])
        ora = I.run_graph_step(prog, list(args), ora_state, mode="bf16")
        assert st == ora.status == I.OK, fail
        losses.append((loss.item(), float(ora.outputs[0])))
        assert rel_err(*losses[-1]) <= tol, losses
        ora_state = ora.state
    got = to_host(dev)
    for k, s in enumerate(prog.slots):
        if not s.param and s.name != "tag":
            assert rel_err(got[k], ora_state[k]) <= tol, s.name
        if s.param:   # accumulated update of 5 steps
            d_g = got[k].astype(np.float64) - state[k]
            d_o = np.asarray(ora_state[k], np.float64) - state[k]
            if s.name != "E":
                assert rel_err(d_g, d_o) <= 5 * tol, s.name
    return losses


def test_c2_five_step_drift():
    B, T, V = 64, 35, 10000
    prog = pg.lstm_lm_program(V=V, E=650, H=650, L=2, B=B, T=T, lr=1.0)
    _drift(prog, list(gen.lm_batches(gen.SEED_C2, B, T, V, 5)), seed=1, scale=0.05)


def test_c3_five_step_drift():
    V, B = 20000, 25
    prog = pg.treelstm_program(V=V, E=300, H=300, C=2, B=B, lr=0.05)
    _drift(prog, [gen.sst_forest(gen.SEED_C3, k, B, V) for k in range(5)], seed=1, scale=0.05)


# ----------------------------------------------------------------------------- session
def test_session_width_miss_join_keeps_both_device_paths():
    """An unrolled LM graph (B, T) missing twice on narrower batches (B, T'): the Figure 4 join
    (B, ?) relaxes the trip count with it (a bounded device While), so the joined graph serves T'
    on the device, and the original (B, T) key still hits its own unrolled graph afterwards."""
    B, T, V = 8, 6, 64
    prog = pg.lstm_lm_program(V=V, E=40, H=48, L=2, B=B, T=T, lr=0.5)
    janus = J()
    sess = janus.Session(prog)
    state = gen.uniform_params(prog, 5, 0.1)
    dev = to_dev(state)
    full = list(gen.lm_batches(gen.SEED_C2, B, T, V, 3))
    narrow = [(a[:, :4].copy(), b[:, :4].copy(), np.full(B, 4, np.int32)) for a, b, _ in full]
    seq = [narrow[0], narrow[1], narrow[2], full[0], narrow[0]]
    events = []
    for args in seq:
        ora = I.run_imperative_step(prog, list(args), state, mode="bf16")
        st, info = sess.step(to_dev(list(args)), dev, outs=[torch.zeros(1, device="cuda")])
        assert st == I.OK
        events.append((info["event"], info["path"]))
        assert_state_parity(prog, state, to_host(dev), ora.state, 2e-2, what=str(events[-1]))
        state = ora.state
        dev = to_dev(state)
    assert events == [("MISS", "imperative"), ("MISS", "imperative"), ("HIT", "graph"),
                      ("HIT", "graph"), ("HIT", "graph")], events
    ents = sess.stats()["entries"]
    assert [e["active"] for e in ents] == [True, True] and ents[1]["origin"] == "miss-join"
    assert any("RANGE" in a for a in ents[1]["assumptions"]) and ents[1]["device"]


def test_step_graph_replay_equals_direct_launches(monkeypatch):
    """With JANUS_STEP_GRAPH=1, from the third call on the same workspace and state tensors
    janus_run replays the step as one captured CUDA graph; the trajectory must equal direct
    launches bit for bit, including the ragged While program and a batch that fails its AssertOp
    mid-sequence. (The switch is read once per process: this test runs in its own process.)"""
    import subprocess
    import sys
    if os.environ.get("JANUS_STEP_GRAPH") != "1":
        env = dict(os.environ, JANUS_STEP_GRAPH="1")
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                            __file__ + "::test_step_graph_replay_equals_direct_launches"],
                           env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
        return
    for speculate in ("unroll", "while"):
        B, T, V = 8, 6, 64
        prog = pg.lstm_lm_program(V=V, E=40, H=48, L=2, B=B, T=T, lr=0.5, speculate=speculate)
        batches = list(gen.lm_batches(gen.SEED_C2, B, T, V, 6))
        if speculate == "while":
            batches = [(tk, tg, gen.rng(60 + k).integers(1, T + 1, B).astype(np.int32)) for k, (tk, tg, _) in
                       enumerate(batches)]
        else:  # step 4 violates TRIP_COUNT: aborts, state untouched, then the graph replays again
            tk, tg, ln = batches[4]
            ln = ln.copy(); ln[2] = T - 1
            batches[4] = (tk, tg, ln)
        state = gen.uniform_params(prog, 5, 0.1)
        runs = []
        for no_graph in (False, True):
            if no_graph:
                monkeypatch.setenv("JANUS_NO_GRAPH", "1")
            g = J().Graph(prog)
            ws = g.new_workspace()
            dev = to_dev(state)
            loss = torch.zeros(1, device="cuda")
            trace = []
            for args in batches:
                st, _ = g.run(to_dev(list(args)), dev, ws, outs=[loss])
                trace.append((st, loss.item()))
            runs.append((trace, to_host(dev), g.counters()))
            monkeypatch.delenv("JANUS_NO_GRAPH", raising=False)
        assert runs[0][0] == runs[1][0]
        assert all(a.tobytes() == b.tobytes() for a, b in zip(runs[0][1], runs[1][1]))
        assert runs[0][2]["launches"] == runs[1][2]["launches"]   # a replay counts its kernels
