"""LSTM language model through the C ABI on the GPU vs the oracle."""
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


def _step(g, ws, args_np, state_dev):
    loss = torch.zeros(1, device="cuda")
    st, fail = g.run(to_dev(args_np), state_dev, ws, outs=[loss])
    return st, fail, float(loss.item())


def _run_parity(prog, mode, tol, batches, seed=5, scale=0.1, gemm=None):
    janus = J()
    g = janus.Graph(prog, gemm=gemm)
    assert g.device_path, g.build_message
    ws = g.new_workspace()
    state = gen.uniform_params(prog, seed, scale)
    dev = to_dev(state)
    for k, args in enumerate(batches):
        ora = I.run_graph_step(prog, list(args), state, mode=mode)
        st, fail, loss = _step(g, ws, args, dev)
        got = to_host(dev)
        assert st == ora.status, (k, st, ora.status, fail, ora.failure)
        if st == I.OK:
            assert rel_err(loss, ora.outputs[0]) <= tol, (k, loss, float(ora.outputs[0]))
            assert_state_parity(prog, state, got, ora.state, tol, what=f"step {k}")
            state = ora.state
            dev = to_dev(state)   # re-sync to the oracle trajectory (no drift accumulation)
        else:
            assert all(a.tobytes() == b.tobytes() for a, b in zip(got, state))
    return g


# ------------------------------------------------------------------ C1: fp32, single launch
def test_c1_toy_fp32_ten_steps_with_forced_failure():
    prog = pg.lstm_lm_program(V=32, E=16, H=16, L=1, B=4, T=8, lr=0.1, gemm="f32")
    janus = J()
    g = janus.Graph(prog)
    assert g.device_path and "fp32_single_cta" in g.describe()
    ws = g.new_workspace()
    state = gen.uniform_params(prog, gen.SEED_C1, 0.1)
    dev = to_dev(state)
    for k, args in enumerate(gen.c1_batches()):
        c0 = g.counters()
        before = to_host(dev)
        ora = I.run_graph_step(prog, list(args), state, mode="f32")
        st, fail, loss = _step(g, ws, args, dev)
        c1 = g.counters()
        got = to_host(dev)
        assert st == ora.status
        assert c1["host_syncs"] - c0["host_syncs"] == 1          # one host sync per step
        assert c1["launches"] - c0["launches"] == 1              # the whole step is one launch
        if k == 3:   # hand-worked failure: TRIP_COUNT id 2, element 2, observed 7
            assert fail == dict(assumption_id=2, rank=0, index=2, observed=7)
            assert all(a.tobytes() == b.tobytes() for a, b in zip(got, before))
            state = I.run_imperative_step(prog, list(args), state, mode="f32").state  # fallback
            dev = to_dev(state)
            continue
        assert st == I.OK
        assert rel_err(loss, ora.outputs[0]) <= 1e-5
        assert_state_parity(prog, state, got, ora.state, 1e-5, what=f"C1 step {k}")
        # drift check: keep the GPU trajectory (no re-sync) and compare to the oracle's
        state = ora.state
        for a, b in zip(got, state):
            assert rel_err(a, b) <= 1e-5


# ------------------------------------------------------------------ bf16 tcgen05 path
def _lm_batches(B, T, V, n, seed=gen.SEED_C2):
    return list(gen.lm_batches(seed, B, T, V, n))


def test_lm_bf16_small_two_layers():
    prog = pg.lstm_lm_program(V=64, E=40, H=48, L=2, B=8, T=6, lr=0.5)
    _run_parity(prog, "bf16", 2e-2, _lm_batches(8, 6, 64, 2))


def test_lm_bf16_ragged_tiles():
    """H=100: last recurrent CTA owns 4 of 16 units; B=33 rows; E, V off the tile grid."""
    prog = pg.lstm_lm_program(V=300, E=72, H=100, L=2, B=33, T=9, lr=0.5)
    _run_parity(prog, "bf16", 2e-2, _lm_batches(33, 9, 300, 2), scale=0.2)


def test_lm_bf16_batch128_one_layer():
    prog = pg.lstm_lm_program(V=200, E=64, H=64, L=1, B=128, T=4, lr=0.5)
    _run_parity(prog, "bf16", 2e-2, _lm_batches(128, 4, 200, 1), scale=0.2)


def test_lm_bf16_three_layers_per_layer_kernels():
    """L=3 does not take the two-layer wavefront: one forward launch per layer (M=64 MMAs)."""
    prog = pg.lstm_lm_program(V=120, E=40, H=48, L=3, B=16, T=7, lr=0.5)
    _run_parity(prog, "bf16", 2e-2, _lm_batches(16, 7, 120, 2), scale=0.2)


@pytest.mark.parametrize("env", [{"JANUS_REC_WF": "0"}, {"JANUS_REC_BWD": "plain"},
                                 {"JANUS_REC_WF": "0", "JANUS_REC_BWD": "plain"}])
def test_lm_bf16_kernel_variants(monkeypatch, env):
    """The per-layer forward and the plain (non-K-split) backward give the same parity."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    prog = pg.lstm_lm_program(V=300, E=72, H=100, L=2, B=33, T=9, lr=0.5)
    _run_parity(prog, "bf16", 2e-2, _lm_batches(33, 9, 300, 1), scale=0.2)


def test_lm_bf16_c2_full_size():
    """BASELINE config C2 at full size: 2x650, T35, B64, V10000 — one step, every output."""
    prog = pg.lstm_lm_program(V=10000, E=650, H=650, L=2, B=64, T=35, lr=1.0)
    _run_parity(prog, "bf16", 2e-2, _lm_batches(64, 35, 10000, 1), scale=0.05)


def test_lm_while_mode_variable_lengths():
    """C4: data-dependent trip count max(lengths) on the device; masked rows carry state."""
    B, W, V = 16, 12, 90
    prog = pg.lstm_lm_program(V=V, E=24, H=32, L=2, B=B, T=W, lr=0.5, speculate="while")
    r = gen.rng(3)
    batches = []
    for k in range(3):
        w = int(r.integers(5, W + 1))
        lens = r.integers(1, w + 1, B).astype(np.int32)
        lens[k] = w
        batches.append((r.integers(0, V, (B, w)).astype(np.int32), r.integers(0, V, (B, w)).astype(np.int32), lens))
    _run_parity(prog, "bf16", 2e-2, batches, scale=0.2)


def test_lm_guards_and_all_or_nothing():
    B, T, V = 8, 6, 64
    prog = pg.lstm_lm_program(V=V, E=40, H=48, L=2, B=B, T=T, lr=0.5)
    janus = J()
    g = janus.Graph(prog)
    ws = g.new_workspace()
    state = gen.uniform_params(prog, 9, 0.1)
    tok, tgt, ln = _lm_batches(B, T, V, 1)[0]
    # RUNTIME TRIP_COUNT (id 2): one row shorter
    bad = ln.copy(); bad[5] = T - 2
    dev = to_dev(state)
    st, fail, _ = _step(g, ws, (tok, tgt, bad), dev)
    ora = I.run_graph_step(prog, [tok, tgt, bad], state)
    assert st == I.ASSUMPTION_FAILED and fail == dict(assumption_id=2, rank=0, index=5, observed=T - 2)
    assert (ora.failure.assumption_id, ora.failure.index, ora.failure.observed) == (2, 5, T - 2)
    assert all(a.tobytes() == b.tobytes() for a, b in zip(to_host(dev), state))
    # RUNTIME TYPE_TAG (id 3): self.state is None
    st2 = [x.copy() for x in state]
    st2[prog.slot_index("tag")][:] = 0
    dev = to_dev(st2)
    st, fail, _ = _step(g, ws, (tok, tgt, ln), dev)
    assert st == I.ASSUMPTION_FAILED and fail["assumption_id"] == 3 and fail["observed"] == 0
    assert all(a.tobytes() == b.tobytes() for a, b in zip(to_host(dev), st2))
    # DISPATCH shape (id 4): nothing launched
    c0 = g.counters()
    st, fail, _ = _step(g, ws, (tok[:B - 1], tgt[:B - 1], ln[:B - 1]), to_dev(state))
    assert st == I.ASSUMPTION_FAILED and fail == dict(assumption_id=4, rank=0, index=0, observed=B - 1)
    assert g.counters()["launches"] == c0["launches"]
    # forced failure of every assumption id (fault injection)
    for a in prog.assumptions:
        gf = janus.Graph(prog, fail_assert_id=a.id)
        dev = to_dev(state)
        st, fail, _ = _step(gf, gf.new_workspace(), (tok, tgt, ln), dev)
        assert st == I.ASSUMPTION_FAILED and fail["assumption_id"] == a.id
        assert all(x.tobytes() == y.tobytes() for x, y in zip(to_host(dev), state))
    # runtime error: token id >= V commits nothing
    tk = tok.copy(); tk[1, 2] = V
    dev = to_dev(state)
    st, _, _ = _step(g, ws, (tk, tgt, ln), dev)
    assert st == I.ERR_RUNTIME
    assert all(a.tobytes() == b.tobytes() for a, b in zip(to_host(dev), state))


def test_lm_dp_collective_path_single_gpu(monkeypatch):
    """The data-parallel step (NCCL allreduce of the gradient arena, dense embedding gradient,
    abort agreement) on a 1-rank communicator equals the single-GPU step bit for bit; a dispatch
    failure runs the null step and still reports the failure."""
    B, T, V = 8, 6, 64
    prog = pg.lstm_lm_program(V=V, E=40, H=48, L=2, B=B, T=T, lr=0.5)
    janus = J()
    g1 = janus.Graph(prog)
    g2 = janus.Graph(prog, force_dp=True)
    state = gen.uniform_params(prog, 9, 0.1)
    args = _lm_batches(B, T, V, 1)[0]
    d1, d2 = to_dev(state), to_dev(state)
    s1, _, l1 = _step(g1, g1.new_workspace(), args, d1)
    ws2 = g2.new_workspace()
    s2, _, l2 = _step(g2, ws2, args, d2)
    assert s1 == s2 == I.OK and l1 == l2
    for a, b in zip(to_host(d1), to_host(d2)):
        assert a.tobytes() == b.tobytes()
    bad = ln = args[2].copy(); bad[3] = T - 1
    st, fail, _ = _step(g2, ws2, (args[0], args[1], bad), d2)
    assert st == I.ASSUMPTION_FAILED and fail == dict(assumption_id=2, rank=0, index=3, observed=T - 1)
    st, fail, _ = _step(g2, ws2, (args[0][:B - 1], args[1][:B - 1], ln[:B - 1]), d2)   # null step
    assert st == I.ASSUMPTION_FAILED and fail["assumption_id"] == 4 and fail["observed"] == B - 1
    assert all(a.tobytes() == b.tobytes() for a, b in zip(to_host(d1), to_host(d2)))


def test_lm_host_buffers_e2e_equal_device_args():
    """janus_run with host (pinned) argument buffers stages them through the workspace."""
    B, T, V = 8, 6, 64
    prog = pg.lstm_lm_program(V=V, E=40, H=48, L=2, B=B, T=T, lr=0.5)
    janus = J()
    g = janus.Graph(prog)
    ws = g.new_workspace()
    state = gen.uniform_params(prog, 9, 0.1)
    args = _lm_batches(B, T, V, 1)[0]
    d1 = to_dev(state)
    st1, _, l1 = _step(g, ws, args, d1)
    d2 = to_dev(state)
    host = [torch.tensor(a).pin_memory() for a in args]
    loss = torch.zeros(1).pin_memory()
    st2, _ = g.run(host, d2, ws, outs=[loss])
    assert st1 == st2 == I.OK and l1 == float(loss.item())
    assert all(a.tobytes() == b.tobytes() for a, b in zip(to_host(d1), to_host(d2)))
