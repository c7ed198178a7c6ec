"""Graph cache + relaxation driver on the GPU: every session step commits
the imperative program's result (end-to-end equivalence), whichever path ran; assumptions
that repeatedly break are relaxed and the regenerated graph then serves the step on the device
(SPEC orchestrator S:478-524)."""
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


def _check(prog, sess, args, state, dev, tol=2e-2, what=""):
    """One session step vs the oracle's imperative execution of the generic program."""
    loss = torch.zeros(1, device="cuda")
    st, info = sess.step(to_dev(args), dev, outs=[loss])
    ora = I.run_imperative_step(prog, list(args), state, mode="bf16")
    assert st == ora.status, (what, st, ora.status, info)
    if st == I.OK:
        assert rel_err(float(loss.item()), ora.outputs[0]) <= tol, what
        assert_state_parity(prog, state, to_host(dev), ora.state, tol, what=what)
        return info, ora.state
    return info, state


def test_session_trip_count_relaxed_to_device_while():
    """TRIP_COUNT (id 2) breaks twice -> regenerated as a bounded device While (RANGE [1, T]);
    batches with short rows then run on the graph path instead of aborting."""
    B, T, V = 8, 6, 64
    prog = pg.lstm_lm_program(V=V, E=40, H=48, L=2, B=B, T=T, lr=0.5)
    sess = J().Session(prog)
    state = gen.uniform_params(prog, 9, 0.1)
    batches = list(gen.lm_batches(gen.SEED_C2, B, T, V, 6))
    short = [(b[0], b[1], b[2].copy()) for b in batches]
    for k, b in enumerate(short):
        b[2][k % B] = 1 + k % (T - 1)
    plan = [(batches[0], "HIT", "graph"), (short[1], "ABORT", "imperative"), (short[2], "ABORT", "imperative"),
            (batches[3], "HIT", "graph"), (short[4], "HIT", "graph"), (short[5], "HIT", "graph")]
    for k, (args, ev, path) in enumerate(plan):
        dev = to_dev(state)
        info, state = _check(prog, sess, args, state, dev, what=f"step {k}")
        assert (info["event"], info["path"]) == (ev, path), (k, info)
        if ev == "ABORT":
            assert info["fail"]["assumption_id"] == 2
        assert info["generated"] == (1 if k == 2 else -1)
    st = sess.stats()
    assert st["aborts"] == {"2": 2} and st["graph_calls"] == 4 and st["imperative_calls"] == 2
    e0, e1 = st["entries"]
    assert not e0["active"] and e1["active"] and e1["device"] and e1["origin"] == "relax:2"
    assert "2:RANGE(arg2,[1,6])" in e1["assumptions"]


def test_session_type_tag_relaxed_to_device_switch():
    """`self.state is None` (TYPE_TAG id 3) breaks twice -> the tag Switch runs on the device."""
    B, T, V = 8, 6, 64
    prog = pg.lstm_lm_program(V=V, E=40, H=48, L=2, B=B, T=T, lr=0.5)
    sess = J().Session(prog)
    state = gen.uniform_params(prog, 11, 0.1)
    tag = prog.slot_index("tag")
    batches = list(gen.lm_batches(gen.SEED_C2, B, T, V, 5))
    events = []
    for k, args in enumerate(batches):
        if k in (1, 2, 4):
            state = [x.copy() for x in state]
            state[tag][:] = pg.TAG_NONE
        dev = to_dev(state)
        info, state = _check(prog, sess, args, state, dev, what=f"step {k}")
        events.append((info["event"], info["path"]))
        assert int(state[tag][0]) == pg.TAG_TENSOR
    assert events == [("HIT", "graph"), ("ABORT", "imperative"), ("ABORT", "imperative"),
                      ("HIT", "graph"), ("HIT", "graph")]
    assert "3:TYPE_TAG" not in " ".join(sess.stats()["entries"][1]["assumptions"])


def test_session_dtype_miss_generates_int64_graph_and_keeps_int32_graph():
    """int64 tokens miss the int32 graph twice; the graph generated for the int64 key (the cache
    keys on argument types) runs on the device beside the int32 one."""
    B, T, V = 8, 6, 64
    prog = pg.lstm_lm_program(V=V, E=40, H=48, L=2, B=B, T=T, lr=0.5)
    sess = J().Session(prog)
    state = gen.uniform_params(prog, 13, 0.1)
    batches = list(gen.lm_batches(gen.SEED_C2, B, T, V, 5))
    seen = []
    for k, (tok, tgt, ln) in enumerate(batches):
        args = (tok.astype(np.int64), tgt, ln) if k != 3 else (tok, tgt, ln)
        dev = to_dev(state)
        info, state = _check(prog, sess, args, state, dev, what=f"step {k}")
        seen.append((info["event"], info["path"], info["generated"]))
    assert seen == [("MISS", "imperative", -1), ("MISS", "imperative", 1), ("HIT", "graph", -1),
                    ("HIT", "graph", -1), ("HIT", "graph", -1)]
    st = sess.stats()
    assert st["misses"] == 2 and st["entries"][0]["active"] and st["entries"][0]["hits"] == 1
    assert st["entries"][1]["device"] and st["entries"][1]["hits"] == 2
    assert "0:DTYPE_EQ(arg0,dt3)" in st["entries"][1]["assumptions"]


def test_session_shape_errors_are_not_specialised():
    """A batch of B-1 rows against B-row carried state is a program error (ERR_RUNTIME in the
    imperative executor, R10): it is returned every time and never generates a graph."""
    B, T, V = 8, 6, 64
    prog = pg.lstm_lm_program(V=V, E=40, H=48, L=2, B=B, T=T, lr=0.5)
    sess = J().Session(prog)
    state = gen.uniform_params(prog, 13, 0.1)
    tok, tgt, ln = list(gen.lm_batches(gen.SEED_C2, B, T, V, 1))[0]
    before = to_dev(state)
    for _ in range(3):
        st, info = sess.step(to_dev((tok[:B - 1], tgt[:B - 1], ln[:B - 1])), before)
        assert st == J().ERR_RUNTIME and info["event"] == "MISS" and info["generated"] == -1
    assert all(a.tobytes() == b.tobytes() for a, b in zip(to_host(before), state))
    assert len(sess.stats()["entries"]) == 1


def test_session_tree_partial_minibatch_gets_its_own_graph():
    """The partial last minibatch misses the B-tree graph twice; the joined '?' batch has
    no device lowering, so a graph specialised to the new batch size is generated beside the old
    one and serves the third such call on the device."""
    Bt, V = 5, 50
    prog = pg.treelstm_program(V=V, E=24, H=32, C=2, B=Bt, lr=0.1)
    sess = J().Session(prog)
    state = gen.uniform_params(prog, 3, 0.1)
    seen = []
    for k, b in enumerate([Bt, Bt - 1, Bt - 1, Bt - 1, Bt]):
        args = gen.sst_forest(gen.SEED_C3, k, b, V, max_leaves=12)
        dev = to_dev(state)
        info, state = _check(prog, sess, args, state, dev, what=f"step {k}")
        seen.append((info["event"], info["path"], info["generated"]))
    assert seen == [("HIT", "graph", -1), ("MISS", "imperative", -1), ("MISS", "imperative", 2),
                    ("HIT", "graph", -1), ("HIT", "graph", -1)]
    ents = sess.stats()["entries"]
    assert [e["active"] for e in ents] == [True, False, True] and ents[2]["origin"] == "miss-key"
    assert "6:SHAPE_MATCH(arg4,(5))" in ents[2]["assumptions"]


def test_int64_specialised_graphs_match_the_oracle():
    """Type-specialised graphs for int64 index arguments (LM tokens/targets/lengths, every tree
    array) run on the device and commit the imperative program's result."""
    janus = J()
    B, T, V = 8, 6, 64
    prog = pg.lstm_lm_program(V=V, E=40, H=48, L=2, B=B, T=T, lr=0.5)
    for a in prog.assumptions:
        if a.kind == "DTYPE_EQ":
            a.dtype = 3
    g = janus.Graph(prog)
    assert g.device_path, g.build_message
    state = gen.uniform_params(prog, 17, 0.1)
    ws = g.new_workspace()
    for k, b in enumerate(gen.lm_batches(gen.SEED_C2, B, T, V, 2)):
        args = [x.astype(np.int64) for x in b]
        dev, loss = to_dev(state), torch.zeros(1, device="cuda")
        st, _ = g.run(to_dev(args), dev, ws, outs=[loss])
        ora = I.run_imperative_step(prog, args, state, mode="bf16")
        assert st == I.OK == ora.status
        assert rel_err(float(loss.item()), ora.outputs[0]) <= 2e-2
        assert_state_parity(prog, state, to_host(dev), ora.state, 2e-2, what=f"lm i64 step {k}")
        state = ora.state
    tp = pg.treelstm_program(V=50, E=24, H=32, C=2, B=5, lr=0.1)
    for a in tp.assumptions:
        if a.kind == "DTYPE_EQ":
            a.dtype = 3
    gt = janus.Graph(tp)
    assert gt.device_path, gt.build_message
    state = gen.uniform_params(tp, 5, 0.1)
    args = [x.astype(np.int64) for x in gen.sst_forest(gen.SEED_C3, 1, 5, 50, max_leaves=12)]
    dev, loss = to_dev(state), torch.zeros(1, device="cuda")
    st, _ = gt.run(to_dev(args), dev, gt.new_workspace(), outs=[loss])
    ora = I.run_imperative_step(tp, args, state, mode="bf16")
    assert st == I.OK == ora.status
    assert rel_err(float(loss.item()), ora.outputs[0]) <= 2e-2
    assert_state_parity(tp, state, to_host(dev), ora.state, 2e-2, what="tree i64")


def test_session_cache_max_evicts_least_recently_dispatched():
    """cache_max=1: the graph generated for int64 tokens evicts the int32 graph (least recently
    dispatched); int32 batches then miss and are served imperatively, with identical results."""
    B, T, V = 8, 6, 64
    prog = pg.lstm_lm_program(V=V, E=40, H=48, L=2, B=B, T=T, lr=0.5)
    sess = J().Session(prog, cache_max=1)
    state = gen.uniform_params(prog, 19, 0.1)
    seen = []
    for k, (tok, tgt, ln) in enumerate(gen.lm_batches(gen.SEED_C2, B, T, V, 4)):
        args = (tok.astype(np.int64), tgt, ln) if k < 3 else (tok, tgt, ln)
        dev = to_dev(state)
        info, state = _check(prog, sess, args, state, dev, what=f"step {k}")
        seen.append((info["event"], info["path"]))
    assert seen == [("MISS", "imperative"), ("MISS", "imperative"), ("HIT", "graph"), ("MISS", "imperative")]
    ents = sess.stats()["entries"]
    assert [e["active"] for e in ents] == [False, True]
