"""Pins of the oracle against things other than itself (paper / SPEC worked examples, library
routines, closed forms, finite differences, brute force). CPU only."""
import json
import math
import os

import numpy as np
import pytest
import torch

from oracle import interp as I
from oracle import numerics as nm
from workloads import gen
from workloads import programs as pg

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ------------------------------------------------------------------ graph semantics (SPEC P2)
def test_spec_p2_running_sum_graph_and_imperative():
    """step([1,2,3]) -> 10.0, state 6.0; then step([1,1,1]) -> 24.0, state 9.0."""
    g = gold("spec_p2.json")
    st_graph = [np.array([0.0], np.float32)]
    st_imp = [np.array([0.0], np.float32)]
    for call in g["calls"]:
        seq = np.array(call["seq"], np.float32)
        prog = pg.running_sum_program(len(seq))
        assert float(st_graph[0][0]) == call["state_before"]
        r = I.run_graph_step(prog, [seq], st_graph, mode="f32")
        ri = I.run_imperative_step(prog, [seq], st_imp, mode="f32")
        assert r.status == I.OK
        assert float(r.outputs[0]) == call["returns"] == float(ri.outputs[0])
        assert float(r.state[0][0]) == call["state_after"] == float(ri.state[0][0])
        st_graph, st_imp = r.state, ri.state


@pytest.mark.parametrize("n", range(0, 7))
def test_loop_trip_counts_closed_form(n):
    """While frames with 0..6 iterations vs the closed form sum_{k=1..n} (s0 + k)."""
    prog = pg.running_sum_program(n)
    s0 = 2.0
    r = I.run_graph_step(prog, [np.ones(n, np.float32)], [np.array([s0], np.float32)], mode="f32")
    assert r.status == I.OK
    assert float(r.outputs[0]) == sum(s0 + k for k in range(1, n + 1))
    assert float(r.state[0][0]) == s0 + n


def test_shape_mismatch_is_dispatch_failure_and_commits_nothing():
    prog = pg.running_sum_program(3)
    st = [np.array([5.0], np.float32)]
    r = I.run_graph_step(prog, [np.ones(4, np.float32)], st, mode="f32")
    assert r.status == I.ASSUMPTION_FAILED
    assert (r.failure.assumption_id, r.failure.index, r.failure.observed) == (0, 0, 4)
    assert r.state[0].tobytes() == st[0].tobytes()


# ------------------------------------------------------------------ LSTM: library + closed form
def test_lstm_cell_closed_form():
    """H=E=1, x=1, W_ih=[1,1,1,1], W_hh=0, b=0, h0=c0=0: c = s(1) tanh(1), h = s(1) tanh(c)
    (SURVEY §8(c) closed form: 0.5567699411 / 0.3696063529)."""
    P = nm.Prec("f32")
    h, c, _ = nm.lstm_fwd(P, np.ones((1, 1)), np.zeros((1, 1)), np.zeros((1, 1)), np.ones((4, 1)),
                          np.zeros((4, 1)), np.zeros(4), np.ones(1))
    s1 = 1 / (1 + math.exp(-1))
    assert abs(c[0, 0] - s1 * math.tanh(1)) < 1e-15
    assert abs(c[0, 0] - 0.5567699411) < 1e-10
    assert abs(h[0, 0] - 0.3696063529) < 1e-10


def _pattern(rows, cols, a, b, m, scale, off):
    return np.array([[scale * ((a * r + b * c) % m) - off for c in range(cols)] for r in range(rows)])


def _plm_state(prog):
    g = gold("p_lm.json")
    st = [np.zeros(s.shape) for s in prog.slots]
    sid = {s.name: k for k, s in enumerate(prog.slots)}
    st[sid["E"]] = np.array(g["E"])
    st[sid["W_ih0"]] = _pattern(8, 2, 2, 1, 5, 0.1, 0.2)
    st[sid["W_hh0"]] = _pattern(8, 2, 2, 1, 7, 0.05, 0.15)
    st[sid["b0"]] = 0.01 * np.arange(8)
    st[sid["W_dec"]] = np.array(g["W_dec"])
    st[sid["b_dec"]] = np.array(g["b_dec"])
    st[sid["tag"]] = np.ones(1, np.int32)
    return g, st, sid


def test_p_lm_golden():
    prog = pg.lstm_lm_program(V=3, E=2, H=2, L=1, B=1, T=2, lr=0.0)
    g, st, sid = _plm_state(prog)
    args = [np.array(g["tokens"], np.int32), np.array(g["targets"], np.int32), np.array([2], np.int32)]
    r = I.run_graph_step(prog, args, st, mode="f32")
    e = g["expected"]
    assert r.status == I.OK
    assert abs(float(r.outputs[0]) - e["loss"]) < 1e-11
    np.testing.assert_allclose(r.state[sid["h0"]][0], e["h_T"], atol=1e-11)
    np.testing.assert_allclose(r.state[sid["c0"]][0], e["c_T"], atol=1e-11)
    gr = r.grads
    assert abs(gr[sid["W_hh0"]][0, 0] - e["dW_hh[0,0]"]) < 1e-15
    assert abs(gr[sid["W_ih0"]][1, 0] - e["dW_ih[1,0]"]) < 1e-14
    assert abs(gr[sid["b0"]][2] - e["db[2]"]) < 1e-15
    np.testing.assert_allclose(gr[sid["E"]][0], e["dE[0]"], atol=1e-14)
    np.testing.assert_allclose(gr[sid["E"]][2], e["dE[2]"], atol=1e-14)
    assert abs(gr[sid["W_dec"]][2, 1] - e["dW_dec[2,1]"]) < 1e-14


def _torch_lm(prog, st, args):
    """The same LM with torch.nn.LSTM / cross_entropy + autograd, fp64 (a library routine)."""
    m = prog.meta
    sid = {s.name: k for k, s in enumerate(prog.slots)}
    L, H, E = m["L"], m["H"], m["E"]
    tok, tgt, lens = args
    T = tok.shape[1]
    P = {k: torch.tensor(np.asarray(st[sid[k]], np.float64), requires_grad=True)
         for k in ["E", "W_dec", "b_dec"] + [f"{p}{l}" for l in range(L) for p in ("W_ih", "W_hh", "b")]}
    lstm = torch.nn.LSTM(E, H, num_layers=L).double()
    x = P["E"][torch.tensor(tok.T.astype(np.int64))]            # [T, B, E]
    h0 = torch.tensor(np.stack([st[sid[f"h{l}"]] for l in range(L)]).astype(np.float64))
    c0 = torch.tensor(np.stack([st[sid[f"c{l}"]] for l in range(L)]).astype(np.float64))
    out, (hT, cT) = torch.func.functional_call(
        lstm, {f"{n}_l{l}": P[f"{k}{l}"] for l in range(L) for n, k in
               (("weight_ih", "W_ih"), ("weight_hh", "W_hh"), ("bias_ih", "b"))} |
        {f"bias_hh_l{l}": torch.zeros(4 * H, dtype=torch.float64) for l in range(L)}, (x, (h0, c0)))
    logits = out.reshape(T * tok.shape[0], H) @ P["W_dec"].T + P["b_dec"]
    loss = torch.nn.functional.cross_entropy(logits, torch.tensor(tgt.T.reshape(-1).astype(np.int64)))
    loss.backward()
    return loss.item(), hT.detach().numpy(), cT.detach().numpy(), {k: v.grad.numpy() for k, v in P.items()}


@pytest.mark.parametrize("L,H,E,V,B,T", [(1, 3, 3, 5, 2, 3), (2, 4, 3, 7, 3, 4)])
def test_lm_matches_torch_lstm_fp64(L, H, E, V, B, T):
    prog = pg.lstm_lm_program(V=V, E=E, H=H, L=L, B=B, T=T, lr=0.0)
    st = [np.asarray(s, np.float64) if s.dtype.kind == "f" else s for s in gen.uniform_params(prog, 7, 0.4)]
    sid = {s.name: k for k, s in enumerate(prog.slots)}
    r0 = gen.rng(3)
    for l in range(L):  # non-zero carried state
        st[sid[f"h{l}"]] = r0.uniform(-0.5, 0.5, (B, H))
        st[sid[f"c{l}"]] = r0.uniform(-0.5, 0.5, (B, H))
    tok = r0.integers(0, V, (B, T)).astype(np.int32)
    tgt = r0.integers(0, V, (B, T)).astype(np.int32)
    args = [tok, tgt, np.full(B, T, np.int32)]
    r = I.run_graph_step(prog, args, st, mode="f32")
    loss, hT, cT, grads = _torch_lm(prog, st, args)
    assert abs(float(r.outputs[0]) - loss) < 1e-12
    for l in range(L):
        np.testing.assert_allclose(r.state[sid[f"h{l}"]], hT[l], atol=1e-12)
        np.testing.assert_allclose(r.state[sid[f"c{l}"]], cT[l], atol=1e-12)
    for k, gt in grads.items():
        np.testing.assert_allclose(r.grads[sid[k]], gt, atol=1e-12, err_msg=k)


def test_lm_fd_gradients():
    prog = pg.lstm_lm_program(V=5, E=3, H=3, L=2, B=2, T=3, lr=0.0)
    st = [np.asarray(s, np.float64) if s.dtype.kind == "f" else s for s in gen.uniform_params(prog, 11, 0.6)]
    r0 = gen.rng(4)
    args = [r0.integers(0, 5, (2, 3)).astype(np.int32), r0.integers(0, 5, (2, 3)).astype(np.int32),
            np.array([3, 3], np.int32)]
    r = I.run_graph_step(prog, args, st, mode="f32")
    eps = 1e-6
    for slot, s in enumerate(prog.slots):
        if not s.param:
            continue
        flat = st[slot].reshape(-1)
        for k in range(0, flat.size, max(1, flat.size // 4)):
            sp = [x.copy() for x in st]
            sm = [x.copy() for x in st]
            sp[slot].reshape(-1)[k] += eps
            sm[slot].reshape(-1)[k] -= eps
            fd = (float(I.run_graph_step(prog, args, sp, mode="f32").outputs[0]) -
                  float(I.run_graph_step(prog, args, sm, mode="f32").outputs[0])) / (2 * eps)
            an = r.grads[slot].reshape(-1)[k]
            assert abs(fd - an) <= 1e-6 * max(1e-3, abs(an)) + 1e-9, (s.name, k, fd, an)


# ------------------------------------------------------------------ softmax cross-entropy
def test_xent_uniform_logits_closed_form():
    V, R = 10000, 6
    logits = np.zeros((R, V))
    tgt = np.arange(R)
    loss, saved = nm.xent_fwd(logits, tgt, np.ones(R))
    assert abs(loss - math.log(V)) < 1e-12 and abs(math.log(V) - 9.210340371976184) < 1e-12
    dy = nm.xent_vjp(logits, saved, 1.0)
    exp = np.full((R, V), 1.0 / V)
    exp[np.arange(R), tgt] -= 1.0
    np.testing.assert_allclose(dy, exp / R, atol=1e-15)


def test_xent_masked_matches_torch():
    r = gen.rng(9)
    logits = r.normal(size=(7, 11))
    tgt = r.integers(0, 11, 7)
    mask = np.array([1, 1, 0, 1, 0, 1, 1])
    loss, _ = nm.xent_fwd(logits, tgt, mask)
    keep = mask.astype(bool)
    ref = torch.nn.functional.cross_entropy(torch.tensor(logits[keep]), torch.tensor(tgt[keep])).item()
    assert abs(loss - ref) < 1e-13
    assert nm.xent_fwd(logits, tgt, np.zeros(7))[0] == 0.0   # reading Q18: empty mean is 0


# ------------------------------------------------------------------ bf16 rounding
def test_bf16_rounding_matches_torch():
    r = gen.rng(1)
    x = np.concatenate([r.normal(size=4000).astype(np.float32),
                        # exact ties: low 16 bits 0x8000 (round half to even)
                        (np.arange(1, 200, dtype=np.uint32) << 16 | 0x8000).view(np.float32),
                        np.array([0.0, -0.0, 1e-40, 3.4e38], np.float32)])
    ref = torch.tensor(x).to(torch.bfloat16).to(torch.float64).numpy()
    np.testing.assert_array_equal(nm.rb(x), ref)


# ------------------------------------------------------------------ TreeLSTM
def _ptree():
    g = gold("p_tree.json")
    prog = pg.treelstm_program(V=3, E=2, H=2, C=2, B=1, lr=0.0)
    sid = {s.name: k for k, s in enumerate(prog.slots)}
    st = [np.zeros(s.shape) for s in prog.slots]
    st[sid["E"]] = np.array(g["E"])
    st[sid["W_leaf"]] = _pattern(6, 2, 3, 1, 7, 0.1, 0.3)
    st[sid["U"]] = _pattern(10, 4, 5, 1, 11, 0.05, 0.25)
    st[sid["b"]] = np.concatenate([g["b_i"], g["b_f"], g["b_o"], g["b_u"]])
    st[sid["W_c"]] = np.array(g["W_c"])
    st[sid["b_c"]] = np.array(g["b_c"])
    args = [np.array(x, np.int32) for x in ([0, 0, 1, 0, 1], [-1, -1, 0, -1, 2], [-1, -1, 1, -1, 3],
                                            [0, 1, -1, 2, -1], [0, 5], [g["label"]])]
    return g, prog, sid, st, args


def test_p_tree_golden():
    g, prog, sid, st, args = _ptree()
    r = I.run_graph_step(prog, args, st, mode="f32")
    e = g["expected"]
    assert r.status == I.OK
    assert abs(float(r.outputs[0]) - e["loss"]) < 1e-11
    assert abs(r.grads[sid["U"]][0, 0] - e["dU[0,0]"]) < 1e-15
    assert abs(r.grads[sid["U"]][9, 3] - e["dU[9,3]"]) < 1e-15
    assert abs(r.grads[sid["W_leaf"]][0, 0] - e["dW_leaf[0,0]"]) < 1e-14
    np.testing.assert_allclose(r.grads[sid["b"]][2:4], e["db_f"], atol=1e-14)
    ex = I.GraphExec(prog, args, st, nm.Prec("f32"))
    ex.run_body(0, None)
    roots = [e_ for e_ in ex.tape.entries if e_[0] == "TA_STACK"][0][2][0].data
    np.testing.assert_allclose(roots[0], e["root_h"], atol=1e-11)


def _depths(shape, d=0):
    return [d] if shape is None else _depths(shape[0], d + 1) + _depths(shape[1], d + 1)


@pytest.mark.parametrize("n", range(1, 9))
def test_tree_closed_form_all_shapes(n):
    """U = 0, b = 0: every internal node has i = f_l = f_r = o = 1/2, u = 0, so
    c_root = sum over leaves of 0.5^depth * c_leaf; all Catalan(n-1) shapes."""
    shapes = gen.all_shapes(n)
    H, E, V = 3, 2, 11
    prog = pg.treelstm_program(V=V, E=E, H=H, C=2, B=len(shapes), lr=0.0)
    sid = {s.name: k for k, s in enumerate(prog.slots)}
    r = gen.rng(n)
    st = [np.zeros(s.shape) for s in prog.slots]
    st[sid["E"]] = r.uniform(-1, 1, (V, E))
    st[sid["W_leaf"]] = r.uniform(-1, 1, (3 * H, E))
    st[sid["W_c"]] = r.uniform(-1, 1, (2, H))
    words = r.integers(0, V, n * len(shapes))
    f = gen.forest_from_shapes(shapes, words)
    args = list(f) + [np.zeros(len(shapes), np.int32)]
    ex = I.GraphExec(prog, args, st, nm.Prec("f32"))
    ex.run_body(0, None)
    leaves = [e for e in ex.tape.entries if e[0] == "TREELSTM_LEAF"]
    cells = [e for e in ex.tape.entries if e[0] == "TREELSTM_CELL"]
    assert len(leaves) == n * len(shapes) and len(cells) == (n - 1) * len(shapes)
    li = 0
    roots = [e_ for e_ in ex.tape.entries if e_[0] == "TA_STACK"][0][1]
    for t, s in enumerate(shapes):
        dep = _depths(s)
        c_leaf = [leaves[li + k][2][1].data[0] for k in range(n)]
        li += n
        c_root = sum(0.5 ** d * c for d, c in zip(dep, c_leaf))
        h_root = roots[t].data[0]
        if n == 1:   # lone root leaf: c = s(z_i) tanh(z_u)
            np.testing.assert_allclose(h_root, leaves[li - 1][2][0].data[0], atol=0)
        else:
            np.testing.assert_allclose(h_root, 0.5 * np.tanh(c_root), atol=1e-15)


def test_tree_fd_gradients():
    prog = pg.treelstm_program(V=6, E=2, H=2, C=2, B=2, lr=0.0)
    st = [np.asarray(s, np.float64) for s in gen.uniform_params(prog, 5, 0.7)]
    f = gen.forest_from_shapes([((None, None), None), (None, (None, None))], [0, 1, 2, 3, 4, 5])
    args = list(f) + [np.array([1, 0], np.int32)]
    r = I.run_graph_step(prog, args, st, mode="f32")
    eps = 1e-6
    for slot, s in enumerate(prog.slots):
        if not s.param:
            continue
        for k in range(st[slot].size):
            sp = [x.copy() for x in st]; sm = [x.copy() for x in st]
            sp[slot].reshape(-1)[k] += eps; sm[slot].reshape(-1)[k] -= eps
            fd = (float(I.run_graph_step(prog, args, sp, mode="f32").outputs[0]) -
                  float(I.run_graph_step(prog, args, sm, mode="f32").outputs[0])) / (2 * eps)
            an = r.grads[slot].reshape(-1)[k]
            assert abs(fd - an) <= 1e-6 * max(1e-3, abs(an)) + 1e-10, (s.name, k, fd, an)


def test_tree_schedule_golden():
    g = gold("p_sched.json")
    s = I.tree_schedule(g["kind"], g["left"], g["right"], g["tree_off"])
    e = g["expected"]
    for k in ("height", "order", "level_offset", "pos"):
        assert s[k].tolist() == e[k], k
    assert s["parent_slot"].tolist() == e["parent_slot"]


def _level_eval(P, kind, left, right, word, off, Emb, W_leaf, U, b):
    """Evaluate a forest level by level with the oracle schedule (batched rows per level)."""
    sch = I.tree_schedule(kind, left, right, off)
    N = len(kind)
    H = W_leaf.shape[0] // 3
    h = np.zeros((N, H)); c = np.zeros((N, H))
    lo = sch["level_offset"]
    for l in range(len(lo) - 1):
        nodes = sch["order"][lo[l]:lo[l + 1]]
        if l == 0:
            hh, cc, _ = nm.tree_leaf_fwd(P, nm.embedding_fwd(P, Emb, word[nodes]), W_leaf, b)
        else:
            hh, cc, _ = nm.tree_cell_fwd(P, h[left[nodes]], c[left[nodes]], h[right[nodes]],
                                         c[right[nodes]], U, b)
        h[nodes], c[nodes] = hh, cc
    return h[np.asarray(off[1:]) - 1]


@pytest.mark.parametrize("mode", ["f32", "bf16"])
def test_level_batched_equals_recursion(mode):
    """The level schedule (reading Q8) is a valid evaluation order: level-batched evaluation equals
    the InvokeOp recursion of the oracle over all shapes with <= 6 leaves + SST forests."""
    P = nm.Prec(mode)
    H, E, V = 3, 2, 13
    prog = pg.treelstm_program(V=V, E=E, H=H, C=2, B=1, lr=0.0)
    st = gen.uniform_params(prog, 2, 0.8)
    sid = {s.name: k for k, s in enumerate(prog.slots)}
    shapes = [s for n in range(1, 7) for s in gen.all_shapes(n)]
    forests = [gen.forest_from_shapes(shapes, gen.rng(0).integers(0, V, sum(map(gen.n_leaves, shapes))))]
    forests += [gen.sst_forest(gen.SEED_C3, k, 6, V, max_leaves=20)[:5] for k in range(3)]
    for f in forests:
        kind, left, right, word, off = (np.asarray(x, np.int64) for x in f)
        prog = pg.treelstm_program(V=V, E=E, H=H, C=2, B=len(off) - 1, lr=0.0)
        ex = I.GraphExec(prog, list(f) + [np.zeros(len(off) - 1, np.int32)], st, P)
        ex.run_body(0, None)
        roots = np.concatenate([v.data for v in [e for e in ex.tape.entries if e[0] == "TA_STACK"][0][1]])
        lv = _level_eval(P, kind, left, right, word, off, *(np.asarray(st[sid[k]], np.float64)
                                                           for k in ("E", "W_leaf", "U", "b")))
        np.testing.assert_allclose(lv, roots, rtol=0, atol=1e-14)


# ------------------------------------------------------------------ guards (AssertOp)
def test_c1_hand_worked_assert_failure():
    """Hand-worked C1 case: TRIP_COUNT(8) is id 2; lengths [8,8,7,8] ->
    ASSUMPTION_FAILED{id 2, index 2, observed 7}, every state byte unchanged."""
    prog = pg.lstm_lm_program(V=32, E=16, H=16, L=1, B=4, T=8, lr=0.1, gemm="f32")
    st = gen.uniform_params(prog, gen.SEED_C1, 0.1)
    tok, tgt, ln = gen.c1_batches()[3]
    assert ln.tolist() == [8, 8, 7, 8]
    r = I.run_graph_step(prog, [tok, tgt, ln], st, mode="f32")
    assert r.status == I.ASSUMPTION_FAILED
    assert (r.failure.assumption_id, r.failure.index, r.failure.observed) == (2, 2, 7)
    assert all(a.tobytes() == b.tobytes() for a, b in zip(r.state, st))
    ri = I.run_imperative_step(prog, [tok, tgt, ln], st, mode="f32")   # fallback
    assert ri.status == I.OK
    assert any(a.tobytes() != b.tobytes() for a, b in zip(ri.state, st))


def test_guard_comparators_spec_examples():
    """PartialShape(?,8) matches (6,8); Shape(4,8) fails on (3,8). S:449-451 EqInt."""
    ok = pg.Program("t", [], [pg.Assumption(0, "SHAPE_MATCH", 0, 0, dims=(-1, 8))], [], [], 0, 0.0)
    assert I.check_dispatch(ok, [np.zeros((6, 8))]) is None
    bad = pg.Program("t", [], [pg.Assumption(3, "SHAPE_MATCH", 0, 0, dims=(4, 8))], [], [], 0, 0.0)
    f = I.check_dispatch(bad, [np.zeros((3, 8))])
    assert (f.assumption_id, f.index, f.observed) == (3, 0, 3)
    eq = pg.Program("t", [], [pg.Assumption(5, "VALUE_EQ", 1, 0, value=3)], [], [], 0, 0.0)
    f = I.check_runtime(eq, [np.array([4], np.int32)], [])
    assert (f.assumption_id, f.observed) == (5, 4)


def test_minimum_failing_id_and_fault_injection():
    prog = pg.lstm_lm_program(V=32, E=16, H=16, L=1, B=4, T=8, lr=0.1)
    st = gen.uniform_params(prog, 1, 0.1)
    st[prog.slot_index("tag")][:] = 0     # TYPE_TAG (id 3) fails too
    tok, tgt, ln = gen.c1_batches()[3]
    f = I.check_guards(prog, [tok, tgt, ln], st)
    assert f.assumption_id == 2            # min(2, 3)
    tok, tgt, ln = gen.c1_batches()[0]
    f = I.check_guards(prog, [tok, tgt, ln], st)
    assert (f.assumption_id, f.index, f.observed) == (3, 0, 0)
    st[prog.slot_index("tag")][:] = 1
    assert I.check_guards(prog, [tok, tgt, ln], st) is None
    for a in prog.assumptions:
        f = I.check_guards(prog, [tok, tgt, ln], st, fail_assert_id=a.id)
        assert f.assumption_id == a.id


def test_tree_binary_violations():
    f = gen.forest_from_shapes([((None, None), None), (None, None)], [0, 1, 2, 3, 4])
    kind, left, right, word, off = (x.copy() for x in f)
    assert I.tree_binary_violation(kind, left, right, word, off, 5, 127) is None
    w2 = word.copy(); w2[3] = 5                               # word out of range
    assert I.tree_binary_violation(kind, left, right, w2, off, 5, 127) == (3, 0)
    r2 = right.copy(); r2[2] = 0                              # l == r (unary node)
    # node 2 is rejected and its orphaned children 0, 1 have no parent: smallest index wins
    assert I.tree_binary_violation(kind, left, r2, word, off, 5, 127) == (0, 0)
    l2 = left.copy(); l2[7] = 1                   # child in another tree: node 7 rejected,
    assert I.tree_binary_violation(kind, l2, right, word, off, 5, 127) == (5, 0)  # 5 orphaned
    assert I.tree_binary_violation(kind, left, right, word, off, 5, 4) == (len(kind) + 1, 5)


# ------------------------------------------------------------------ data parallel
def test_dp_average_equals_global_batch():
    """Equal shards: mean of shard-mean gradients = global-batch mean gradient (identity); every
    rank commits identical parameters."""
    B, T, V = 3, 4, 9
    prog1 = pg.lstm_lm_program(V=V, E=4, H=5, L=2, B=B, T=T, lr=0.5)
    prog2 = pg.lstm_lm_program(V=V, E=4, H=5, L=2, B=2 * B, T=T, lr=0.5)
    st = [np.asarray(s, np.float64) if s.dtype.kind == "f" else s for s in gen.uniform_params(prog1, 3, 0.3)]
    sid = {s.name: k for k, s in enumerate(prog1.slots)}
    r0 = gen.rng(8)
    tok = r0.integers(0, V, (2 * B, T)).astype(np.int32)
    tgt = r0.integers(0, V, (2 * B, T)).astype(np.int32)
    ln = np.full(2 * B, T, np.int32)
    hs = {k: r0.uniform(-1, 1, (2 * B, 5)) for k in ("h0", "c0", "h1", "c1")}
    shard_st = []
    for r in range(2):
        s = [x.copy() for x in st]
        for k, v in hs.items():
            s[sid[k]] = v[r * B:(r + 1) * B].copy()
        shard_st.append(s)
    dp = I.run_dp_step(prog1, [[tok[r * B:(r + 1) * B], tgt[r * B:(r + 1) * B], ln[:B]] for r in range(2)],
                       shard_st, mode="f32")
    g_st = [x.copy() for x in st]
    for k, v in hs.items():
        g_st[sid[k]] = v
    full = I.run_graph_step(prog2, [tok, tgt, ln], g_st, mode="f32")
    for s in prog1.slots:
        if s.param:
            k = sid[s.name]
            np.testing.assert_allclose(dp[0].state[k], full.state[k], atol=1e-13)
            assert dp[0].state[k].tobytes() == dp[1].state[k].tobytes()
    f = I.run_dp_step(prog1, [[tok[:B], tgt[:B], ln[:B]], [tok[B:], tgt[B:], np.array([T, T - 1, T], np.int32)]],
                      shard_st, mode="f32")
    assert all(r.status == I.ASSUMPTION_FAILED and r.failure.rank == 1 for r in f)
    assert all(a.tobytes() == b.tobytes() for r, s in zip(f, shard_st) for a, b in zip(r.state, s))


def test_runtime_error_commits_nothing():
    prog = pg.lstm_lm_program(V=8, E=3, H=3, L=1, B=2, T=2, lr=0.1)
    st = gen.uniform_params(prog, 1, 0.1)
    tok = np.array([[0, 9], [1, 2]], np.int32)   # token 9 >= V
    r = I.run_graph_step(prog, [tok, tok, np.array([2, 2], np.int32)], st)
    assert r.status == I.ERR_RUNTIME
    assert all(a.tobytes() == b.tobytes() for a, b in zip(r.state, st))


def test_tree_program_batch_from_len_partial_minibatch():
    """The TreeLSTM op list loops `for i < len(label)` (LEN, the whitelisted `len` of P:230): the
    graph interpretation of a program written for B trees, run on a partial last minibatch of B-1
    (P:314), equals the imperative program on the same forest — and a program whose loop bound
    were the constant B would index past tree_off instead."""
    V, B = 17, 5
    prog = pg.treelstm_program(V=V, E=4, H=3, C=2, B=B, lr=0.3, speculate="none")
    prog.assumptions = [a for a in prog.assumptions if a.kind != "SHAPE_MATCH"]   # any batch size
    st = gen.uniform_params(prog, 7, 0.5)
    f = list(gen.sst_forest(gen.SEED_C3, 3, B - 1, V, max_leaves=6))
    g = I.run_graph_step(prog, f, st, mode="f32")
    m = I.run_imperative_step(prog, f, st, mode="f32")
    assert g.status == m.status == I.OK
    assert abs(float(g.outputs[0]) - float(m.outputs[0])) <= 1e-6 * abs(float(m.outputs[0]))
    for a, b in zip(g.state, m.state):
        np.testing.assert_allclose(np.asarray(a, np.float64), np.asarray(b, np.float64), rtol=1e-5, atol=1e-7)
    # the loop really ran over the 4 trees: the mean loss equals the mean of single-tree losses
    offs = f[4]
    per = []
    for t in range(B - 1):
        lo, hi = int(offs[t]), int(offs[t + 1])
        sub = [np.asarray(x[lo:hi]) for x in f[:4]]
        sub[1] = np.where(sub[0] == 1, sub[1] - lo, sub[1])
        sub[2] = np.where(sub[0] == 1, sub[2] - lo, sub[2])
        one = sub + [np.array([0, hi - lo], np.int32), np.asarray(f[5][t:t + 1])]
        per.append(float(I.run_imperative_step(prog, one, st, mode="f32").outputs[0]))
    assert abs(float(m.outputs[0]) - np.mean(per)) <= 1e-5 * abs(np.mean(per))
