"""Pins of the oracle parts the round-1 pins left open (VERDICT r1 "What's weak" 1): masked LSTM
rows (C4, reading Q18), the RANGE guard with its shape bound, the imperative LM program, the SGD
commit, and the bf16 rounding placement R1-R4. Every expected value comes from something other
than the oracle: torch (a library routine with autograd), finite differences, or a case worked
by hand below. CPU only."""
import numpy as np
import pytest
import torch

from oracle import interp as I
from oracle import numerics as nm
from workloads import gen
from workloads import programs as pg


@pytest.fixture(autouse=True)
def _fp64_default():
    """fp64 torch references for this module only (the GPU tests allocate fp32 by default)."""
    old = torch.get_default_dtype()
    torch.set_default_dtype(torch.float64)
    yield
    torch.set_default_dtype(old)


# ----------------------------------------------------------------------------- torch references
def _rbt(x):
    """RNE to bf16 through fp32 with torch's own conversions (pinned in test_bf16_rounding)."""
    return x.to(torch.float32).to(torch.bfloat16).to(torch.float64)


class _RoundFwd(torch.autograd.Function):
    """R1/R2: a GEMM operand copy rb(x); the gradient reaches x unchanged (the copy is a cast)."""

    @staticmethod
    def forward(ctx, x):
        return _rbt(x)

    @staticmethod
    def backward(ctx, g):
        return g


class _RoundBwd(torch.autograd.Function):
    """R3: identity forward; the incoming gradient (dz, dy) is rounded before it reaches the
    GEMMs (and the bias add) that produced the value."""

    @staticmethod
    def forward(ctx, x):
        return x.clone()

    @staticmethod
    def backward(ctx, g):
        return _rbt(g)


def _torch_lm(prog, st, args, bf16, training=True):
    """The LM step written directly in torch (cell equations of reading Q1, masked rows of Q18,
    mean over valid tokens of Q3), backward by torch autograd. bf16=True inserts the rounding
    points R1-R3 (R4 follows: the bias add's gradient is the rounded dz)."""
    m = prog.meta
    sid = {s.name: k for k, s in enumerate(prog.slots)}
    L, H = m["L"], m["H"]
    tok, tgt, lens = (np.asarray(a, np.int64) for a in args[:3])
    B = tok.shape[0]
    T = int(lens.max())
    R = _RoundFwd.apply if bf16 else (lambda x: x)
    G = _RoundBwd.apply if bf16 else (lambda x: x)
    names = ["E", "W_dec", "b_dec"] + [f"{p}{l}" for l in range(L) for p in ("W_ih", "W_hh", "b")]
    P = {k: torch.tensor(np.asarray(st[sid[k]], np.float64), requires_grad=True) for k in names}
    is_tensor = int(np.asarray(st[sid["tag"]]).reshape(-1)[0]) == 1
    h = [torch.tensor(np.asarray(st[sid[f"h{l}"]], np.float64)) * (1.0 if is_tensor else 0.0) for l in range(L)]
    c = [torch.tensor(np.asarray(st[sid[f"c{l}"]], np.float64)) * (1.0 if is_tensor else 0.0) for l in range(L)]
    Er = R(P["E"])
    outs = []
    for t in range(T):
        x = Er[torch.tensor(tok[:, t])]
        v = torch.tensor((t < lens).astype(np.float64))[:, None]
        for l in range(L):
            z = G(R(x) @ R(P[f"W_ih{l}"]).T + R(h[l]) @ R(P[f"W_hh{l}"]).T + P[f"b{l}"])
            i, f = torch.sigmoid(z[:, :H]), torch.sigmoid(z[:, H:2 * H])
            g, o = torch.tanh(z[:, 2 * H:3 * H]), torch.sigmoid(z[:, 3 * H:])
            c2 = f * c[l] + i * g
            h2 = o * torch.tanh(c2)
            h[l] = v * h2 + (1 - v) * h[l]
            c[l] = v * c2 + (1 - v) * c[l]
            x = h[l]
        outs.append(x)
    hs = torch.cat(outs, 0)                                     # time-major rows t*B + b
    logits = G(R(hs) @ R(P["W_dec"]).T + P["b_dec"])
    mask = torch.tensor((np.arange(T)[:, None] < lens[None, :]).reshape(-1))
    tg = torch.tensor(tgt[:, :T].T.reshape(-1))
    per = torch.nn.functional.cross_entropy(logits, tg, reduction="none")
    n = max(1, int(mask.sum()))
    loss = (per * mask).sum() / n
    loss.backward()
    grads = {k: v.grad.numpy().copy() for k, v in P.items()}
    return float(loss.detach()), [x.detach().numpy() for x in h], [x.detach().numpy() for x in c], grads


def _lm_state(prog, seed, scale, B, H, L, carried=True):
    st = [np.asarray(s, np.float64) if s.dtype.kind == "f" else s for s in gen.uniform_params(prog, seed, scale)]
    sid = {s.name: k for k, s in enumerate(prog.slots)}
    if carried:
        r0 = gen.rng(seed + 100)
        for l in range(L):
            st[sid[f"h{l}"]] = r0.uniform(-0.5, 0.5, (B, H))
            st[sid[f"c{l}"]] = r0.uniform(-0.5, 0.5, (B, H))
    return st, sid


def _ragged(B, W, V, lens, seed=5):
    r = gen.rng(seed)
    return [r.integers(0, V, (B, W)).astype(np.int32), r.integers(0, V, (B, W)).astype(np.int32),
            np.asarray(lens, np.int32)]


# ----------------------------------------------------------------------------- masked rows (C4)
def test_masked_rows_match_per_row_torch_lstm():
    """Ragged lengths through the While program (reading Q18): each row's final state equals a
    torch.nn.LSTM run over that row's own len_b tokens alone, from its own carried state; the loss
    is the mean over the valid tokens of those per-row runs (library routines, fp64)."""
    B, W, V, E, H, L = 4, 5, 9, 3, 4, 2
    lens = [5, 2, 1, 3]
    prog = pg.lstm_lm_program(V=V, E=E, H=H, L=L, B=B, T=W, lr=0.0, speculate="while")
    st, sid = _lm_state(prog, 21, 0.5, B, H, L)
    args = _ragged(B, W, V, lens)
    r = I.run_graph_step(prog, args, st, mode="f32")
    assert r.status == I.OK and set(r.trace["trip_counts"]) == {max(lens)}
    lstm = torch.nn.LSTM(E, H, num_layers=L)
    names = {f"{n}_l{l}": torch.tensor(np.asarray(st[sid[f"{k}{l}"]], np.float64)) for l in range(L)
             for n, k in (("weight_ih", "W_ih"), ("weight_hh", "W_hh"), ("bias_ih", "b"))}
    names |= {f"bias_hh_l{l}": torch.zeros(4 * H) for l in range(L)}
    Emb = torch.tensor(st[sid["E"]])
    Wd, bd = torch.tensor(st[sid["W_dec"]]), torch.tensor(st[sid["b_dec"]])
    tot, n = 0.0, 0
    for b, lb in enumerate(lens):
        x = Emb[torch.tensor(args[0][b, :lb].astype(np.int64))][:, None, :]
        h0 = torch.tensor(np.stack([st[sid[f"h{l}"]][b:b + 1] for l in range(L)]))
        c0 = torch.tensor(np.stack([st[sid[f"c{l}"]][b:b + 1] for l in range(L)]))
        out, (hT, cT) = torch.func.functional_call(lstm, names, (x, (h0, c0)))
        for l in range(L):
            np.testing.assert_allclose(r.state[sid[f"h{l}"]][b], hT[l, 0].numpy(), atol=1e-13)
            np.testing.assert_allclose(r.state[sid[f"c{l}"]][b], cT[l, 0].numpy(), atol=1e-13)
        logits = out[:, 0, :] @ Wd.T + bd
        tot += float(torch.nn.functional.cross_entropy(
            logits, torch.tensor(args[1][b, :lb].astype(np.int64)), reduction="sum"))
        n += lb
    assert abs(float(r.outputs[0]) - tot / n) < 1e-12


def test_masked_rows_gradients_match_torch_and_fd():
    """The masked backward (dh, dc pass through rows with t >= len_b) against torch autograd of
    the per-row computation, and a central finite difference of the oracle's own loss."""
    B, W, V, E, H, L = 3, 4, 7, 3, 3, 2
    lens = [4, 2, 1]
    prog = pg.lstm_lm_program(V=V, E=E, H=H, L=L, B=B, T=W, lr=0.0, speculate="while")
    st, sid = _lm_state(prog, 23, 0.6, B, H, L)
    args = _ragged(B, W, V, lens, seed=8)
    r = I.run_graph_step(prog, args, st, mode="f32")
    loss, hT, cT, grads = _torch_lm(prog, st, args, bf16=False)
    assert abs(float(r.outputs[0]) - loss) < 1e-12
    for k, gt in grads.items():
        np.testing.assert_allclose(r.grads[sid[k]], gt, atol=1e-12, err_msg=k)
    eps = 1e-6
    for name in ("W_hh0", "W_ih1", "E", "b1"):
        slot = sid[name]
        flat = st[slot].reshape(-1)
        for k in range(0, flat.size, max(1, flat.size // 5)):
            sp = [x.copy() for x in st]; sm = [x.copy() for x in st]
            sp[slot].reshape(-1)[k] += eps; sm[slot].reshape(-1)[k] -= eps
            fd = (float(I.run_graph_step(prog, args, sp, mode="f32").outputs[0]) -
                  float(I.run_graph_step(prog, args, sm, mode="f32").outputs[0])) / (2 * eps)
            an = r.grads[slot].reshape(-1)[k]
            assert abs(fd - an) <= 1e-6 * max(1e-3, abs(an)) + 1e-10, (name, k, fd, an)


def test_padding_tokens_do_not_matter():
    """Tokens and targets at t >= len_b never influence the result (masked rows, Q18)."""
    B, W, V = 3, 6, 11
    lens = [6, 3, 1]
    prog = pg.lstm_lm_program(V=V, E=3, H=4, L=2, B=B, T=W, lr=0.5, speculate="while")
    st, _ = _lm_state(prog, 3, 0.5, B, 4, 2)
    a = _ragged(B, W, V, lens, seed=1)
    b = [x.copy() for x in a]
    for row, lb in enumerate(lens):
        b[0][row, lb:] = (b[0][row, lb:] + 5) % V
        b[1][row, lb:] = (b[1][row, lb:] + 3) % V
    ra, rb_ = I.run_graph_step(prog, a, st, mode="f32"), I.run_graph_step(prog, b, st, mode="f32")
    assert float(ra.outputs[0]) == float(rb_.outputs[0])
    assert all(np.array_equal(x, y) for x, y in zip(ra.state, rb_.state))


# ----------------------------------------------------------------------------- RANGE guard
def test_range_guard_hand_worked():
    """RANGE(id 2): 1 <= lengths[b] <= min(hi, tokens.shape[1]) (janus.h JA_RANGE with ref_arg).
    Worked by hand: the first failing element is reported, the minimum id wins over TYPE_TAG
    (id 3), and nothing is committed."""
    B, W, V = 4, 5, 9
    prog = pg.lstm_lm_program(V=V, E=3, H=3, L=1, B=B, T=W, lr=0.5, speculate="while")
    rng_a = [a for a in prog.assumptions if a.kind == "RANGE"][0]
    assert (rng_a.id, rng_a.lo, rng_a.hi, rng_a.ref_arg, rng_a.ref_dim) == (2, 1, W, 0, 1)
    st = gen.uniform_params(prog, 1, 0.2)
    tok = np.zeros((B, W), np.int32)
    cases = [
        (tok, [3, 0, 2, 7], (2, 1, 0)),          # length 0 < lo: element 1 (the first of two)
        (tok, [5, 5, 6, 1], (2, 2, 6)),          # 6 > hi = 5
        (tok[:, :3], [3, 4, 2, 1], (2, 1, 4)),   # 4 > width 3 of this batch (hi = min(5, 3))
        (tok[:, :3], [3, 3, 3, 3], None),        # all within [1, 3]
    ]
    for t_, lens, exp in cases:
        args = [t_, t_.copy(), np.array(lens, np.int32)]
        r = I.run_graph_step(prog, args, st, mode="f32")
        if exp is None:
            assert r.status == I.OK
            continue
        assert r.status == I.ASSUMPTION_FAILED
        assert (r.failure.assumption_id, r.failure.index, r.failure.observed) == exp
        assert all(x.tobytes() == y.tobytes() for x, y in zip(r.state, st))
    st2 = [x.copy() for x in st]
    st2[prog.slot_index("tag")][:] = 0                 # TYPE_TAG (id 3) fails as well
    r = I.run_graph_step(prog, [tok, tok, np.array([3, 0, 2, 7], np.int32)], st2, mode="f32")
    assert (r.failure.assumption_id, r.failure.index, r.failure.observed) == (2, 1, 0)
    r = I.run_graph_step(prog, [tok, tok, np.array([3, 1, 2, 4], np.int32)], st2, mode="f32")
    assert (r.failure.assumption_id, r.failure.index, r.failure.observed) == (3, 0, 0)


# ----------------------------------------------------------------------------- imperative program
@pytest.mark.parametrize("tag", [1, 0])
def test_imperative_lm_equals_graph_and_torch(tag):
    """run_imperative_step's LM branch (Python control flow) against the dataflow interpreter of
    the generic graph (Switch/Merge, loop frames) AND against torch, with ragged lengths and
    `self.state` None (tag 0: zeros initial state) or a tensor (tag 1)."""
    B, W, V, E, H, L = 3, 5, 8, 3, 4, 2
    lens = [5, 1, 3]
    prog = pg.lstm_lm_program(V=V, E=E, H=H, L=L, B=B, T=W, lr=0.7, speculate="none")
    st, sid = _lm_state(prog, 31, 0.5, B, H, L)
    st[sid["tag"]] = np.array([tag], np.int32)
    args = _ragged(B, W, V, lens, seed=2)
    g = I.run_graph_step(prog, args, st, mode="f32")
    m = I.run_imperative_step(prog, args, st, mode="f32")
    assert g.status == m.status == I.OK
    assert abs(float(g.outputs[0]) - float(m.outputs[0])) < 1e-13
    for s, a, b in zip(prog.slots, g.state, m.state):
        np.testing.assert_allclose(np.asarray(a, np.float64), np.asarray(b, np.float64), atol=1e-13, err_msg=s.name)
    loss, hT, cT, grads = _torch_lm(prog, st, args, bf16=False)
    assert abs(float(m.outputs[0]) - loss) < 1e-12
    for l in range(L):
        np.testing.assert_allclose(m.state[sid[f"h{l}"]], hT[l], atol=1e-13)
        np.testing.assert_allclose(m.state[sid[f"c{l}"]], cT[l], atol=1e-13)
    for k, gt in grads.items():
        np.testing.assert_allclose(m.grads[sid[k]], gt, atol=1e-12, err_msg=k)
    assert int(m.state[sid["tag"]][0]) == 1


# ----------------------------------------------------------------------------- SGD commit
def test_sgd_commit_equals_torch_update():
    """One committed step: W' = fl32(W - lr * g) with g from torch autograd (P:154 inserted update,
    P:282 deferred effect); carried state := (h_T, c_T); tag := TENSOR. Data parallel: the update
    uses the mean of the two shards' gradients."""
    B, T, V, E, H, L, lr = 2, 3, 7, 3, 4, 2, 0.37
    prog = pg.lstm_lm_program(V=V, E=E, H=H, L=L, B=B, T=T, lr=lr)
    st32 = gen.uniform_params(prog, 41, 0.4)
    sid = {s.name: k for k, s in enumerate(prog.slots)}
    r0 = gen.rng(41)
    for l in range(L):
        st32[sid[f"h{l}"]] = r0.uniform(-0.5, 0.5, (B, H)).astype(np.float32)
        st32[sid[f"c{l}"]] = r0.uniform(-0.5, 0.5, (B, H)).astype(np.float32)
    args = _ragged(B, T, V, [T] * B, seed=6)
    r = I.run_graph_step(prog, args, st32, mode="f32")
    assert r.status == I.OK
    loss, hT, cT, grads = _torch_lm(prog, st32, args, bf16=False)
    for s in prog.slots:
        k = sid[s.name]
        if s.param:
            exp = (st32[k].astype(np.float64) - lr * grads[s.name]).astype(np.float32)
            # fl32 of values that agree to ~1e-15: equal, or one fp32 ulp apart on a rounding tie
            assert np.all(np.abs(r.state[k].astype(np.float64) - exp) <= np.spacing(np.abs(exp))), s.name
            assert r.state[k].dtype == np.float32
    for l in range(L):
        np.testing.assert_allclose(r.state[sid[f"h{l}"]], hT[l].astype(np.float32), atol=1e-7)
        np.testing.assert_allclose(r.state[sid[f"c{l}"]], cT[l].astype(np.float32), atol=1e-7)
    assert int(r.state[sid["tag"]][0]) == 1
    # data parallel: shard 1 = another batch, same parameters and carried state
    args2 = _ragged(B, T, V, [T] * B, seed=7)
    dp = I.run_dp_step(prog, [args, args2], [st32, [x.copy() for x in st32]], mode="f32")
    g2 = _torch_lm(prog, st32, args2, bf16=False)[3]
    for s in prog.slots:
        if s.param:
            k = sid[s.name]
            exp = (st32[k].astype(np.float64) - lr * 0.5 * (grads[s.name] + g2[s.name])).astype(np.float32)
            assert np.all(np.abs(dp[0].state[k].astype(np.float64) - exp) <= np.spacing(np.abs(exp))), s.name
            assert dp[0].state[k].tobytes() == dp[1].state[k].tobytes()


# ----------------------------------------------------------------------------- bf16 placement
@pytest.mark.parametrize("lens", [None, [5, 2, 4]])
def test_bf16_rounding_points_lm_match_torch(lens):
    """bf16 mode against torch fp64 with the operands rounded at R1 (weight copies), R2 (every h /
    x feeding a GEMM) and R3 (dz, dy before dgrad / wgrad) by torch's own conversions; R4 (bias
    gradients = sums of rounded dz / dy rows) is what autograd gives for z = x W^T + b with the
    gradient of z rounded."""
    B, W, V, E, H, L = 3, 5, 10, 4, 4, 2
    spec = "unroll" if lens is None else "while"
    prog = pg.lstm_lm_program(V=V, E=E, H=H, L=L, B=B, T=W, lr=0.0, speculate=spec)
    st, sid = _lm_state(prog, 51, 0.7, B, H, L)
    args = _ragged(B, W, V, lens or [W] * B, seed=9)
    r = I.run_graph_step(prog, args, st, mode="bf16")
    assert r.status == I.OK
    loss, hT, cT, grads = _torch_lm(prog, st, args, bf16=True)
    assert abs(float(r.outputs[0]) - loss) < 1e-12
    for l in range(L):
        np.testing.assert_allclose(r.state[sid[f"h{l}"]], hT[l], atol=1e-12)
    for k, gt in grads.items():
        np.testing.assert_allclose(r.grads[sid[k]], gt, atol=1e-12, rtol=1e-12, err_msg=k)
    # and the placement matters: the unrounded (f32-mode) gradients differ at the bf16 scale
    f32 = I.run_graph_step(prog, args, st, mode="f32")
    assert max(np.abs(f32.grads[sid[k]] - gt).max() for k, gt in grads.items()) > 1e-5


def _torch_tree(prog, st, forest, bf16):
    """TreeLSTM by torch recursion + autograd (readings Q5/Q6), rounding points as above."""
    sid = {s.name: k for k, s in enumerate(prog.slots)}
    R = _RoundFwd.apply if bf16 else (lambda x: x)
    G = _RoundBwd.apply if bf16 else (lambda x: x)
    kind, left, right, word, off, label = (np.asarray(a, np.int64) for a in forest)
    H = prog.meta["H"]
    P = {k: torch.tensor(np.asarray(st[sid[k]], np.float64), requires_grad=True)
         for k in ("W_leaf", "U", "b", "W_c", "b_c")}
    Emb = torch.tensor(np.asarray(st[sid["E"]], np.float64))
    b = P["b"]
    bi, bf_, bo, bu = b[:H], b[H:2 * H], b[2 * H:3 * H], b[3 * H:]

    def node(n):
        if kind[n] == 0:
            x = R(Emb[int(word[n])])[None, :]
            z = G(x @ R(P["W_leaf"]).T + torch.cat([bi, bo, bu]))
            i, o, u = torch.sigmoid(z[:, :H]), torch.sigmoid(z[:, H:2 * H]), torch.tanh(z[:, 2 * H:])
            c = i * u
            return o * torch.tanh(c), c
        hl, cl = node(int(left[n]))
        hr, cr = node(int(right[n]))
        z = G(R(torch.cat([hl, hr], 1)) @ R(P["U"]).T + torch.cat([bi, bf_, bf_, bo, bu]))
        i, fl, fr = torch.sigmoid(z[:, :H]), torch.sigmoid(z[:, H:2 * H]), torch.sigmoid(z[:, 2 * H:3 * H])
        o, u = torch.sigmoid(z[:, 3 * H:4 * H]), torch.tanh(z[:, 4 * H:])
        c = i * u + fl * cl + fr * cr
        return o * torch.tanh(c), c

    roots = torch.cat([node(int(off[t + 1]) - 1)[0] for t in range(len(off) - 1)], 0)
    logits = G(R(roots) @ R(P["W_c"]).T + P["b_c"])
    loss = torch.nn.functional.cross_entropy(logits, torch.tensor(label))
    loss.backward()
    return float(loss.detach()), {k: v.grad.numpy().copy() for k, v in P.items()}


@pytest.mark.parametrize("bf16", [False, True])
def test_tree_matches_torch_recursion(bf16):
    """TreeLSTM loss and gradients against a torch recursion with autograd (f32 and bf16 modes)."""
    V, E, H = 12, 3, 4
    forest = gen.sst_forest(gen.SEED_C3, 1, 4, V, max_leaves=7)
    prog = pg.treelstm_program(V=V, E=E, H=H, C=2, B=4, lr=0.0)
    st = [np.asarray(s, np.float64) for s in gen.uniform_params(prog, 9, 0.6)]
    sid = {s.name: k for k, s in enumerate(prog.slots)}
    r = I.run_graph_step(prog, list(forest), st, mode="bf16" if bf16 else "f32")
    assert r.status == I.OK
    loss, grads = _torch_tree(prog, st, forest, bf16)
    assert abs(float(r.outputs[0]) - loss) < 1e-12
    for k, gt in grads.items():
        np.testing.assert_allclose(r.grads[sid[k]], gt, atol=1e-12, rtol=1e-12, err_msg=k)


# ----------------------------------------------------------------------------- training switch
def test_training_switch_eval_step_and_value_eq_guard():
    """`if training: update` (P:312 train / evaluate branch). Evaluate step (training = 0): loss
    and carried state equal torch's forward, no parameter changes — through the generic graph's
    Switch (dead arm: no SGD effect) and the imperative program alike. Speculated graph (VALUE_EQ
    id 8): training = 0 or 2 fails with {8, index 0, observed}, no commit."""
    B, T, V, E, H, L = 2, 3, 7, 3, 4, 2
    gen_prog = pg.lstm_lm_program(V=V, E=E, H=H, L=L, B=B, T=T, lr=0.5, training_flag=True, speculate="none")
    st, sid = _lm_state(gen_prog, 61, 0.5, B, H, L)
    st = [np.asarray(x, np.float32) if np.asarray(x).dtype.kind == "f" else x for x in st]
    a3 = _ragged(B, T, V, [T] * B, seed=4)
    ev = a3 + [np.array([0], np.int32)]
    g = I.run_graph_step(gen_prog, ev, st, mode="f32")
    m = I.run_imperative_step(gen_prog, ev, st, mode="f32")
    assert g.status == m.status == I.OK
    loss, hT, cT, _ = _torch_lm(gen_prog, st, a3, bf16=False)
    for r in (g, m):
        assert abs(float(r.outputs[0]) - loss) < 1e-12
        for s in gen_prog.slots:
            if s.param:
                assert r.state[sid[s.name]].tobytes() == st[sid[s.name]].tobytes(), s.name
        for l in range(L):
            np.testing.assert_allclose(r.state[sid[f"h{l}"]], hT[l].astype(np.float32), atol=1e-7)
            np.testing.assert_allclose(r.state[sid[f"c{l}"]], cT[l].astype(np.float32), atol=1e-7)
    tr = a3 + [np.array([1], np.int32)]        # training step: the update of the plain program
    plain = pg.lstm_lm_program(V=V, E=E, H=H, L=L, B=B, T=T, lr=0.5, speculate="none")
    g1, p1 = I.run_graph_step(gen_prog, tr, st, mode="f32"), I.run_graph_step(plain, a3, st, mode="f32")
    assert all(x.tobytes() == y.tobytes() for x, y in zip(g1.state, p1.state))
    spec = pg.lstm_lm_program(V=V, E=E, H=H, L=L, B=B, T=T, lr=0.5, training_flag=True)
    assert [(a.id, a.kind, a.target, a.value) for a in spec.assumptions if a.kind == "VALUE_EQ"] == [(8, "VALUE_EQ", 3, 1)]
    for flag in (0, 2):
        r = I.run_graph_step(spec, a3 + [np.array([flag], np.int32)], st, mode="f32")
        assert r.status == I.ASSUMPTION_FAILED
        assert (r.failure.assumption_id, r.failure.index, r.failure.observed) == (8, 0, flag)
        assert all(x.tobytes() == y.tobytes() for x, y in zip(r.state, st))
    assert I.run_graph_step(spec, tr, st, mode="f32").status == I.OK


def test_branch_arm_speculation():
    """BRANCH_ARM (the branch is speculated, the untaken arm dropped, the branch
    asserted): the true-arm assumption holds for every non-zero predicate — a speculated graph step
    with training = 1 or 7 equals the plain program's training step bit for bit — and fails only
    on 0, reporting {8, index 0, observed 0}; the false-arm form holds only for 0."""
    B, T, V, E, H, L = 2, 3, 7, 3, 4, 2
    spec = pg.lstm_lm_program(V=V, E=E, H=H, L=L, B=B, T=T, lr=0.5, training_flag=True, flag_speculation="branch")
    assert [(a.id, a.kind, a.target, a.value) for a in spec.assumptions if a.kind == "BRANCH_ARM"] == \
        [(8, "BRANCH_ARM", 3, 1)]
    plain = pg.lstm_lm_program(V=V, E=E, H=H, L=L, B=B, T=T, lr=0.5, speculate="none")
    st, _ = _lm_state(plain, 61, 0.5, B, H, L)
    st = [np.asarray(x, np.float32) if np.asarray(x).dtype.kind == "f" else x for x in st]
    a3 = _ragged(B, T, V, [T] * B, seed=4)
    ref = I.run_graph_step(plain, a3, st, mode="f32")
    for flag in (1, 7):
        r = I.run_graph_step(spec, a3 + [np.array([flag], np.int32)], st, mode="f32")
        assert r.status == I.OK
        assert all(x.tobytes() == y.tobytes() for x, y in zip(r.state, ref.state))
    r = I.run_graph_step(spec, a3 + [np.array([0], np.int32)], st, mode="f32")
    assert r.status == I.ASSUMPTION_FAILED
    assert (r.failure.assumption_id, r.failure.index, r.failure.observed) == (8, 0, 0)
    assert all(x.tobytes() == y.tobytes() for x, y in zip(r.state, st))
    false_arm = pg.Program("t", [], [pg.Assumption(4, "BRANCH_ARM", 1, 0, value=0)], [], [], 0, 0.0)
    assert I.check_runtime(false_arm, [np.array([0], np.int32)], []) is None
    f = I.check_runtime(false_arm, [np.array([5], np.int32)], [])
    assert (f.assumption_id, f.index, f.observed) == (4, 0, 5)
