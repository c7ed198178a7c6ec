"""Pins of the oracle's TreeRNN (NEXT-4; Table 2 TreeRNN on SST; Socher et al. [37]):
h(leaf) = word vector, h(node) = tanh([h_l; h_r] W^T + b), root classifier + mean xent. Expected
values come from torch autograd (a library routine, fp64, written recursively over the trees), a
closed form and central finite differences — never from the oracle itself. CPU only."""
import numpy as np
import pytest
import torch

from oracle import interp as I
from workloads import gen, programs as pg


@pytest.fixture(autouse=True)
def _fp64_default():
    old = torch.get_default_dtype()
    torch.set_default_dtype(torch.float64)
    yield
    torch.set_default_dtype(old)


def _rbt(x):
    return x.to(torch.float32).to(torch.bfloat16).to(torch.float64)


class _RoundFwd(torch.autograd.Function):
    """R1/R2: a GEMM operand copy rb(x); the gradient passes through (the copy is a cast)."""
    @staticmethod
    def forward(ctx, x):
        return _rbt(x)

    @staticmethod
    def backward(ctx, g):
        return g


class _RoundBwd(torch.autograd.Function):
    """R3: identity forward; the gradient of the affine op's output is rounded."""
    @staticmethod
    def forward(ctx, x):
        return x.clone()

    @staticmethod
    def backward(ctx, g):
        return _rbt(g)


def _torch_step(prog, args, state, bf16):
    """Loss and gradients of every parameter slot, recursion in torch (fp64)."""
    sid = {s.name: k for k, s in enumerate(prog.slots)}
    kind, left, right, word, off, label = (np.asarray(a, np.int64) for a in args)
    P = {k: torch.tensor(np.asarray(state[sid[k]], np.float64), requires_grad=True) for k in ("W", "b", "W_c", "b_c")}
    E = torch.tensor(np.asarray(state[sid["E"]], np.float64))
    R = _RoundFwd.apply if bf16 else (lambda x: x)
    D = _RoundBwd.apply if bf16 else (lambda x: x)

    def node(n):
        if kind[n] == 0:
            return R(E[int(word[n])][None, :])      # the leaf IS its (rounded) word vector
        hh = torch.cat([node(int(left[n])), node(int(right[n]))], dim=1)
        z = D(R(hh) @ R(P["W"]).T + P["b"])
        return torch.tanh(z)

    roots = torch.cat([node(int(off[i + 1]) - 1) for i in range(len(off) - 1)], dim=0)
    logits = D(R(roots) @ R(P["W_c"]).T + P["b_c"])
    loss = torch.nn.functional.cross_entropy(logits, torch.tensor(label))
    loss.backward()
    return float(loss.detach()), {k: v.grad.numpy() for k, v in P.items()}


def _case(B=5, V=37, H=6, seed=2, max_leaves=7, lr=0.4):
    prog = pg.treernn_program(V=V, H=H, C=2, B=B, lr=lr)
    state = gen.uniform_params(prog, seed, 0.5)
    args = list(gen.sst_forest(gen.SEED_C3, seed, B, V, max_leaves=max_leaves))
    return prog, state, args


@pytest.mark.parametrize("mode", ["f32", "bf16"])
def test_treernn_step_matches_torch_autograd(mode):
    prog, state, args = _case()
    loss, grads = _torch_step(prog, args, state, mode == "bf16")
    for run in (I.run_graph_step, I.run_imperative_step):
        r = run(prog, args, state, mode=mode)
        assert r.status == I.OK
        assert abs(float(r.outputs[0]) - loss) <= 1e-12
        for k, s in enumerate(prog.slots):
            if s.param:   # SGD commit: new = old - lr * grad
                ref = np.asarray(state[k], np.float64) - prog.lr * grads[s.name]
                np.testing.assert_allclose(np.asarray(r.state[k], np.float64), ref, rtol=0,
                                           atol=2e-7 * max(1.0, np.abs(ref).max()))
            else:
                assert np.asarray(r.state[k]).tobytes() == np.asarray(state[k]).tobytes()


def test_treernn_closed_form_zero_weights():
    """W = 0, b = beta: every internal node is tanh(beta) whatever its children; a one-leaf tree's
    root is its word vector. W_c = 0: logits = b_c for every tree, loss = xent(b_c, label)."""
    B, V, H = 4, 20, 5
    prog = pg.treernn_program(V=V, H=H, C=2, B=B, lr=0.0)
    sid = {s.name: k for k, s in enumerate(prog.slots)}
    st = [np.asarray(x, np.float64).copy() for x in gen.uniform_params(prog, 1, 0.5)]
    st[sid["W"]][:] = 0.0
    beta = np.linspace(-0.7, 0.9, H)
    st[sid["b"]][:] = beta
    st[sid["W_c"]][:] = 0.0
    st[sid["b_c"]][:] = [0.3, -0.2]
    args = list(gen.sst_forest(gen.SEED_C3, 4, B, V, max_leaves=6))
    label = np.asarray(args[5])
    lse = np.log(np.exp(0.3) + np.exp(-0.2))
    expect = np.mean([lse - (0.3 if y == 0 else -0.2) for y in label])
    r = I.run_dp_step(prog, [args], [st], mode="f32")[0]
    assert abs(float(r.outputs[0]) - expect) <= 1e-14
    # the root features reach W_c's gradient: dW_c = mean over trees of (p - onehot) h_root^T
    p = np.exp([0.3, -0.2]) / np.exp([0.3, -0.2]).sum()
    kind, off, word = np.asarray(args[0]), np.asarray(args[4]), np.asarray(args[3])
    roots = []
    for i in range(B):
        rt = off[i + 1] - 1
        roots.append(st[sid["E"]][word[rt]] if kind[rt] == 0 else np.tanh(beta))
    dWc = sum(np.outer(p - np.eye(2)[y], h) for y, h in zip(label, roots)) / B
    np.testing.assert_allclose(r.grads[sid["W_c"]], dWc, atol=1e-14)


def test_treernn_finite_differences():
    prog, state, args = _case(B=3, V=17, H=4, max_leaves=5)
    sid = {s.name: k for k, s in enumerate(prog.slots)}
    g = I.run_dp_step(prog, [args], [state], mode="f32")[0].grads
    eps = 1e-6
    rng = np.random.default_rng(0)
    for name in ("W", "b", "W_c"):
        k = sid[name]
        for flat in rng.choice(np.asarray(state[k]).size, 4, replace=False):
            plus = [np.asarray(x, np.float64).copy() for x in state]
            minus = [np.asarray(x, np.float64).copy() for x in state]
            plus[k].reshape(-1)[flat] += eps
            minus[k].reshape(-1)[flat] -= eps
            lp = float(I.run_graph_step(prog, args, plus, mode="f32").outputs[0])
            lm = float(I.run_graph_step(prog, args, minus, mode="f32").outputs[0])
            assert abs((lp - lm) / (2 * eps) - g[k].reshape(-1)[flat]) <= 1e-7, (name, flat)
