"""Pins of the oracle's gradient clipping (janus_build_opts.clip_norm; reading R15: the global L2
norm of the step's rank-averaged gradient clipped to c, as Zaremba et al. [51] do for the LM of
P:312 — SURVEY Q2: "clip off by default (5.0 optional)").

* c above the gradient norm: bit-identical to no clipping (graph step and imperative step).
* Against torch: the same LM step in torch autograd, `torch.nn.utils.clip_grad_norm_` over every
  parameter, then SGD — the oracle's new parameters agree (torch's 1e-6 guard in its coefficient
  is far below the tolerance).
* Data parallel: the norm is that of the rank-AVERAGED gradient (reading Q13), checked from the
  averaged gradients the oracle reports; the tree programs follow the same rule.
CPU only."""
import numpy as np
import pytest
import torch

from oracle import interp as I
from workloads import gen, programs as pg

from tests.test_oracle_pins_r2 import _lm_state, _ragged, _torch_lm


@pytest.fixture(autouse=True)
def _fp64_default():
    old = torch.get_default_dtype()
    torch.set_default_dtype(torch.float64)
    yield
    torch.set_default_dtype(old)


def _lm(clip):
    B, T, V, E, H, L = 3, 4, 11, 5, 6, 2
    prog = pg.lstm_lm_program(V=V, E=E, H=H, L=L, B=B, T=T, lr=0.5, speculate="none", clip_norm=clip)
    st, sid = _lm_state(prog, 17, 0.5, B, H, L)
    st = [np.asarray(x, np.float32) if np.asarray(x).dtype.kind == "f" else x for x in st]
    return prog, st, sid, _ragged(B, T, V, [4, 2, 3], seed=9)


def test_clip_above_the_norm_is_no_clip():
    prog0, st, _, args = _lm(0.0)
    prog1, _, _, _ = _lm(1e9)
    for run in (I.run_graph_step, I.run_imperative_step):
        a, b = run(prog0, args, st, mode="f32"), run(prog1, args, st, mode="f32")
        assert a.status == b.status == I.OK
        assert all(x.tobytes() == y.tobytes() for x, y in zip(a.state, b.state))


@pytest.mark.parametrize("clip", [0.05, 0.3])
def test_clip_matches_torch_clip_grad_norm(clip):
    prog, st, sid, args = _lm(clip)
    _, _, _, grads = _torch_lm(prog, st, args, bf16=False)
    params = []
    for k, g in grads.items():
        p = torch.tensor(np.asarray(st[sid[k]], np.float64), requires_grad=True)
        p.grad = torch.tensor(g)
        params.append((k, p))
    total = float(torch.nn.utils.clip_grad_norm_([p for _, p in params], clip))
    assert total > clip                                 # the case actually clips
    for run in (I.run_graph_step, I.run_imperative_step):
        r = run(prog, args, st, mode="f32")
        assert r.status == I.OK
        for k, p in params:
            ref = np.asarray(st[sid[k]], np.float64) - prog.lr * p.grad.numpy()
            np.testing.assert_allclose(np.asarray(r.state[sid[k]], np.float64), ref, rtol=0,
                                       atol=1e-6 * max(1.0, np.abs(ref).max()), err_msg=k)


def test_clip_uses_the_rank_averaged_gradient():
    prog, st, sid, args = _lm(0.02)
    B = 3
    shard2 = _ragged(B, 4, 11, [1, 4, 4], seed=31)
    res = I.run_dp_step(prog, [args, shard2], [st, st], mode="f32")
    assert all(r.status == I.OK for r in res)
    avg = res[0].grads                                  # slot -> rank-averaged gradient
    norm = np.sqrt(sum(float(np.sum(np.asarray(g, np.float64) ** 2)) for g in avg.values()))
    assert norm > 0.02
    for k, g in avg.items():
        ref = np.asarray(st[k], np.float64) - prog.lr * (0.02 / norm) * np.asarray(g, np.float64)
        for r in res:
            np.testing.assert_allclose(np.asarray(r.state[k], np.float64), ref, rtol=0,
                                       atol=1e-6 * max(1.0, np.abs(ref).max()))


@pytest.mark.parametrize("rnn", [False, True])
def test_clip_tree_programs(rnn):
    V, B = 40, 4
    mk = (lambda c: pg.treernn_program(V=V, H=8, C=2, B=B, lr=0.4, clip_norm=c)) if rnn else \
        (lambda c: pg.treelstm_program(V=V, E=6, H=8, C=2, B=B, lr=0.4, clip_norm=c))
    p0, p1 = mk(0.0), mk(0.01)
    st = gen.uniform_params(p0, 3, 0.3)
    args = gen.sst_forest(gen.SEED_C3, 0, B, V, max_leaves=8)
    a, b = I.run_graph_step(p0, args, st, mode="f32"), I.run_graph_step(p1, args, st, mode="f32")
    assert a.status == b.status == I.OK
    norm = np.sqrt(sum(float(np.sum(np.asarray(g, np.float64) ** 2)) for g in a.grads.values()))
    assert norm > 0.01
    for k, g in a.grads.items():
        ref = np.asarray(st[k], np.float64) - p1.lr * (0.01 / norm) * np.asarray(g, np.float64)
        np.testing.assert_allclose(np.asarray(b.state[k], np.float64), ref, rtol=0,
                                   atol=1e-6 * max(1.0, np.abs(ref).max()))
    m = I.run_imperative_step(p1, args, st, mode="f32")
    assert all(np.allclose(x, y, atol=1e-6) for x, y in zip(m.state, b.state))
