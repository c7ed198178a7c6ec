"""Pins of the oracle's dropout LM (NEXT-4: the Zaremba et al. [51] model of P:312 — PTB medium:
2 x 650, dropout 0.5 on the non-recurrent connections) and its counter-based generator.

* Philox4x32-10 against the known-answer vectors published with the generator (Salmon, Moraes,
  Dror, Shaw, "Parallel random numbers: as easy as 1, 2, 3", SC'11; Random123 kat_vectors).
* The whole step against the same model written directly in torch (fp64 autograd) with the same
  masks — the masks come from the generator pinned above; torch checks WHERE they apply (every
  non-recurrent connection, inverted scaling, the backward) and everything around them.
* p -> 0 reduces to the plain LM; the keep rate of p = 0.5 is 1/2 within binomial error.
CPU only."""
import numpy as np
import pytest
import torch

from oracle import interp as I
from oracle import numerics as nm
from workloads import gen, programs as pg

from tests.test_oracle_pins_r2 import _RoundBwd, _RoundFwd, _lm_state


@pytest.fixture(autouse=True)
def _fp64_default():
    old = torch.get_default_dtype()
    torch.set_default_dtype(torch.float64)
    yield
    torch.set_default_dtype(old)


# (counter, key, output) — Random123 kat_vectors, philox4x32_10
KAT = [((0x00000000, 0x00000000, 0x00000000, 0x00000000), (0x00000000, 0x00000000),
        (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
       ((0xffffffff, 0xffffffff, 0xffffffff, 0xffffffff), (0xffffffff, 0xffffffff),
        (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
       ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0),
        (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1))]


@pytest.mark.parametrize("ctr,key,out", KAT)
def test_philox4x32_10_known_answers(ctr, key, out):
    got = nm.philox4x32_10(np.array(ctr, np.uint64), np.array(key, np.uint64))
    assert tuple(int(x) for x in got) == out


def _torch_lm_dropout(prog, st, args, bf16):
    """The dropout LM step in torch: x_t = D0(E[tok_t]); for l: h_l = cell(x, h_l); x = D_{l+1}(h_l);
    logits = x W_dec^T + b_dec. D_s(x) = x * mask_s / (1 - p), masks from the pinned generator."""
    m = prog.meta
    sid = {s.name: k for k, s in enumerate(prog.slots)}
    L, H, p = m["L"], m["H"], m["dropout"]
    tok, tgt, lens = (np.asarray(a, np.int64) for a in args[:3])
    key = np.asarray(args[m["key_arg"]])
    B = tok.shape[0]
    T = int(lens.max())
    R = _RoundFwd.apply if bf16 else (lambda x: x)
    G = _RoundBwd.apply if bf16 else (lambda x: x)
    names = ["E", "W_dec", "b_dec"] + [f"{q}{l}" for l in range(L) for q in ("W_ih", "W_hh", "b")]
    P = {k: torch.tensor(np.asarray(st[sid[k]], np.float64), requires_grad=True) for k in names}
    h = [torch.tensor(np.asarray(st[sid[f"h{l}"]], np.float64)) for l in range(L)]
    c = [torch.tensor(np.asarray(st[sid[f"c{l}"]], np.float64)) for l in range(L)]

    def D(x, site, t):
        mk = nm.dropout_mask(key, site, t * B + np.arange(B), x.shape[1], p) / (1.0 - p)
        return x * torch.tensor(mk)

    outs = []
    for t in range(T):
        x = D(R(P["E"])[torch.tensor(tok[:, t])], 0, t)
        v = torch.tensor((t < lens).astype(np.float64))[:, None]
        for l in range(L):
            z = G(R(x) @ R(P[f"W_ih{l}"]).T + R(h[l]) @ R(P[f"W_hh{l}"]).T + P[f"b{l}"])
            i, f = torch.sigmoid(z[:, :H]), torch.sigmoid(z[:, H:2 * H])
            g, o = torch.tanh(z[:, 2 * H:3 * H]), torch.sigmoid(z[:, 3 * H:])
            c2 = f * c[l] + i * g
            h2 = o * torch.tanh(c2)
            h[l] = v * h2 + (1 - v) * h[l]
            c[l] = v * c2 + (1 - v) * c[l]
            x = D(h[l], l + 1, t)
        outs.append(x)
    logits = G(R(torch.cat(outs, 0)) @ R(P["W_dec"]).T + P["b_dec"])
    mask = torch.tensor((np.arange(T)[:, None] < lens[None, :]).reshape(-1))
    per = torch.nn.functional.cross_entropy(logits, torch.tensor(tgt[:, :T].T.reshape(-1)), reduction="none")
    loss = (per * mask).sum() / max(1, int(mask.sum()))
    loss.backward()
    return float(loss.detach()), [x.detach().numpy() for x in h], {k: v.grad.numpy() for k, v in P.items()}


@pytest.mark.parametrize("mode", ["f32", "bf16"])
def test_dropout_lm_step_matches_torch(mode):
    B, T, V, H, L = 5, 6, 23, 7, 2
    prog = pg.lstm_lm_program(V=V, E=9, H=H, L=L, B=B, T=T, lr=0.3, dropout=0.5, speculate="while")
    st, sid = _lm_state(prog, 4, 0.4, B, H, L)
    r = gen.rng(3)
    lens = np.array([6, 4, 6, 1, 5], np.int32)   # ragged rows (masked steps carry h, c)
    args = [r.integers(0, V, (B, T)).astype(np.int32), r.integers(0, V, (B, T)).astype(np.int32), lens,
            np.array([0x1234, 0xBEEF], np.int32)]
    loss, h, grads = _torch_lm_dropout(prog, st, args, mode == "bf16")
    for run in (I.run_imperative_step, I.run_graph_step):
        res = run(prog, args, st, mode=mode)
        assert res.status == I.OK
        assert abs(float(res.outputs[0]) - loss) <= 1e-12
        for k, s in enumerate(prog.slots):
            if s.param:
                ref = np.asarray(st[k], np.float64) - prog.lr * grads[s.name]
                np.testing.assert_allclose(np.asarray(res.state[k], np.float64), ref, rtol=0,
                                           atol=2e-7 * max(1.0, np.abs(ref).max()), err_msg=s.name)
        for l in range(L):
            np.testing.assert_allclose(np.asarray(res.state[sid[f"h{l}"]], np.float64), h[l], atol=2e-7)


def test_dropout_p_to_zero_is_the_plain_lm():
    B, T, V = 3, 4, 17
    plain = pg.lstm_lm_program(V=V, E=6, H=5, L=2, B=B, T=T, lr=0.3)
    drop = pg.lstm_lm_program(V=V, E=6, H=5, L=2, B=B, T=T, lr=0.3, dropout=1e-12)
    st = gen.uniform_params(plain, 2, 0.3)
    r = gen.rng(9)
    args = [r.integers(0, V, (B, T)).astype(np.int32), r.integers(0, V, (B, T)).astype(np.int32),
            np.full(B, T, np.int32)]
    a = I.run_graph_step(plain, args, st, mode="f32")
    b = I.run_graph_step(drop, args + [np.array([5, 6], np.int32)], st, mode="f32")
    assert abs(float(a.outputs[0]) - float(b.outputs[0])) <= 1e-9
    for x, y in zip(a.state, b.state):
        np.testing.assert_allclose(np.asarray(x, np.float64), np.asarray(y, np.float64), atol=1e-9)


def test_dropout_keep_rate_and_site_independence():
    key = np.array([2024, 7], np.uint32)
    m0 = nm.dropout_mask(key, 0, np.arange(64), 650, 0.5)
    m1 = nm.dropout_mask(key, 1, np.arange(64), 650, 0.5)
    n = m0.size
    assert abs(m0.mean() - 0.5) <= 4 * np.sqrt(0.25 / n)           # binomial, 4 sigma
    assert abs((m0 == m1).mean() - 0.5) <= 4 * np.sqrt(0.25 / n)   # sites draw independent masks
    m2 = nm.dropout_mask(key, 0, np.arange(64), 650, 0.25)
    assert abs(m2.mean() - 0.75) <= 4 * np.sqrt(0.1875 / n)
    assert ((m2 >= m0)).all()                                      # same words, lower threshold
