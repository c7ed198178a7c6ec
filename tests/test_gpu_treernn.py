"""TreeRNN (NEXT-4; Table 2 TreeRNN on SST) through the C ABI on the GPU vs the oracle: the
same device level schedule as the TreeLSTM (bit-exact), one tanh gate per unit on tensor cores,
leaves = word vectors; the imperative executor on the same program; guard outcomes exact."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import interp as I  # noqa: E402
from workloads import gen, programs as pg  # noqa: E402
from tests.helpers import assert_state_parity, rel_err, to_dev, to_host  # noqa: E402
from tests.test_gpu_tree import _check  # noqa: E402


def J():
    from paper_1812_01329_b200 import janus
    return janus


def test_treernn_small_forests():
    V, B = 50, 6
    prog = pg.treernn_program(V=V, H=32, C=2, B=B, lr=0.3)
    _check(prog, [gen.sst_forest(gen.SEED_C3, k, B, V, max_leaves=12) for k in range(3)], scale=0.4)


def test_treernn_ragged_hidden_chains_and_one_leaf_trees():
    V, B = 40, 9
    prog = pg.treernn_program(V=V, H=84, C=2, B=B, lr=0.3)  # H not a multiple of 80 or 64
    forests = [gen.sst_forest(gen.SEED_C3, 3, B, V, max_leaves=20, chain=True),
               gen.sst_forest(gen.SEED_C3, 4, B, V, max_leaves=1),
               gen.sst_forest(gen.SEED_C3, 5, B, V, max_leaves=40)]
    _check(prog, forests, scale=0.3)


def test_treernn_c3_full_size():
    """TreeRNN at the C3 shape: B=25, H=E=300, V=20000."""
    V, B = 20000, 25
    prog = pg.treernn_program(V=V, H=300, C=2, B=B, lr=0.05)
    _check(prog, [gen.sst_forest(gen.SEED_C3, 0, B, V), gen.sst_forest(gen.SEED_C3, 1, B, V)], scale=0.05)


def test_treernn_guard_failure_and_imperative():
    V, B = 50, 4
    prog = pg.treernn_program(V=V, H=32, C=2, B=B, lr=0.2)
    kind, left, right, word, off, label = gen.sst_forest(gen.SEED_C3, 7, B, V, max_leaves=8)
    bad = word.copy(); bad[int(np.argmax(kind == 0))] = V + 3
    _check(prog, [(kind, left, right, bad, off, label)], check_sched=False)
    janus = J()
    g = janus.Graph(prog)
    state = gen.uniform_params(prog, 3, 0.3)
    args = [kind, left, right, word, off, label]
    dev = to_dev(state)
    loss = torch.zeros(1, device="cuda")
    st = g.run_imperative(to_dev(args), dev, g.new_workspace(), outs=[loss])
    ora = I.run_imperative_step(prog, args, state, mode="bf16")
    assert st == I.OK == ora.status
    assert rel_err(loss.item(), ora.outputs[0]) <= 2e-2
    assert_state_parity(prog, state, to_host(dev), ora.state, 2e-2, what="treernn imperative")
