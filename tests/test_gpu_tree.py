"""TreeLSTM (C3) through the C ABI on the GPU vs the oracle: device level schedule bit-exact,
level-batched tensor-core numerics within the bf16 tolerance, forest AssertOp outcomes exact."""
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


def _check(prog, forests, seed=3, scale=0.3, tol=2e-2, check_sched=True, **ablation):
    janus = J()
    g = janus.Graph(prog, **ablation)
    assert g.device_path, g.build_message
    ws = g.new_workspace()
    state = gen.uniform_params(prog, seed, scale)
    for f in forests:
        args = list(f)
        dev = to_dev(state)
        loss = torch.zeros(1, device="cuda")
        st, fail = g.run(to_dev(args), dev, ws, outs=[loss])
        ora = I.run_graph_step(prog, args, state, mode="bf16")
        assert st == ora.status, (st, fail, ora.failure)
        got = to_host(dev)
        if st != I.OK:
            assert (fail["assumption_id"], fail["index"], fail["observed"]) == \
                (ora.failure.assumption_id, ora.failure.index, ora.failure.observed)
            assert all(a.tobytes() == b.tobytes() for a, b in zip(got, state))
            continue
        assert rel_err(loss.item(), ora.outputs[0]) <= tol
        assert_state_parity(prog, state, got, ora.state, tol, what="tree")
        if check_sched:
            kind, left, right, word, off = f[:5]
            sch = I.tree_schedule(kind, left, right, off)
            N = len(kind)
            meta = janus.dev_workspace_region(g, ws, "tree.meta")
            L = len(sch["level_offset"]) - 1
            assert meta[0] == L and meta[1] == N
            np.testing.assert_array_equal(janus.dev_workspace_region(g, ws, "tree.height")[:N], sch["height"])
            np.testing.assert_array_equal(janus.dev_workspace_region(g, ws, "tree.order")[:N], sch["order"])
            np.testing.assert_array_equal(janus.dev_workspace_region(g, ws, "tree.lvl_off")[:L + 1],
                                          sch["level_offset"])
            ps = janus.dev_workspace_region(g, ws, "tree.pslot")[:N]
            ref = np.where(sch["parent_slot"][:, 0] >= 0, sch["parent_slot"][:, 0] * 2 + sch["parent_slot"][:, 1], -1)
            np.testing.assert_array_equal(ps, ref)
        state = ora.state
    return g


def test_tree_small_forests():
    V, B = 50, 6
    prog = pg.treelstm_program(V=V, E=24, H=32, C=2, B=B, lr=0.2)
    forests = [gen.sst_forest(gen.SEED_C3, k, B, V, max_leaves=12) for k in range(3)]
    _check(prog, forests)


def test_tree_ragged_units_and_chains():
    """H=100 (last 16-unit tile has 4 units), E=70, right-branching chains up to 64 leaves (height 63)."""
    V, B = 120, 5
    prog = pg.treelstm_program(V=V, E=70, H=100, C=2, B=B, lr=0.2)
    forests = [gen.sst_forest(gen.SEED_C3, 7, B, V, max_leaves=64, chain=True),
               gen.sst_forest(gen.SEED_C3, 8, B, V, max_leaves=64)]
    _check(prog, forests, scale=0.2)


def test_tree_hidden_not_multiple_of_four_and_many_trees():
    """H=30 (H % 4 != 0: the epilogues' scalar paths), odd E, B=40 trees (five root-classifier
    blocks; the level schedule spans several 128-row tiles at the leaves)."""
    V, B = 77, 40
    prog = pg.treelstm_program(V=V, E=21, H=30, C=2, B=B, lr=0.2)
    forests = [gen.sst_forest(gen.SEED_C3, 11, B, V, max_leaves=20),
               gen.sst_forest(gen.SEED_C3, 12, B, V, max_leaves=20, chain=True)]
    _check(prog, forests, scale=0.2)


def test_tree_large_forest_small_cells():
    """N > 2048 nodes (the schedule's per-tree walk instead of the parallel relaxation; several
    128-row tiles per level; 17 root-classifier blocks) at a small H so the oracle stays fast."""
    V, B = 50, 130
    prog = pg.treelstm_program(V=V, E=8, H=16, C=2, B=B, lr=0.2)
    f = gen.sst_forest(gen.SEED_C3, 21, B, V, max_leaves=40)
    assert len(f[0]) > 2048
    _check(prog, [f], scale=0.3)


@pytest.mark.parametrize("H", [320, 800])
def test_tree_wide_hidden_kernel_variants(H):
    """H=320: 5H > 1536, so the backward streams U^T through its ring instead of keeping it
    resident; H=800: the forward's 4-deep ring (the 6-deep one no longer fits beside the
    epilogue staging)."""
    V, B = 40, 3
    prog = pg.treelstm_program(V=V, E=24, H=H, C=2, B=B, lr=0.2)
    _check(prog, [gen.sst_forest(gen.SEED_C3, 5, B, V, max_leaves=6)], scale=0.1)


def test_tree_one_leaf_trees_and_all_shapes():
    """Degenerate cases: a lone root leaf, and every shape with <= 5 leaves in one forest."""
    V = 40
    shapes = [None, None] + [s for n in range(2, 6) for s in gen.all_shapes(n)]
    words = gen.rng(2).integers(0, V, sum(map(gen.n_leaves, shapes)))
    f = gen.forest_from_shapes(shapes, words)
    B = len(shapes)
    prog = pg.treelstm_program(V=V, E=16, H=32, C=2, B=B, lr=0.2)
    labels = gen.rng(3).integers(0, 2, B).astype(np.int32)
    _check(prog, [tuple(f) + (labels,)])


def test_tree_c3_full_size():
    """C3: SST-shaped forests, B=25, H=E=300, V=20000."""
    V, B = 20000, 25
    prog = pg.treelstm_program(V=V, E=300, H=300, C=2, B=B, lr=0.05)
    _check(prog, [gen.sst_forest(gen.SEED_C3, 0, B, V)], scale=0.05)


def test_tree_guard_failures():
    V, B = 50, 4
    prog = pg.treelstm_program(V=V, E=16, H=32, C=2, B=B, lr=0.2)
    kind, left, right, word, off, label = gen.sst_forest(gen.SEED_C3, 1, B, V, max_leaves=8)
    bad_word = word.copy(); bad_word[int(np.argmax(kind == 0))] = V          # leaf word out of range
    unary = right.copy(); i = int(np.argmax(kind == 1)); unary[i] = left[i]  # l == r
    bad_off = off.copy(); bad_off[2] = bad_off[1]                          # empty tree
    forests = [(kind, left, right, bad_word, off, label), (kind, left, unary, word, off, label),
               (kind, left, right, word, bad_off, label)]
    _check(prog, forests, check_sched=False)
    janus = J()
    gf = janus.Graph(prog, fail_assert_id=8)
    state = gen.uniform_params(prog, 3, 0.3)
    dev = to_dev(state)
    st, fail = gf.run(to_dev([kind, left, right, word, off, label]), dev, gf.new_workspace())
    assert st == I.ASSUMPTION_FAILED and fail["assumption_id"] == 8
    assert all(a.tobytes() == b.tobytes() for a, b in zip(to_host(dev), state))


def test_tree_level_loops_on_one_cta():
    """The ablation's -PARL configuration (tree_grid=1: every tile of a level on one CTA, the
    backward streaming U^T) computes the same step."""
    V, B = 50, 6
    prog = pg.treelstm_program(V=V, E=24, H=32, C=2, B=B, lr=0.2)
    _check(prog, [gen.sst_forest(gen.SEED_C3, 9, B, V, max_leaves=12)], tree_grid=1)
