"""libjanus's own data-parallel protocol (host_dp.cpp) driven by two CPU processes over gloo.

P:298 §5: the step averages gradients over workers with collectives inside the step; reading
Q12 / R7: one failing rank aborts every rank, and every rank reports the same failure (minimum
assumption id, then minimum rank). The library's collective sequence — the gradient-arena
allreduces of janus_dev_dp_segments in issue order, then the abort agreement — runs through
janus_dev_dp_host_step with the transport swapped for a gloo allreduce on host buffers. The
agreement arithmetic is the same code the device kernels run (step_kernels.h dp_pack /
dp_observed / dp_unpack); the arena layout is the graph's real workspace plan."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from workloads import programs as pg

OK, ASSUMPTION_FAILED, ERR_RUNTIME = 0, 1, 4
LM_GRADS = ["lm.gWdec", "lm.gWih0", "lm.gWhh0", "lm.gWih1", "lm.gWhh1", "lm.dEd"]
TREE_GRADS = ["tree.gU", "tree.gWl", "tree.gWc", "tree.gbc"]
# (rank-0 local outcome, rank-1 local outcome); outcome = (failure (id, index, observed) | None,
# runtime error)
CASES = [
    ((None, 0), (None, 0)),
    ((None, 0), ((2, 3, 34), 0)),          # one rank's AssertOp fails -> every rank aborts
    (((5, 0, 1), 0), ((2, 7, 30), 0)),     # smallest id wins, whatever the rank
    (((2, 7, 9), 0), ((2, 1, 4), 0)),      # same id: smallest rank wins, with ITS index/observed
    (((2, -1, -1), 0), (None, 0)),         # forced failure (R5: index / observed -1)
    ((None, 1), (None, 0)),                # runtime error on one rank -> ERR_RUNTIME everywhere
    ((None, 0), ((0xFFFFFFFF, 0, 0), 0)),  # null step with invalid arguments -> ERR_RUNTIME
    ((None, 1), ((3, 2, 8), 0)),           # an assumption failure outranks a runtime error
]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _allreduce(arr, op):
    t = torch.from_numpy(arr)
    dist.all_reduce(t, op={0: dist.ReduceOp.SUM, 1: dist.ReduceOp.MIN, 2: dist.ReduceOp.MAX}[op])


def _graphs(rank):
    from paper_1812_01329_b200 import janus as J
    nid = bytes(128)  # no NCCL communicator is created on this path
    lm = J.Graph(pg.lstm_lm_program(V=64, E=40, H=48, L=2, B=8, T=6, lr=0.5), world_size=2, rank=rank,
                 nccl_id=nid)
    tree = J.Graph(pg.treelstm_program(V=50, E=24, H=32, C=2, B=6, lr=0.2), world_size=2, rank=rank,
                   nccl_id=nid)
    return J, [("lm", lm, LM_GRADS), ("tree", tree, TREE_GRADS)]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        J, graphs = _graphs(rank)
        res = {}
        for name, g, grads in graphs:
            J.dev_dp_set_host_collective(g, _allreduce)
            segs = J.dev_dp_segments(g)
            regions = {k: J.dev_workspace_region_bytes(g, k) for k in grads + ["arena"]}
            # host workspace: every gradient float = (rank + 1) * (1 + element index mod 97); the
            # bytes outside the arena are a rank-specific filler that must survive
            ws = np.full(g.workspace_bytes, 0x11 * (rank + 1), np.uint8)
            for k in grads:
                off, n = regions[k]
                ws[off:off + n].view(np.float32)[:] = (rank + 1) * (1 + np.arange(n // 4) % 97)
            outcomes = []
            for c in CASES:
                fl, rt = c[rank]
                outcomes.append(J.dev_dp_host_step(g, ws, fl, rt))
            res[name] = dict(segs=segs, regions=regions, ws=ws, outcomes=outcomes)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def two_ranks():
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    return out


@pytest.mark.parametrize("name", ["lm", "tree"])
def test_arena_segments_cover_every_gradient(two_ranks, name):
    """Both ranks issue the same segments; they tile the arena exactly; every gradient buffer of
    the plan lies inside it (so one sequence of collectives reduces every gradient)."""
    r0, r1 = two_ranks[0][name], two_ranks[1][name]
    assert r0["segs"] == r1["segs"] and r0["regions"] == r1["regions"]
    segs, reg = r0["segs"], r0["regions"]
    a_off, a_len = reg["arena"]
    assert segs[0][1] == a_off and sum(s[2] for s in segs) == a_len
    for (c0, o0, n0), (c1, o1, n1) in zip(segs, segs[1:]):
        assert o0 + n0 == o1                               # contiguous, in order
    grads = [reg[k] for k in reg if k != "arena"]
    for off, n in grads:
        assert a_off <= off and off + n <= a_off + a_len
    for (o0, n0), (o1, n1) in zip(sorted(grads), sorted(grads)[1:]):
        assert o0 + n0 <= o1                               # disjoint
    if name == "lm":  # the overlapped early segment is exactly dW_dec | db_dec (split communicator)
        assert segs[0][0] == 2 and (segs[0][1], segs[0][2]) == reg["lm.gWdec"]
        assert [s[0] for s in segs[1:]] == [1]
    else:
        assert [s[0] for s in segs] == [1]


@pytest.mark.parametrize("name", ["lm", "tree"])
def test_arena_allreduce_sums_gradients_only(two_ranks, name):
    r0, r1 = two_ranks[0][name], two_ranks[1][name]
    a_off, a_len = r0["regions"]["arena"]
    # every step (failed or not) reduces the arena: (1 + 2) * pattern after the first, doubled by
    # every later one (both ranks then hold the same values)
    scale = 3.0 * 2.0 ** (len(CASES) - 1)
    for k, (off, n) in r0["regions"].items():
        if k == "arena":
            continue
        pat = (1 + np.arange(n // 4) % 97).astype(np.float64)
        for r in (r0, r1):
            np.testing.assert_array_equal(r["ws"][off:off + n].view(np.float32), (scale * pat).astype(np.float32))
    for rank, r in ((0, r0), (1, r1)):   # bytes outside the arena untouched
        outside = np.concatenate([r["ws"][:a_off], r["ws"][a_off + a_len:]])
        assert (outside == 0x11 * (rank + 1)).all()


@pytest.mark.parametrize("name", ["lm", "tree"])
def test_agreement_every_rank_decodes_the_same_outcome(two_ranks, name):
    o0, o1 = two_ranks[0][name]["outcomes"], two_ranks[1][name]["outcomes"]
    assert o0 == o1
    expect = [
        (OK, None),
        (ASSUMPTION_FAILED, dict(assumption_id=2, rank=1, index=3, observed=34)),
        (ASSUMPTION_FAILED, dict(assumption_id=2, rank=1, index=7, observed=30)),
        (ASSUMPTION_FAILED, dict(assumption_id=2, rank=0, index=7, observed=9)),
        (ASSUMPTION_FAILED, dict(assumption_id=2, rank=0, index=-1, observed=-1)),
        (ERR_RUNTIME, None),
        (ERR_RUNTIME, None),
        (ASSUMPTION_FAILED, dict(assumption_id=3, rank=1, index=2, observed=8)),
    ]
    assert o0 == expect


def test_fused_reduction_leaves_only_the_embedding_gradient_to_nccl():
    """With fused_allreduce the weight gradients are reduced in the GEMM epilogue (NEXT-3); the
    step's NCCL segments shrink to the dense embedding gradient (rank-independent plan)."""
    from paper_1812_01329_b200 import janus as J
    prog = pg.lstm_lm_program(V=64, E=40, H=48, L=2, B=8, T=6, lr=0.5)
    plain = J.Graph(prog, world_size=2, rank=0, nccl_id=bytes(128))
    fused = J.Graph(prog, world_size=2, rank=1, nccl_id=bytes(128), fused_allreduce=True)
    ed = J.dev_workspace_region_bytes(plain, "lm.dEd")
    a0, alen = J.dev_workspace_region_bytes(plain, "arena")
    assert [s[0] for s in J.dev_dp_segments(plain)] == [2, 1]
    assert J.dev_dp_segments(fused) == [(1, ed[0], a0 + alen - ed[0])]
