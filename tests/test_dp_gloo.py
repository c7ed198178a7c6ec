"""Data-parallel host logic on CPU with world_size 2 over gloo (gradients averaged over
workers; reading Q12: one failing rank aborts every rank).

Each process runs its shard of the step with the oracle, then follows the same protocol as the
GPU path (host_dp.cpp): allreduce(sum) of the gradient arena, global agreement = MIN of the packed
failure key (id << 48 | rank << 40 | index), commit with sum / N. The result must equal the
in-process DP emulation oracle.run_dp_step, and every rank must commit identical parameters.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import interp as I
from oracle import numerics as nm
from workloads import gen, programs as pg

KEY_PASS = (1 << 64) - 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup(B=3, T=4, V=9):
    prog = pg.lstm_lm_program(V=V, E=4, H=5, L=2, B=B, T=T, lr=0.5)
    st = [np.asarray(s, np.float64) if s.dtype.kind == "f" else s for s in gen.uniform_params(prog, 3, 0.3)]
    r0 = gen.rng(8)
    tok = r0.integers(0, V, (2 * B, T)).astype(np.int32)
    tgt = r0.integers(0, V, (2 * B, T)).astype(np.int32)
    return prog, st, tok, tgt


def _worker(rank, world, port, bad_rank, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1812_01329_b200 import janus as J
        # the unique-id plumbing of bench.py (bytes broadcast from rank 0)
        payload = J.broadcast_bytes(bytes(range(128)) if rank == 0 else None, rank)
        assert payload == bytes(range(128))
        prog, st, tok, tgt = _setup()
        B, T = 3, 4
        ln = np.full(B, T, np.int32)
        if rank == bad_rank:
            ln = ln.copy(); ln[1] = T - 1          # TRIP_COUNT (id 2) fails on this rank only
        args = [tok[rank * B:(rank + 1) * B], tgt[rank * B:(rank + 1) * B], ln]
        f = I.check_guards(prog, args, st)
        key = KEY_PASS if f is None else (f.assumption_id << 48) | (rank << 40) | f.index
        ex, grads = I._forward_backward(prog, args, st, nm.Prec("f32"))
        # arena allreduce (sum) — every rank issues it, whatever its outcome
        arena = torch.tensor(np.concatenate([grads[k].reshape(-1) for k in sorted(grads)]))
        dist.all_reduce(arena, op=dist.ReduceOp.SUM)
        # agreement: MIN of the packed key (as signed int64 with the pass value mapped to max)
        kt = torch.tensor([key - (1 << 63)], dtype=torch.int64)
        dist.all_reduce(kt, op=dist.ReduceOp.MIN)
        gkey = int(kt.item()) + (1 << 63)
        if gkey != KEY_PASS:
            q.put((rank, "failed", gkey >> 48, (gkey >> 40) & 0xFF, gkey & ((1 << 40) - 1)))
            return
        tot, o = {}, 0
        for k in sorted(grads):
            n = grads[k].size
            tot[k] = arena[o:o + n].numpy().reshape(grads[k].shape)
            o += n
        new = I._commit(prog, st, ex.effects, tot, world)
        q.put((rank, "ok", [x.tolist() for x in new]))
    finally:
        dist.destroy_process_group()


def _run(bad_rank):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, bad_rank, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = [q.get(timeout=240) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    return sorted(out, key=lambda x: x[0])


def test_dp_two_ranks_gloo_matches_oracle_dp():
    out = _run(bad_rank=-1)
    assert all(o[1] == "ok" for o in out)
    prog, st, tok, tgt = _setup()
    B, T = 3, 4
    ref = I.run_dp_step(prog, [[tok[r * B:(r + 1) * B], tgt[r * B:(r + 1) * B], np.full(B, T, np.int32)]
                               for r in range(2)], [st, st], mode="f32")
    for k, s in enumerate(prog.slots):
        if s.param:
            a0 = np.asarray(out[0][2][k]); a1 = np.asarray(out[1][2][k])
            assert a0.tobytes() == a1.tobytes(), s.name        # identical params on every rank
            np.testing.assert_allclose(a0, ref[0].state[k], atol=1e-14)


def test_dp_one_rank_failure_aborts_all_ranks():
    out = _run(bad_rank=1)
    assert [o[1] for o in out] == ["failed", "failed"]
    assert all((o[2], o[3], o[4]) == (2, 1, 1) for o in out)   # id 2, rank 1, element 1
