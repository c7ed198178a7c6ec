"""Is a step host-bound? Per-phase device times of the TreeLSTM (C3, B=25) and LM (C2) steps as
launched normally, and with a spin kernel queued first so that every launch of the step is
enqueued before the GPU reaches it (phase times then exclude host-issue gaps); plus the host
time of one janus_run.  usage: python scripts/host_bound.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1812_01329_b200 import janus as J
from workloads import gen, programs as pg


def phases(g, run, n, spin):
    J.dev_profile(g, True)
    wall = 0.0
    for k in range(n):
        if spin:
            torch.cuda._sleep(2_000_000)  # ~1 ms of spinning: the step is queued behind it
        t0 = time.perf_counter()
        run(k)
        wall += time.perf_counter() - t0
    ph = J.dev_phase_report(g)
    J.dev_profile(g, False)
    return {k: round(v[0] / n * 1e3, 1) for k, v in ph.items()}, wall / n * 1e6


def report(name, g, run, n=20):
    for k in range(3):
        run(k)
    torch.cuda.synchronize()
    for spin in (False, True):
        ph, wall = phases(g, run, n, spin)
        tot = sum(v for k, v in ph.items())
        print(f"{name} spin={spin}: phases sum {tot:.1f} us, host wall per call {wall:.1f} us  {ph}")


tp = pg.treelstm_program(V=20000, E=300, H=300, C=2, B=25, lr=0.05)
gt = J.Graph(tp)
wst = gt.new_workspace()
stt = [torch.tensor(x, device="cuda") for x in gen.uniform_params(tp, 1, 0.05)]
forests = [[torch.tensor(a, device="cuda") for a in gen.sst_forest(gen.SEED_C3, k, 25, 20000)] for k in range(4)]
report("tree_b25", gt, lambda k: gt.run(forests[k % 4], stt, wst))

B, T, V = 64, 35, 10000
prog = pg.lstm_lm_program(V=V, E=650, H=650, L=2, B=B, T=T, lr=1.0)
g = J.Graph(prog)
ws = g.new_workspace()
st = [torch.tensor(x, device="cuda") for x in gen.uniform_params(prog, 1, 0.05)]
batches = [[torch.tensor(a, device="cuda") for a in b] for b in gen.lm_batches(gen.SEED_C2, B, T, V, 4)]
loss = torch.zeros(1, device="cuda")
report("lm_c2", g, lambda k: g.run(batches[k % 4], st, ws, outs=[loss]))
