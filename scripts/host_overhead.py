"""Host-side cost of one janus_run (C3 TreeLSTM and C2 LM): wall time per call vs the GPU time of
its kernels (per-phase events), and the host time to enqueue (call return without the sync is not
observable, so: wall - GPU busy)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1812_01329_b200 import janus as J
from workloads import gen, programs as pg

for B in (25, 256):
    tp = pg.treelstm_program(V=20000, E=300, H=300, C=2, B=B, lr=0.05)
    g = J.Graph(tp)
    ws = g.new_workspace()
    st = [torch.tensor(x, device="cuda") for x in gen.uniform_params(tp, 1, 0.05)]
    fs = [[torch.tensor(a, device="cuda") for a in gen.sst_forest(gen.SEED_C3, k, B, 20000)] for k in range(4)]
    for k in range(5):
        g.run(fs[k % 4], st, ws)
    torch.cuda.synchronize()
    K = 50
    t0 = time.perf_counter()
    for k in range(K):
        g.run(fs[k % 4], st, ws)
    wall = (time.perf_counter() - t0) / K * 1e3
    J.dev_profile(g, True)
    for k in range(K):
        g.run(fs[k % 4], st, ws)
    ph = J.dev_phase_report(g)
    J.dev_profile(g, False)
    gpu = sum(v[0] for v in ph.values()) / K
    print(f"C3 B={B}: wall {wall:.3f} ms/step, event-timed phases {gpu:.3f} ms", flush=True)
