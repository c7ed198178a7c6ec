"""One (or N) imperative C2 steps through janus_run_imperative (for ncu launch lists / host timing)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1812_01329_b200 import janus as J  # noqa: E402
from workloads import gen, programs as pg  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
prog = pg.lstm_lm_program(V=10000, E=650, H=650, L=2, B=64, T=35, lr=1.0)
g = J.Graph(prog)
ws = g.new_workspace()
state = [torch.tensor(x, device="cuda") for x in gen.uniform_params(prog, 5, 0.05)]
batches = [[torch.tensor(np.asarray(a), device="cuda") for a in b] for b in gen.lm_batches(gen.SEED_C2, 64, 35, 10000, 2)]
g.run_imperative(batches[0], state, ws)
torch.cuda.synchronize()
for k in range(steps):
    t0 = time.perf_counter()
    g.run_imperative(batches[k % 2], state, ws)
    torch.cuda.synchronize()
    print(f"imperative step {k}: {1e3 * (time.perf_counter() - t0):.1f} ms wall", flush=True)
