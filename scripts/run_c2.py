"""Run N C2 training steps through janus_run (for ncu / sanitizer captures; no timing).

usage: python scripts/run_c2.py [steps] [c2|c2big|c3|c4|c1]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1812_01329_b200 import janus as J  # noqa: E402
from workloads import gen, programs as pg  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
wl = sys.argv[2] if len(sys.argv) > 2 else "c2"
if wl == "c2":
    prog = pg.lstm_lm_program(V=10000, E=650, H=650, L=2, B=64, T=35, lr=1.0)
    batches = list(gen.lm_batches(gen.SEED_C2, 64, 35, 10000, steps))
elif wl == "c2big":  # V = 10^5: the xent / commit / embedding-gradient kernels stream >= 256 MB
    prog = pg.lstm_lm_program(V=100000, E=650, H=650, L=2, B=64, T=35, lr=1.0)
    batches = list(gen.lm_batches(gen.SEED_C2, 64, 35, 100000, steps))
elif wl == "c1":
    prog = pg.lstm_lm_program(V=32, E=16, H=16, L=1, B=4, T=8, lr=0.1, gemm="f32")
    batches = [b for b in gen.c1_batches()[:steps]]
elif wl == "c2small":
    prog = pg.lstm_lm_program(V=300, E=72, H=100, L=2, B=33, T=9, lr=0.5)
    batches = list(gen.lm_batches(gen.SEED_C2, 33, 9, 300, steps))
elif wl == "c2v":  # V >= 4096: the split-K reduce-add dh_top launch, small otherwise
    prog = pg.lstm_lm_program(V=5000, E=64, H=64, L=2, B=16, T=5, lr=0.5)
    batches = list(gen.lm_batches(gen.SEED_C2, 16, 5, 5000, steps))
elif wl == "c3rnn":
    prog = pg.treernn_program(V=50, H=32, C=2, B=6, lr=0.2)
    batches = [gen.sst_forest(gen.SEED_C3, k, 6, 50, max_leaves=12) for k in range(steps)]
elif wl == "c3":
    prog = pg.treelstm_program(V=20000, E=300, H=300, C=2, B=25, lr=0.05)
    batches = [gen.sst_forest(gen.SEED_C3, k, 25, 20000) for k in range(steps)]
elif wl == "c3small":
    prog = pg.treelstm_program(V=50, E=24, H=32, C=2, B=6, lr=0.2)
    batches = [gen.sst_forest(gen.SEED_C3, k, 6, 50, max_leaves=12) for k in range(steps)]
else:
    raise SystemExit(wl)
g = J.Graph(prog)
ws = g.new_workspace()
state = [torch.tensor(x, device="cuda") for x in gen.uniform_params(prog, 5, 0.05)]
for k in range(steps):
    st, fail = g.run([torch.tensor(np.asarray(a), device="cuda") for a in batches[k % len(batches)]], state, ws)
    print("step", k, J.STATUS_NAMES[st], fail)
torch.cuda.synchronize()
