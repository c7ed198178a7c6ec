"""Run a few C3 TreeLSTM training steps (for ncu launch lists). usage: python scripts/run_tree.py [B] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1812_01329_b200 import janus as J
from workloads import gen, programs as pg

B = int(sys.argv[1]) if len(sys.argv) > 1 else 25
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
tp = pg.treelstm_program(V=20000, E=300, H=300, C=2, B=B, lr=0.05)
g = J.Graph(tp)
ws = g.new_workspace()
st = [torch.tensor(x, device="cuda") for x in gen.uniform_params(tp, 1, 0.05)]
fs = [[torch.tensor(a, device="cuda") for a in gen.sst_forest(gen.SEED_C3, k, B, 20000)] for k in range(n)]
for k in range(n):
    print(g.run(fs[k], st, ws))
torch.cuda.synchronize()
