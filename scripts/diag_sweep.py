import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import interp as I
from workloads import gen, programs as pg
from tests.helpers import rel_err, to_dev, to_host
from paper_1812_01329_b200 import janus as J

def run(V, E, H, L, B, T):
    prog = pg.lstm_lm_program(V=V, E=E, H=H, L=L, B=B, T=T, lr=0.5)
    g = J.Graph(prog); ws = g.new_workspace()
    state = gen.uniform_params(prog, 5, 0.2)
    args = list(gen.lm_batches(gen.SEED_C2, B, T, V, 1))[0]
    ora = I.run_graph_step(prog, list(args), state, mode="bf16")
    dev = to_dev(state); loss = torch.zeros(1, device="cuda")
    st, fail = g.run(to_dev(args), dev, ws, outs=[loss]); got = to_host(dev)
    sid = {s.name: k for k, s in enumerate(prog.slots)}
    eh = max(rel_err(got[sid[f"h{l}"]], ora.state[sid[f"h{l}"]]) for l in range(L))
    print(f"V{V} E{E} H{H} L{L} B{B} T{T}: loss {loss.item():.6f} vs {float(ora.outputs[0]):.6f}  h err {eh:.2e}", flush=True)

for cfg in [(64,40,48,1,8,6),(64,40,96,1,8,6),(64,40,100,1,8,6),(64,40,48,1,33,6),(64,40,48,1,32,6),(64,72,48,1,8,6),(300,40,48,1,8,6),(64,40,48,1,8,9),(64,40,112,1,8,6),(64,40,80,1,8,6)]:
    run(*cfg)
