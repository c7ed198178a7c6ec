import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import interp as I
from workloads import gen, programs as pg
from tests.helpers import rel_err, to_dev, to_host
from paper_1812_01329_b200 import janus as J

def case(V, E, H, B, maxl, seed=3, chain=False):
    prog = pg.treelstm_program(V=V, E=E, H=H, C=2, B=B, lr=0.2)
    g = J.Graph(prog); ws = g.new_workspace()
    state = gen.uniform_params(prog, seed, 0.3)
    f = list(gen.sst_forest(gen.SEED_C3, 0, B, V, max_leaves=maxl, chain=chain))
    dev = to_dev(state); loss = torch.zeros(1, device="cuda")
    st, fail = g.run(to_dev(f), dev, ws, outs=[loss]); got = to_host(dev)
    ora = I.run_graph_step(prog, f, state, mode="bf16")
    print(f"== V{V} E{E} H{H} B{B}: st {st} loss {loss.item():.6f} vs {float(ora.outputs[0]):.6f}")
    for k, s in enumerate(prog.slots):
        if not s.param: continue
        do = np.asarray(ora.state[k], np.float64) - state[k]; dg = np.asarray(got[k], np.float64) - state[k]
        print(f"   {s.name:7s} rel {rel_err(dg, do):.3e}  |do| {np.abs(do).max():.3e} |dg| {np.abs(dg).max():.3e}")
        if s.name == "b":
            print("     b blocks do", [np.abs(do[i*H:(i+1)*H]).max() for i in range(4)], "dg", [np.abs(dg[i*H:(i+1)*H]).max() for i in range(4)])
case(50, 24, 32, 6, 12)
case(50, 24, 32, 1, 1)
case(50, 24, 32, 2, 2)
case(50, 24, 32, 3, 3, chain=True)
