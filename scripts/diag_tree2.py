import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import interp as I
from workloads import gen, programs as pg
from tests.helpers import rel_err, to_dev, to_host
from paper_1812_01329_b200 import janus as J
H = 32
def case(shapes, name):
    V = 40
    words = gen.rng(2).integers(0, V, sum(map(gen.n_leaves, shapes)))
    f = list(gen.forest_from_shapes(shapes, words)) + [np.ones(len(shapes), np.int32)]
    prog = pg.treelstm_program(V=V, E=16, H=H, C=2, B=len(shapes), lr=0.2)
    g = J.Graph(prog); ws = g.new_workspace()
    state = gen.uniform_params(prog, 3, 0.3)
    dev = to_dev(state); loss = torch.zeros(1, device="cuda")
    st, fail = g.run(to_dev(f), dev, ws, outs=[loss]); got = to_host(dev)
    ora = I.run_graph_step(prog, f, state, mode="bf16")
    errs = []
    for k, s in enumerate(prog.slots):
        if not s.param: continue
        do = np.asarray(ora.state[k], np.float64) - state[k]; dg = np.asarray(got[k], np.float64) - state[k]
        errs.append(f"{s.name} {rel_err(dg, do):.1e}")
    print(f"{name:28s} loss ok {abs(loss.item()-float(ora.outputs[0]))<1e-4}  " + "  ".join(errs), flush=True)
L = None
case([(None, None)], "(l,l)")
case([((None, None), None)], "((l,l),l)")
case([(None, (None, None))], "(l,(l,l))")
case([((None, None), (None, None))], "((l,l),(l,l))")
case([((None, None), None), None], "((l,l),l) + l")
case([(None, None), ((None, None), None)], "(l,l) + ((l,l),l)")
