import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import interp as I, numerics as nm
from workloads import gen, programs as pg
from tests.helpers import rel_err, to_dev, to_host
from paper_1812_01329_b200 import janus as J
V, E, H, B = 50, 24, 32, 3
prog = pg.treelstm_program(V=V, E=E, H=H, C=2, B=B, lr=0.2)
state = gen.uniform_params(prog, 3, 0.3)
f = list(gen.sst_forest(gen.SEED_C3, 0, B, V, max_leaves=3, chain=True))
print("kind", f[0].tolist()); print("left", f[1].tolist()); print("right", f[2].tolist()); print("off", f[4].tolist())
g = J.Graph(prog); ws = g.new_workspace()
dev = to_dev(state)
st, fail = g.run(to_dev(f), dev, ws, outs=[torch.zeros(1, device="cuda")])
dh = J.dev_workspace_region(g, ws, "tree.dh_node", np.float32).reshape(-1, H)
dc = J.dev_workspace_region(g, ws, "tree.dc_node", np.float32).reshape(-1, H)
ex = I.GraphExec(prog, f, state, nm.Prec("bf16")); ex.run_body(0, None)
grads = ex.tape.backward(ex.outputs[0])
kind = f[0]
leaves = [n for n in range(len(kind)) if kind[n] == 0]
ents = [e for e in ex.tape.entries if e[0] == "TREELSTM_LEAF"]
cells = [n for n in range(len(kind)) if kind[n] == 1]
cents = [e for e in ex.tape.entries if e[0] == "TREELSTM_CELL"]
for n, e in zip(leaves, ents):
    oh, oc = e[2]
    gh = grads.get(oh.id); gc = grads.get(oc.id)
    print(f"leaf {n}: dh err {rel_err(dh[n], gh.reshape(-1)) if gh is not None else None:.2e}  dc err {rel_err(dc[n], gc.reshape(-1)) if gc is not None else 'none'}")
for n, e in zip(cells, cents):
    oh, oc = e[2]
    gh = grads.get(oh.id); gc = grads.get(oc.id)
    print(f"cell {n}: dh err {rel_err(dh[n], gh.reshape(-1)):.2e}  dc err {rel_err(dc[n], gc.reshape(-1)) if gc is not None else 'none (root)'}")
