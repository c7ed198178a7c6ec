"""Diagnostics: per-slot parity of one LM step (GPU vs oracle) under several metrics."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import interp as I
from workloads import gen, programs as pg
from tests.helpers import rel_err, to_dev, to_host
from paper_1812_01329_b200 import janus as J

def case(name, prog, batches, scale=0.1, seed=5):
    g = J.Graph(prog); ws = g.new_workspace()
    state = gen.uniform_params(prog, seed, scale)
    args = batches[0]
    ora = I.run_graph_step(prog, list(args), state, mode=prog.meta.get("gemm", "bf16") if prog.meta.get("gemm") == "f32" else "bf16")
    dev = to_dev(state); loss = torch.zeros(1, device="cuda")
    st, fail = g.run(to_dev(args), dev, ws, outs=[loss]); got = to_host(dev)
    print(f"== {name}: status {st} {fail} loss gpu {loss.item():.6f} ora {float(ora.outputs[0]):.6f}")
    for k, s in enumerate(prog.slots):
        o = np.asarray(ora.state[k], np.float64); gg = np.asarray(got[k], np.float64); old = np.asarray(state[k], np.float64)
        if s.param:
            do, dg = o - old, gg - old
            nz = np.abs(do) > 0
            print(f"  {s.name:8s} rel {rel_err(dg, do):.3e} maxabs/max {np.abs(dg-do).max()/max(np.abs(do).max(),1e-30):.3e} "
                  f"rel(nonzero) {rel_err(dg[nz], do[nz]) if nz.any() else 0:.3e} |do|max {np.abs(do).max():.3e} nz {nz.mean():.3f}")
        else:
            print(f"  {s.name:8s} rel {rel_err(gg, o):.3e}")

V, B, T = 64, 8, 6
case("small", pg.lstm_lm_program(V=V, E=40, H=48, L=2, B=B, T=T, lr=0.5), list(gen.lm_batches(gen.SEED_C2, B, T, V, 1)))
case("ragged", pg.lstm_lm_program(V=300, E=72, H=100, L=2, B=33, T=9, lr=0.5), list(gen.lm_batches(gen.SEED_C2, 33, 9, 300, 1)), scale=0.2)
case("b128", pg.lstm_lm_program(V=200, E=64, H=64, L=1, B=128, T=4, lr=0.5), list(gen.lm_batches(gen.SEED_C2, 128, 4, 200, 1)), scale=0.2)
if len(sys.argv) > 1:
    case("c2", pg.lstm_lm_program(V=10000, E=650, H=650, L=2, B=64, T=35, lr=1.0), list(gen.lm_batches(gen.SEED_C2, 64, 35, 10000, 1)), scale=0.05)
