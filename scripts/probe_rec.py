"""Timeline of the layer-0 recurrent kernels (CTA 0) for the C2 step via %globaltimer probes."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from workloads import gen, programs as pg
from paper_1812_01329_b200 import janus as J
J.lib.janus_dev_set_probe.restype = C.c_int32
J.lib.janus_dev_set_probe.argtypes = [C.c_void_p, C.c_void_p]
B, T = 64, 35
prog = pg.lstm_lm_program(V=10000, E=650, H=650, L=2, B=B, T=T, lr=1.0)
g = J.Graph(prog); ws = g.new_workspace()
state = [torch.tensor(x, device="cuda") for x in gen.uniform_params(prog, 1, 0.05)]
args = [torch.tensor(a, device="cuda") for a in list(gen.lm_batches(gen.SEED_C2, B, T, 10000, 1))[0]]
buf = torch.zeros(16 * T, dtype=torch.int64, device="cuda")
for k in range(3):
    g.run(args, state, ws, outs=[torch.zeros(1, device="cuda")])
J.lib.janus_dev_set_probe(g.h, buf.data_ptr())
g.run(args, state, ws, outs=[torch.zeros(1, device="cuda")])
torch.cuda.synchronize()
d = buf.cpu().numpy().astype(np.float64).reshape(2, T, 8)
names = ["start", "flags_ok", "tma_issued", "chunk0_landed", "mma_issued", "mma_done", "epi_done", "published"]
for dirn, a in (("fwd", d[0]), ("bwd", d[1])):
    rel = a - a[:, :1]
    print(f"== {dirn}: step period {np.median(np.diff(a[:, 0])):.0f} ns; median offsets from step start (ns):")
    for k, n in enumerate(names):
        print(f"   {n:14s} {np.median(rel[1:-1, k]):8.0f}")
