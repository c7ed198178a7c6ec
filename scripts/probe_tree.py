"""Per-barrier timeline of the TreeLSTM forward / backward kernels (C3) via %globaltimer probes:
for every grid barrier, the work phase before it (last CTA arrival - previous release) and the
barrier itself (median release - last arrival).  usage: python scripts/probe_tree.py [B]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1812_01329_b200 import janus as J
from workloads import gen, programs as pg

J.lib.janus_dev_set_probe.restype = C.c_int32
J.lib.janus_dev_set_probe.argtypes = [C.c_void_p, C.c_void_p]
B = int(sys.argv[1]) if len(sys.argv) > 1 else 25
tp = pg.treelstm_program(V=20000, E=300, H=300, C=2, B=B, lr=0.05)
g = J.Graph(tp)
ws = g.new_workspace()
st = [torch.tensor(x, device="cuda") for x in gen.uniform_params(tp, 1, 0.05)]
f = [torch.tensor(a, device="cuda") for a in gen.sst_forest(gen.SEED_C3, 0, B, 20000)]
for _ in range(3):
    g.run(f, st, ws)
buf = torch.zeros(5 * 256 * 256 * 2, dtype=torch.int64, device="cuda")
J.lib.janus_dev_set_probe(g.h, buf.data_ptr())
g.run(f, st, ws)
torch.cuda.synchronize()
J.lib.janus_dev_set_probe(g.h, None)
lvl = J.dev_workspace_region(g, ws, "tree.lvl_off")
meta = J.dev_workspace_region(g, ws, "tree.meta")
L = int(meta[0])
print(f"B={B} levels={L} nodes/level={[int(lvl[l + 1] - lvl[l]) for l in range(L)]}")
pp = buf.cpu().numpy()
p = pp[:3 * 256 * 256 * 2].reshape(3, 256, 256, 2)
q4 = pp[2 * 256 * 256 * 2:4 * 256 * 256 * 2].reshape(256, 256, 4)
q5 = pp[3 * 256 * 256 * 2:5 * 256 * 256 * 2].reshape(256, 256, 4)
grid = 148  # host_tree.cpp: one CTA per SM
for kern, name in ((0, "fwd"), (1, "bwd")):
    a, r = p[kern, :, :grid, 0], p[kern, :, :grid, 1]
    ks = [k for k in range(256) if (a[k] > 0).all()]
    if not ks:
        continue
    t0 = a[ks[0]].min()
    print(f"-- {name}: {len(ks)} barriers, span {(np.median(r[ks[-1]]) - t0) / 1e3:.1f} us (from first arrival)")
    prev = None
    tot_w = tot_b = 0.0
    for k in ks:
        last = a[k].max()
        rel = np.median(r[k])
        w = (last - prev) / 1e3 if prev is not None else float("nan")
        bsync = (rel - last) / 1e3
        spread = (last - a[k].min()) / 1e3
        if prev is not None:
            tot_w += w
        tot_b += bsync
        print(f"  sync {k:3d}: work {w:6.2f} us  barrier {bsync:5.2f} us  arrival spread {spread:6.2f} us  slowest cta {int(a[k].argmax())}")
        prev = rel
    print(f"  total work {tot_w:.1f} us, barriers {tot_b:.1f} us")

# forward internal levels: mainloop (release of the level's start barrier -> last TMEM-full) and
# epilogue (TMEM-full -> epilogue done), slowest CTA
a, r = p[0, :, :grid, 0], p[0, :, :grid, 1]
for l in range(1, L):
    pr = q4[l, :grid]
    act = pr[:, 0] > 0
    if not act.any():
        continue
    start = np.median(r[l + 1])
    print(f"  level {l:2d} ({int(lvl[l + 1] - lvl[l]):4d} nodes, {int(act.sum())} CTAs): "
          f"mainloop {(pr[act, 0].max() - start) / 1e3:5.2f} us  tmem {((pr[act, 2] - pr[act, 0]).max()) / 1e3:5.2f} us  epilogue {((pr[act, 1] - pr[act, 2]).max()) / 1e3:5.2f} us")

# backward dgrad tile loops (one barrier per level: the cell backward runs in the dgrad
# epilogue): level l runs after barrier L - 2 - l of the backward kernel (the top level at entry)
print("-- backward dgrad levels (+ fused cell backward)")
ab, rb = p[1, :, :grid, 0], p[1, :, :grid, 1]
for l in range(L - 1, 0, -1):
    pr = q5[l, :grid]
    act = pr[:, 0] > 0
    if not act.any():
        continue
    k = L - 2 - l
    start = np.median(rb[k]) if k >= 0 else np.min(ab[0])
    print(f"  level {l:2d} ({int(lvl[l + 1] - lvl[l]):4d} nodes, {int(act.sum())} CTAs): "
          f"mainloop {(pr[act, 0].max() - start) / 1e3:5.2f} us  tmem {((pr[act, 2] - pr[act, 0]).max()) / 1e3:5.2f} us  epilogue {((pr[act, 1] - pr[act, 2]).max()) / 1e3:5.2f} us")

sc = pp[4 * 256 * 256 * 2: 4 * 256 * 256 * 2 + 8]
if sc[0] > 0:
    names = ["init + stage children", "heights", "histogram+offsets", "stable placement", "parent slots"]
    print("-- schedule kernel phases (us):", {names[i]: round((sc[i + 1] - sc[i]) / 1e3, 2) for i in range(5)})  # interval i = probe i+1 - probe i
