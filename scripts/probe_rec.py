"""Timeline of the layer-0 recurrent kernels (every CTA) for the C2 step via %globaltimer probes.

usage: python scripts/probe_rec.py [JANUS_REC_CH values ...]   (one report per value)
"""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from workloads import gen, programs as pg
from paper_1812_01329_b200 import janus as J
J.lib.janus_dev_set_probe.restype = C.c_int32
J.lib.janus_dev_set_probe.argtypes = [C.c_void_p, C.c_void_p]
B, T, H = 64, 35, 650
NC = 4 * ((H + 63) // 64)
NAMES = ["start", "flags_ok", "tma_issued", "tmem_read", "mma_issued", "mma_done", "epi_done", "published",
         "op0_land", "op0_mma", "op1_land", "op1_mma", "op2_land", "op2_mma", "sent/op3_land", "peers_ok/op3_mma"]


def report(buf):
    full = buf.cpu().numpy().astype(np.float64).reshape(2, 128, T, 16)
    g0 = (H + 15) // 16
    parts = [("fwd layer0", full[0, :g0])]
    if full[0, g0:, 1:-1, 7].any():  # wavefront launch: layer-1 CTAs follow
        parts.append(("fwd layer1 (wavefront)", full[0, g0:g0 + (H + 7) // 8]))
    nb1 = 4 * ((H + 63) // 64)  # K-split clusters of layer 1 (or of the only layer)
    parts.append(("bwd layer1 (or single layer)", full[1, :nb1]))
    if full[1, nb1:, 1:-1, 7].any():  # backward wavefront: layer-0 CTAs follow
        parts.append(("bwd layer0 (wavefront)", full[1, nb1:nb1 + 4 * ((H + 31) // 32)]))
    for dirn, a in parts:
        t0 = a[:, :, 0].min(axis=0)  # earliest CTA start of each step
        per = np.median(np.diff(t0))
        print(f"== {dirn}: step period {per:.0f} ns; offsets from the step's earliest start (ns)")
        for k, n in enumerate(NAMES):
            if n == "-" or np.all(a[:, 1:-1, k] == 0):
                continue
            rel = a[:, 1:-1, k] - t0[None, 1:-1]
            print(f"   {n:12s} med {np.median(rel):7.0f}  p90 {np.percentile(rel, 90):7.0f}  "
                  f"max-cta-median {np.median(rel, axis=1).max():7.0f} (cta {np.median(rel, axis=1).argmax()})")
        pub = a[:, 1:-1, 7] - t0[None, 1:-1]
        print("   last publisher histogram:", np.bincount(pub.argmax(axis=0), minlength=NC).tolist())
        own = a[:, 1:-1, 7] - a[:, 1:-1, 1]
        print(f"   own work flags_ok->published: med {np.median(own):.0f} max {own.max():.0f}")


prog = pg.lstm_lm_program(V=10000, E=H, H=H, L=2, B=B, T=T, lr=1.0)
g = J.Graph(prog)
ws = g.new_workspace()
state = [torch.tensor(x, device="cuda") for x in gen.uniform_params(prog, 1, 0.05)]
args = [torch.tensor(a, device="cuda") for a in list(gen.lm_batches(gen.SEED_C2, B, T, 10000, 1))[0]]
buf = torch.zeros(2 * 128 * 16 * T, dtype=torch.int64, device="cuda")
for k in range(3):
    g.run(args, state, ws, outs=[torch.zeros(1, device="cuda")])
for ch in (sys.argv[1:] or [None]):
    if ch is not None:
        os.environ["JANUS_REC_CH"] = ch
        print(f"######## JANUS_REC_CH={ch}")
    buf.zero_()
    J.lib.janus_dev_set_probe(g.h, buf.data_ptr())
    g.run(args, state, ws, outs=[torch.zeros(1, device="cuda")])
    torch.cuda.synchronize()
    J.lib.janus_dev_set_probe(g.h, None)
    report(buf)
