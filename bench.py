#!/usr/bin/env python
"""Benchmark: LSTM-LM training step of the speculative graph on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c3|c4] [--impl janus|reference]

One JSON line on rank 0. `value` = whole-job samples/s (a sample = one 35-token sequence) with
inputs resident in HBM, timed with CUDA events on the launch stream, max over ranks. `e2e` = the
same metric through janus_run with pinned HOST argument buffers (H2D inside the call) and the loss
read back to the host every step. `roofline` is the dominant kernel of the step, timed live with
per-phase CUDA events; `cpu_baseline` is the oracle on the host cores on a bounded sample.

--impl reference times the oracle (oracle/, the plain CPU interpreter of the paper's semantics) on
the host cores, each step a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import gen, programs as pg  # noqa: E402

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
BASELINE_METRIC = "LSTM/TreeLSTM train samples/s at 1/2/4/8 B200; tensor-pipe %; guard overhead"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        d["source"] = "measured (MEASURED_PEAKS.json)"
        return d
    d = dict(PEAKS_FALLBACK)
    d["source"] = "fallback (B200_PROFILING.md)"
    return d


# ----------------------------------------------------------------------------- workloads
def c2_program(B, speculate="unroll"):
    """C2: the Figure 1 program with `if training: update` (training = 1, VALUE_EQ-speculated)."""
    return pg.lstm_lm_program(V=10000, E=650, H=650, L=2, B=B, T=35, lr=1.0, speculate=speculate,
                              max_T=35, training_flag=True)


def c4_program(B):
    """C4: the C2 model with data-dependent widths (device While, RANGE guard), SURVEY §8(d)."""
    return pg.lstm_lm_program(V=10000, E=650, H=650, L=2, B=B, T=64, lr=1.0, speculate="while",
                              training_flag=True)


WORKLOADS = {
    "c2": dict(desc="C2 PTB-shaped LSTM LM: 2 layers, H=E=650, V=10000, T=35, B=64 per GPU, bf16 GEMM "
                    "operands / fp32 accumulate, unrolled speculative graph (TRIP_COUNT=35, training "
                    "flag speculated by VALUE_EQ)",
               B=64, T=35),
    "c4": dict(desc="C4 variable-length RNN: the C2 model, per-batch width W ~ U{5..64}, ragged lengths "
                    "U{1..W}, device While (RANGE guard), B=64 per GPU, bf16 / fp32 accumulate",
               B=64, T=64),
}


def lm_flops_per_sample(V, E, H, L, T):
    """Algorithmic training FLOPs of one sequence: 3x forward (fwd + dgrad + wgrad)."""
    cell = sum(2 * 4 * H * ((E if l == 0 else H) + H) for l in range(L))
    dec = 2 * H * V
    return 3 * T * (cell + dec)


def gemm_flops(name, V, E, H, TB):
    G4 = 4 * H
    table = {"gemm_in0": 2 * TB * G4 * E, "gemm_in1": 2 * TB * G4 * H, "gemm_dec": 2 * TB * V * H,
             "gemm_dWdec": 2 * V * (H + 1) * TB, "gemm_dh": 2 * TB * H * V,
             "gemm_dWhh0": 2 * G4 * H * TB, "gemm_dWhh1": 2 * G4 * H * TB,
             "gemm_dWih0": 2 * G4 * (E + 1) * TB, "gemm_dWih1": 2 * G4 * (H + 1) * TB,
             "gemm_dx0": 2 * TB * E * G4, "gemm_dx1": 2 * TB * H * G4}
    return table.get(name)


# ----------------------------------------------------------------------------- clocks
class Clocks:
    """nvidia-smi sampler (50 ms) started before the warm-up; a reader thread timestamps every
    line, and the summary keeps the samples taken inside the timed window (the warm-up steps keep
    the GPU busy until the sampler is producing, so a short timed region still gets samples)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.p = None
        self.lines = []  # (arrival time, fields)
        self.t0 = self.t1 = None

    def start(self):
        import threading
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True, bufsize=1)
        except OSError:
            self.p = None
            return self

        def reader():
            for line in self.p.stdout:
                if line.strip():
                    self.lines.append((time.time(), line.strip().split(",")))
        self.th = threading.Thread(target=reader, daemon=True)
        self.th.start()
        return self

    def producing(self):
        return self.p is None or len(self.lines) > 0

    def __enter__(self):  # the timed window
        self.t0 = time.time()
        return self

    def __exit__(self, *a):
        self.t1 = time.time()

    def stop(self):
        if self.p is None:
            return
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.th.join(timeout=2)

    def summary(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        lo, hi = (self.t0 or 0.0) - 0.06, (self.t1 or 1e30) + 0.06  # one sampling period of slack
        rows = [r for t, r in self.lines if lo <= t <= hi]
        window = "timed region"
        if not rows:  # no sample landed inside a very short window: the nearest ones after it
            rows = [r for t, r in self.lines if t >= lo][:3]
            window = "first samples after the timed region began"
        sm = [float(r[1]) for r in rows if len(r) > 2 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) > 2 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if "Active" in v and "Not" not in v})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "window": window}


# ----------------------------------------------------------------------------- CPU baselines
def _blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        return 1


def oracle_sample(B, T):
    """Time the oracle (as it stands) on one bounded sample: B sequences x T tokens of the C2 model."""
    from oracle import interp as I
    prog = pg.lstm_lm_program(V=10000, E=650, H=650, L=2, B=B, T=T, lr=1.0, training_flag=True)
    state = gen.uniform_params(prog, 1, 0.05)
    args = list(list(gen.lm_batches(gen.SEED_C2, B, T, 10000, 1))[0]) + [np.ones(1, np.int32)]
    t0 = time.perf_counter()
    r = I.run_graph_step(prog, list(args), state)
    dt = time.perf_counter() - t0
    assert r.status == I.OK
    return dt


def cpu_baseline():
    B, T = 64, 35
    dt = oracle_sample(B, T)
    return {"value": B / dt, "unit": "samples/s", "cores": _blas_threads(), "kind": "oracle",
            "sample": f"one C2 training step (B={B} sequences x T={T} tokens, full model) through "
                      f"oracle.run_graph_step in {dt:.1f} s",
            "host_cpus": os.cpu_count()}


def cpu_baseline_modes():
    """SURVEY §8(d) oracle modes beside the headline baseline: the C2 step on ONE thread (BLAS
    limited through threadpoolctl) and a C3 TreeLSTM step (B=25) on all threads."""
    from oracle import interp as I
    res = {}
    try:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=1):
            dt = oracle_sample(8, 35)
        res["c2_1thread"] = {"value": 8 / dt, "unit": "samples/s", "cores": 1,
                             "sample": f"B=8 sequences x T=35 of the C2 model through oracle.run_graph_step in {dt:.1f} s"}
    except Exception as e:  # threadpoolctl missing: report why
        res["c2_1thread"] = {"unavailable": str(e)[:120]}
    tp = pg.treelstm_program(V=20000, E=300, H=300, C=2, B=25, lr=0.05)
    state = gen.uniform_params(tp, 1, 0.05)
    forest = list(gen.sst_forest(gen.SEED_C3, 0, 25, 20000))
    t0 = time.perf_counter()
    r = I.run_graph_step(tp, forest, state)
    dt = time.perf_counter() - t0
    assert r.status == I.OK
    res["c3_b25"] = {"value": 25 / dt, "unit": "sentences/s", "cores": _blas_threads(),
                     "sample": f"one C3 step (B=25 trees, H=E=300) through oracle.run_graph_step in {dt:.2f} s"}
    return res


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # bounded per-step sample: B=8 sequences x T tokens of the C2 model, T sized (by timing a 1-token
    # sample) so the whole --steps K --warmup W run takes about two minutes
    B = 8
    t1 = oracle_sample(B, 1)
    T = int(max(1, min(35, 120.0 / max(1, args.steps + args.warmup) / max(t1, 1e-3))))
    for _ in range(args.warmup):
        oracle_sample(B, T)
    times = [oracle_sample(B, T) for _ in range(args.steps)]
    tot = sum(times)
    v = args.steps * B * T / 35.0 / tot
    cb = {"value": v, "unit": "samples/s", "cores": _blas_threads(), "kind": "oracle",
          "sample": f"each step: oracle.run_graph_step on B={B} sequences x T={T} tokens of the C2 model; "
                    f"value in 35-token sequence equivalents"}
    emit({"impl": "reference", "metric": BASELINE_METRIC, "value": v, "unit": "samples/s",
                      "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                      "ms_per_step": 1000 * tot / args.steps, "higher_is_better": True,
                      "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                      "config": {"workload": WORKLOADS["c2"]["desc"], "global_batch": 64, "seq_len": 35,
                                 "parallelism": "none (host oracle)"},
                      "cpu_baseline": cb,
                      "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})


# ----------------------------------------------------------------------------- extra measurements
def c4_extra(J, torch, stream, timed, K):
    """C4 on one GPU: samples/s, valid tokens/s, padded fraction, and host syncs per step of the
    graph path (1) against the imperative executor (one per control decision)."""
    B = 64
    prog = c4_program(B)
    g = J.Graph(prog)
    ws = g.new_workspace()
    state = [torch.tensor(x, device="cuda") for x in gen.uniform_params(prog, 1, 0.05)]
    one = np.ones(1, np.int32)
    nb = 8
    bs = [list(gen.c4_batch(gen.SEED_C4, k, B, 10000)) + [one] for k in range(nb)]
    dev = [[torch.tensor(a, device="cuda") for a in b] for b in bs]
    loss = torch.zeros(1, device="cuda")
    for k in range(3):
        g.run(dev[k], state, ws, outs=[loss], stream=stream)
    Kc = max(nb, (K // nb) * nb)
    c0 = g.counters()
    ms = timed(lambda k: g.run(dev[k % nb], state, ws, outs=[loss], stream=stream), Kc) / Kc
    c1 = g.counters()
    valid = np.mean([int(b[2].sum()) for b in bs])
    width = np.mean([b[0].shape[1] for b in bs])
    st_i = [s.clone() for s in state]
    ci0 = g.counters()
    ms_i = timed(lambda k: g.run_imperative(dev[k], st_i, ws, outs=[loss], stream=stream), 2) / 2
    ci1 = g.counters()
    J.dev_profile(g, True)
    timed(lambda k: g.run(dev[k % nb], state, ws, outs=[loss], stream=stream), nb)
    ph = J.dev_phase_report(g)
    J.dev_profile(g, False)
    return {"samples_per_s": B * 1000.0 / ms, "valid_tokens_per_s": valid * 1000.0 / ms, "ms_per_step": ms,
            "mean_width": float(width), "padded_fraction": float(1.0 - valid / (B * width)),
            "graph_host_syncs_per_step": (c1["host_syncs"] - c0["host_syncs"]) / Kc,
            "graph_launches_per_step": (c1["launches"] - c0["launches"]) / Kc,
            "imperative_ms_per_step": ms_i,
            "imperative_host_syncs_per_step": (ci1["host_syncs"] - ci0["host_syncs"]) / 2,
            "imperative_launches_per_step": (ci1["launches"] - ci0["launches"]) / 2,
            "phases_ms_per_step": {n: round(v[0] / nb, 4) for n, v in ph.items()},
            "step_flop_frac_of_sustained": lm_flops_per_sample(10000, 650, 650, 2, 1) * valid /
                                           (ms * 1e-3) / 1e12 / peaks().get("bf16_tflops_sustained", 1400.0),
            "workload": "C4: C2 model, W ~ U{5..64}, lengths ~ U{1..W} (one row = W), B=64, seed 1815; "
                        "8 batches cycled; FLOPs counted on valid tokens"}


def extras(J, torch, g, ws, state, dev_batches, stream, timed, args, world, rank, ms_step):
    """TreeLSTM (C3) throughput, the imperative baseline (Table 3 "Imp."), assertion overhead
    (strip_asserts A/B) and the C5 speculation-failure stress, all on this rank's GPU."""
    out = {}
    K = max(3, min(args.steps, 40))
    B, T = 64, 35
    prog = c2_program(B)
    # --- guard overhead: same graph without RUNTIME AssertOps, interleaved A/B
    g0 = J.Graph(prog, world_size=world, rank=rank, nccl_id=getattr(g, "_nccl_id", None)) if world == 1 else None
    if g0 is not None:
        gs = J.Graph(prog, strip_asserts=True)
        ws_s = gs.new_workspace()
        st_s = [s.clone() for s in state]
        loss = torch.zeros(1, device="cuda")
        ab = {"with": [], "without": []}
        for rep in range(5):
            for name, gg, w, s in (("with", g, ws, state), ("without", gs, ws_s, st_s)):
                for k in range(2):
                    gg.run(dev_batches[k], s, w, outs=[loss], stream=stream)
                ab[name].append(timed(lambda k: gg.run(dev_batches[k % len(dev_batches)], s, w, outs=[loss],
                                                       stream=stream), K) / K)
        w_ms, wo_ms = statistics.median(ab["with"]), statistics.median(ab["without"])
        out["guard_overhead"] = {"ms_with_asserts": w_ms, "ms_without": wo_ms, "overhead": w_ms / wo_ms - 1.0,
                                 "method": f"C2, strip_asserts A/B, interleaved, median of 5 x {K} steps "
                                           "(noise ~ +-2%; the runtime guards run inside the step's first launch, phases_ms_per_step['init'])"}
    # --- imperative per-op executor on the same workload (the paper's "Imp." column)
    if world == 1:
        loss = torch.zeros(1, device="cuda")
        st_i = [s.clone() for s in state]
        c0 = g.counters()
        g.run_imperative(dev_batches[0], st_i, ws_i := torch.zeros(g.workspace_bytes, dtype=torch.uint8, device="cuda"),
                         outs=[loss], stream=stream)
        c1 = g.counters()
        KI = 3
        ms_i = timed(lambda k: g.run_imperative(dev_batches[k % len(dev_batches)], st_i, ws_i, outs=[loss],
                                                stream=stream), KI) / KI
        c2 = g.counters()
        out["imperative"] = {"samples_per_s": B * 1000.0 / ms_i, "ms_per_step": ms_i,
                             "launches_per_step": (c2["launches"] - c1["launches"]) // KI,
                             "host_syncs_per_step": (c2["host_syncs"] - c1["host_syncs"]) / KI,
                             "graph_speedup": ms_i / ms_step}
        del ws_i
        # --- C5: 10% of batches violate an assumption and fall back to the imperative path
        r = gen.rng(gen.SEED_C5)
        nb = 200
        viol = r.random(nb) < 0.10
        viol[0] = True
        kinds = ["dtype", "shape", "tag", "trip"]
        st5 = [s.clone() for s in state]
        tag_slot = prog.slot_index("tag")
        ws5 = torch.zeros(g.workspace_bytes, dtype=torch.uint8, device="cuda")
        loss = torch.zeros(1, device="cuda")
        aborts = {k: [] for k in kinds}
        fb = {k: [] for k in kinds}
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        nv = 0
        for k in range(nb):
            tok, tgt, ln, tr = dev_batches[k % len(dev_batches)]
            if viol[k]:
                kind = kinds[nv % 4]
                nv += 1
                if kind == "dtype":
                    a = [tok.long(), tgt, ln, tr]
                elif kind == "shape":
                    a = [tok[:B - 1].contiguous(), tgt[:B - 1].contiguous(), ln[:B - 1].contiguous(), tr]
                elif kind == "tag":
                    st5[tag_slot].zero_()
                    a = [tok, tgt, ln, tr]
                else:
                    l2 = ln.clone(); l2[3] = T - 1
                    a = [tok, tgt, l2, tr]
                ta = time.perf_counter()
                s, f = g.run(a, st5, ws5, outs=[loss], stream=stream)
                aborts[kind].append(1000 * (time.perf_counter() - ta))
                if s == J.ASSUMPTION_FAILED:   # fallback to the imperative executor
                    fb[kind].append(J.STATUS_NAMES[g.run_imperative(a, st5, ws5, outs=[loss], stream=stream)])
            else:
                g.run([tok, tgt, ln, tr], st5, ws5, outs=[loss], stream=stream)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        out["c5_stress"] = {"batches": nb, "violations": int(viol.sum()),
                            "blended_samples_per_s": nb * B / dt,
                            "abort_latency_ms": {k: (statistics.median(v) if v else None) for k, v in aborts.items()},
                            "fallback_status": fb,
                            "note": "wall clock incl. the host syncs of the imperative fallbacks"}
        del ws5
        # --- C5 through the graph cache + relaxation driver (NEXT-1): the same violation stream;
        # assumptions that break twice are relaxed and their batches return to the device path
        sess = J.Session(prog)
        st5 = [s.clone() for s in state]
        paths = {"graph": 0, "imperative": 0}
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        nv = 0
        for k in range(nb):
            tok, tgt, ln, tr = dev_batches[k % len(dev_batches)]
            a = [tok, tgt, ln, tr]
            if viol[k]:
                kind = kinds[nv % 4]
                nv += 1
                if kind == "dtype":
                    a = [tok.long(), tgt, ln, tr]
                elif kind == "shape":
                    a = [tok[:B - 1].contiguous(), tgt[:B - 1].contiguous(), ln[:B - 1].contiguous(), tr]
                elif kind == "tag":
                    st5[tag_slot].zero_()
                else:
                    l2 = ln.clone(); l2[3] = T - 1
                    a = [tok, tgt, l2, tr]
            s, info = sess.step(a, st5, outs=[loss], stream=stream)
            paths[info["path"]] += 1
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        sst = sess.stats()
        out["c5_stress_session"] = {
            "batches": nb, "violations": int(viol.sum()), "blended_samples_per_s": nb * B / dt,
            "paths": paths, "misses": sst["misses"], "aborts": sst["aborts"], "generated": sst["generated"],
            "entries": [{k: e[k] for k in ("id", "active", "device", "hits", "origin")} for e in sst["entries"]],
            "note": "janus_session_step: cache lookup, imperative fallback in the same call, relax after 2 "
                    "failures of one assumption (TRIP_COUNT -> device While, TYPE_TAG -> device Switch); "
                    "the first relaxed graph's build and workspace allocation are inside the timed loop"}
        del sess
        # --- C4: data-dependent trip counts on the device (While + RANGE guard), SURVEY §8(d)
        out["c4"] = c4_extra(J, torch, stream, timed, K)
        # --- the data-parallel step on a 1-rank communicator (force_dp): NCCL allreduce of the
        # gradient arena vs the reduction fused into the weight-gradient GEMM epilogue (NEXT-3)
        dp1 = {}
        for name, kw in (("nccl_allreduce", {}), ("fused_epilogue", {"fused_allreduce": True})):
            gp = J.Graph(prog, force_dp=True, no_dp_overlap=True, **kw)
            wsp = gp.new_workspace()
            stp = [s.clone() for s in state]
            lossp = torch.zeros(1, device="cuda")
            for k in range(3):
                gp.run(dev_batches[k % len(dev_batches)], stp, wsp, outs=[lossp], stream=stream)
            msp = timed(lambda k: gp.run(dev_batches[k % len(dev_batches)], stp, wsp, outs=[lossp], stream=stream), K) / K
            dp1[name] = {"samples_per_s": B * 1000.0 / msp, "ms_per_step": msp}
            del wsp, gp
        out["dp_1rank"] = dict(dp1, note="force_dp on one GPU: the collective sequence runs on a 1-rank "
                                         "communicator (no NVLink traffic); measures the protocol's own cost")
        # --- the Zaremba regularised LM (NEXT-4; [51] via P:312, PTB medium = the C2 shape): dropout
        # 0.5 on every non-recurrent connection, Philox masks keyed per step (layers run serially)
        pd = pg.lstm_lm_program(V=10000, E=650, H=650, L=2, B=B, T=35, lr=1.0, dropout=0.5, training_flag=True)
        gd = J.Graph(pd)
        wsd = gd.new_workspace()
        std = [s.clone() for s in state]
        loss = torch.zeros(1, device="cuda")
        keys = [torch.tensor([k, 2024], dtype=torch.int32, device="cuda") for k in range(4)]
        for k in range(3):
            gd.run(dev_batches[k % len(dev_batches)] + [keys[k % 4]], std, wsd, outs=[loss], stream=stream)
        ms_d = timed(lambda k: gd.run(dev_batches[k % len(dev_batches)] + [keys[k % 4]], std, wsd, outs=[loss],
                                      stream=stream), K) / K
        out["c2_dropout"] = {"samples_per_s": B * 1000.0 / ms_d, "ms_per_step": ms_d,
                             "workload": "Zaremba medium LM (C2 shape: 2 x 650, V=10000, T=35, B=64), dropout "
                                         "0.5 on the non-recurrent connections, Philox4x32-10 masks"}
        del wsd, gd
        # --- TreeRNN (Table 2) on the same SST-shaped forests, B=25, H=E=300
        tp = pg.treernn_program(V=20000, H=300, C=2, B=25, lr=0.05)
        gr = J.Graph(tp)
        wsr = gr.new_workspace()
        str_ = [torch.tensor(x, device="cuda") for x in gen.uniform_params(tp, 1, 0.05)]
        forests = [[torch.tensor(a, device="cuda") for a in gen.sst_forest(gen.SEED_C3, k, 25, 20000)]
                   for k in range(4)]
        for k in range(3):
            gr.run(forests[k % 4], str_, wsr, stream=stream)
        ms_r = timed(lambda k: gr.run(forests[k % 4], str_, wsr, stream=stream), K) / K
        st_i = [x.clone() for x in str_]
        gr.run_imperative(forests[0], st_i, wsr, stream=stream)
        ms_ri = timed(lambda k: gr.run_imperative(forests[k % 4], st_i, wsr, stream=stream), 2) / 2
        out["treernn_b25"] = {"sentences_per_s": 25 * 1000.0 / ms_r, "ms_per_step": ms_r,
                              "imperative_sentences_per_s": 25 * 1000.0 / ms_ri,
                              "workload": "TreeRNN (Socher et al. [37]) on C3 SST-shaped forests, B=25, "
                                          "H=E=300, V=20000, <=64 leaves",
                              "paper_context": "JANUS TreeRNN 988.72 sentences/s on CPUs (P:365)"}
        del wsr, gr
        # --- C3 TreeLSTM
        for Bt in (25, 256):
            tp = pg.treelstm_program(V=20000, E=300, H=300, C=2, B=Bt, lr=0.05)
            gt = J.Graph(tp)
            wst = gt.new_workspace()
            stt = [torch.tensor(x, device="cuda") for x in gen.uniform_params(tp, 1, 0.05)]
            forests = [[torch.tensor(a, device="cuda") for a in gen.sst_forest(gen.SEED_C3, k, Bt, 20000)]
                       for k in range(4)]
            for k in range(3):
                gt.run(forests[k % 4], stt, wst, stream=stream)
            ms_t = timed(lambda k: gt.run(forests[k % 4], stt, wst, stream=stream), K) / K
            J.dev_profile(gt, True)
            timed(lambda k: gt.run(forests[k % 4], stt, wst, stream=stream), K)
            ph = J.dev_phase_report(gt)
            J.dev_profile(gt, False)
            out[f"treelstm_b{Bt}"] = {"sentences_per_s": Bt * 1000.0 / ms_t, "ms_per_step": ms_t,
                                      "phases_ms_per_step": {n: round(v[0] / K, 4) for n, v in ph.items()},
                                      "workload": f"C3 SST-shaped forests, B={Bt}, H=E=300, V=20000, <=64 leaves"}
            if Bt == 25:   # ablation (Figure 7): the imperative executor on the same forests
                st_i = [x.clone() for x in stt]
                gt.run_imperative(forests[0], st_i, wst, stream=stream)
                ms_ti = timed(lambda k: gt.run_imperative(forests[k % 4], st_i, wst, stream=stream), 2) / 2
                # -PARL: the same device program with the level loops on one CTA (no parallelism
                # across the nodes of a level)
                gt1 = J.Graph(tp, tree_grid=1)
                gt1.run(forests[0], st_i, wst, stream=stream)
                ms_t1 = timed(lambda k: gt1.run(forests[k % 4], st_i, wst, stream=stream), 3) / 3
                del gt1
                c3_abl = {"IMP": Bt * 1000.0 / ms_ti, "graph_one_cta_per_level": Bt * 1000.0 / ms_t1,
                          "graph_level_batched": Bt * 1000.0 / ms_t}
            del wst
        # --- Figure 7 ablation on B200, stacked as in the paper: each arm adds one
        # optimisation to the previous one. Same C2 batches, same state, samples/s.
        #   BASE  : speculative graph, loop as a device While, runtime width (SHAPE_MATCH (B, ?),
        #           RANGE lengths in [1, 64]: planned for any width <= 64), stacked layers serial
        #   +SPCN : the same While graph specialised to the profiled shape (B, 35)
        #   +UNRL : unrolled to the asserted trip count (TRIP_COUNT = 35), layers serial
        #   +PARL : + the two-layer wavefront (layer 1's step t beside layer 0's step t+1, fwd and
        #           bwd): the product graph
        import copy
        from workloads.programs import Assumption

        def arm(program, serial):
            g_ = J.Graph(program, serial_layers=serial)
            ws_ = g_.new_workspace()
            st_ = [s.clone() for s in state]
            loss_ = torch.zeros(1, device="cuda")
            for k in range(3):
                st_r, _ = g_.run(dev_batches[k % len(dev_batches)], st_, ws_, outs=[loss_], stream=stream)
                assert st_r == J.OK, (program.name, st_r)
            ms_ = timed(lambda k: g_.run(dev_batches[k % len(dev_batches)], st_, ws_, outs=[loss_], stream=stream), K) / K
            del ws_, g_
            return B * 1000.0 / ms_

        p_rt = pg.lstm_lm_program(V=10000, E=650, H=650, L=2, B=B, T=64, lr=1.0, speculate="while",
                                  training_flag=True)              # runtime width <= 64
        p_sp = copy.deepcopy(c2_program(B, speculate="while"))     # width specialised to 35
        p_sp.assumptions = [Assumption(a.id, a.kind, a.mode, a.target, dims=(B, 35))
                            if a.kind == "SHAPE_MATCH" and a.target in (0, 1) else a for a in p_sp.assumptions]
        c2_abl = {"IMP": out["imperative"]["samples_per_s"], "BASE": arm(p_rt, True), "+SPCN": arm(p_sp, True),
                  "+UNRL": arm(prog, True), "+PARL": B * 1000.0 / ms_step}
        out["ablation_fig7"] = {
            "c2_samples_per_s": c2_abl,
            "c2_while_runtime_width_wavefront": arm(p_rt, False),
            "c3_b25_sentences_per_s": c3_abl,
            "note": "stacked arms (P:384-390): IMP = janus_run_imperative (one launch per op, host-side "
                    "control flow); BASE = device While, runtime width (B, ?) planned for W <= 64, layers "
                    "serial; +SPCN = the While graph specialised to (B, 35); +UNRL = unrolled (TRIP_COUNT), "
                    "layers serial; +PARL = + the two-layer wavefront (the product). C3: "
                    "graph_one_cta_per_level = level loops on one CTA (-PARL)"}
    return out


# ----------------------------------------------------------------------------- main arm
_JSON_FD = None


def emit(obj):
    """The one JSON line of the run, on the process's original stdout."""
    line = (json.dumps(obj) + "\n").encode()
    if _JSON_FD is None:
        sys.stdout.write(line.decode())
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, line)


def main():
    # stdout carries exactly one JSON line: everything else written to file descriptor 1 — NCCL's
    # version banner and NCCL_DEBUG output, any native print — is sent to stderr
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--impl", default="janus", choices=["janus", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip TreeLSTM / imperative / guard / C5 keys")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1812_01329_b200 import janus as J

    wl = WORKLOADS[args.workload]
    B, T = wl["B"], wl["T"]
    prog = c2_program(B) if args.workload == "c2" else c4_program(B)
    nccl_id = J.nccl_unique_id_bcast(rank, world) if world > 1 else None
    g = J.Graph(prog, world_size=world, rank=rank, nccl_id=nccl_id)
    assert g.device_path, g.build_message
    ws = g.new_workspace()
    state = [torch.tensor(x, device="cuda") for x in gen.uniform_params(prog, 1, 0.05)]
    n_batches = 8
    one = np.ones(1, np.int32)   # training = 1 (the VALUE_EQ-speculated flag)
    if args.workload == "c2":
        batches = [[a[rank * B:(rank + 1) * B] for a in b] + [one]
                   for b in gen.lm_batches(gen.SEED_C2, B, T, 10000, n_batches, ranks=world)]
    else:   # every rank draws its own C4 batches (weak scaling)
        batches = [list(gen.c4_batch(gen.SEED_C4, k * world + rank, B, 10000)) + [one] for k in range(n_batches)]
    widths = [b[0].shape[1] for b in batches]
    valid = [int(b[2].sum()) for b in batches]
    dev_batches = [[torch.tensor(a, device="cuda") for a in b] for b in batches]
    host_batches = [[torch.tensor(a).pin_memory() for a in b] for b in batches]
    loss_d = torch.zeros(1, device="cuda")
    stream = torch.cuda.current_stream()

    def step(k, host=False, loss_out=None):
        a = host_batches[k % n_batches] if host else dev_batches[k % n_batches]
        st, fail = g.run(a, state, ws, outs=[loss_out if loss_out is not None else loss_d], stream=stream)
        if st != J.OK:
            raise RuntimeError(f"janus_run: {J.STATUS_NAMES[st]} {fail}")

    def timed(fn, K):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for k in range(K):
            fn(k)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    clk = Clocks(local).start()
    for k in range(args.warmup):
        step(k)
    t_wait = time.time()
    k = args.warmup
    while not clk.producing() and time.time() - t_wait < 3.0:  # keep the GPU busy until sampling
        step(k)
        k += 1
    torch.cuda.synchronize()
    c0 = g.counters()
    with clk:
        ms = timed(lambda k: step(k), args.steps)
    clk.stop()
    c1 = g.counters()
    launches = (c1["launches"] - c0["launches"]) // args.steps
    syncs = (c1["host_syncs"] - c0["host_syncs"]) / args.steps
    ms_step = ms / args.steps
    value = world * B * 1000.0 / ms_step

    # e2e: pinned host buffers in, loss out to host memory, every step, through janus_run
    loss_h = torch.zeros(1).pin_memory()
    for k in range(2):
        step(k, host=True, loss_out=loss_h)
    ms_e2e = timed(lambda k: step(k, host=True, loss_out=loss_h), args.steps)
    e2e = {"value": world * B * 1000.0 / (ms_e2e / args.steps), "unit": "samples/s",
           "h2d_bytes_per_step": int(np.mean([sum(a.numel() * 4 for a in hb) for hb in host_batches])),
           "d2h_bytes_per_step": 48}

    # per-phase device timing (separate pass of the same steps, CUDA events on the launch stream)
    J.dev_profile(g, True)
    timed(lambda k: step(k), args.steps)
    phases = J.dev_phase_report(g)
    J.dev_profile(g, False)
    pk = peaks()
    T = float(np.mean([widths[k % n_batches] for k in range(args.steps)]))  # C2: 35; C4: mean width
    TB = int(round(B * T))
    rows = []
    step_ms = sum(v[0] for v in phases.values()) / args.steps
    for name, (tot_ms, cnt) in phases.items():
        fl = gemm_flops(name, 10000, 650, 650, TB)
        rows.append((tot_ms / args.steps, name, cnt // args.steps, fl))
    rows.sort(reverse=True)
    peak = pk.get("bf16_tflops_sustained", pk.get("bf16_tflops"))
    peak_src = pk["source"] + " bf16_tflops_sustained (kernels timed inside the step)"
    ncu = {}
    try:
        with open(os.path.join(ROOT, "profiles", "r2e_ncu_traffic.json")) as f:
            ncu = json.load(f)
    except (OSError, ValueError):
        pass

    def traffic(key):
        d = ncu.get(key)
        return None if not d else d["dram_read_bytes"] + d["dram_write_bytes"]

    # the dominant kernel of the step: the backward recurrence (two launches, one per layer).
    # Algorithmic tensor work per launch: the (T-1) recurrent products dh_t = W_hh^T dz_{t+1},
    # 2 * B * 4H * H flops each; the launch is latency-bound (T dependent steps), see DESIGN.md.
    rec = [r for r in rows if r[1].startswith("rec_bwd")]
    rec_ms = sum(r[0] for r in rec)
    rec_n = sum(r[2] for r in rec)
    rec_avg = rec_ms / max(1, rec_n)
    wave = any(r[1] == "rec_bwd01" for r in rec)
    Hh = 650
    # per launch: the recurrent products dh_t = W_hh^T dz_{t+1} (T-1 per layer) and, in the
    # two-layer wavefront, the fused input dgrad W_ih1^T dz1_t (T of them), 2*B*4H*H flops each
    rec_fl = 2.0 * B * 4 * Hh * Hh * ((T - 1) * 2 + T if wave else (T - 1))
    rec_ach = rec_fl / (rec_avg * 1e-3) / 1e12 if rec_avg else None
    roofline = {"kernel": ("rec_bwd01 (lstm_rec_bwd_wf_kernel: both layers, K-split clusters)" if wave
                           else "rec_bwd (lstm_rec_bwd_ks_kernel, K-split clusters)"),
                "bound": "tensor",
                "achieved": rec_ach, "peak": peak, "unit": "TFLOP/s",
                "frac": rec_ach / peak if rec_ach else None, "traffic": traffic("rec_bwd"),
                "flops_per_launch": rec_fl, "avg_launch_ms": rec_avg,
                "step_period_us": rec_avg * 1000.0 / T,
                "peak_source": peak_src, "share_of_step": rec_ms / step_ms if step_ms else None,
                "traffic_source": "profiles/r2e_ncu_traffic.json (ncu --set full of one C2 step, dram read+write per launch; summary profiles/r2e_ncu_c2_summary.txt)",
                "note": "latency-bound: T=35 dependent steps per launch; the step period is the bound, not the tensor pipe"}
    gemms = [r for r in rows if r[3]]
    top = gemms[0] if gemms else rows[0]
    avg_ms = top[0] / max(1, top[2])
    achieved = top[3] / (avg_ms * 1e-3) / 1e12 if top[3] else None
    roofline_gemm = {"kernel": top[1], "bound": "tensor", "achieved": achieved, "peak": peak,
                     "unit": "TFLOP/s", "frac": achieved / peak if achieved else None,
                     "traffic": traffic("gemm_dec") if top[1] == "gemm_dec" else None,
                     "flops_per_launch": top[3], "avg_launch_ms": avg_ms, "peak_source": peak_src,
                     "share_of_step": top[0] / step_ms if step_ms else None}
    # algorithmic FLOPs of the step: per VALID token (C4's padded rows are work the method skips)
    vtok = float(np.mean([valid[k % n_batches] for k in range(args.steps)]))
    flops = lm_flops_per_sample(10000, 650, 650, 2, 1) * vtok
    out = {
        "metric": BASELINE_METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": wl["desc"], "global_batch": B * world, "seq_len": T,
                   "parallelism": f"dp{world}",
                   "l2": "no flush: the step's working set (~340 MB workspace + 79 MB params) exceeds the 126 MB L2"},
        "words_per_s": world * vtok * 1000.0 / ms_step,
        "step_tflops": flops * world / (ms_step * 1e-3) / 1e12 / world,
        "step_flop_frac_of_sustained": flops / (ms_step * 1e-3) / 1e12 / peak,
        "e2e": e2e, "gpu_launches": int(launches), "host_syncs_per_step": syncs,
        "roofline": roofline, "roofline_gemm": roofline_gemm,
        "phases_ms_per_step": {r[1]: round(r[0], 4) for r in rows},
        "paper_context": "JANUS LSTM (PTB, BS 20) 22.06k words/s on 1 TITAN Xp, fp32 (P:363) — other hardware/config",
    }
    if args.workload == "c4":
        out["c4"] = {"valid_tokens_per_s": world * vtok * 1000.0 / ms_step,
                     "mean_width": T, "padded_fraction": 1.0 - vtok / (B * T),
                     "host_syncs_per_step": syncs}
    out["clocks"] = clk.summary()
    if not args.no_extras and args.workload == "c2" and world == 1:  # the scaling runs time the headline only
        out.update(extras(J, torch, g, ws, state, dev_batches, stream, timed, args, world, rank, ms_step))
    if rank == 0 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline()
        if not args.no_extras and world == 1:
            out["cpu_baseline_modes"] = cpu_baseline_modes()
    if rank == 0:
        emit(out)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
