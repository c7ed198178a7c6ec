"""Thin ctypes binding of libjanus (include/janus.h, include/janus_dev.h).

Argument marshalling only: every step of the path runs inside libjanus's CUDA kernels. PyTorch
supplies device memory and streams. There is no CPU fallback: if the shared library is missing
the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import weakref

import numpy as np

from workloads import programs as pg

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, f"libjanus_{os.environ['JANUS_VARIANT']}.so" if os.environ.get("JANUS_VARIANT")
                        else "libjanus.so")  # JANUS_VARIANT: dev-only A/B builds (build.py)

OK, ASSUMPTION_FAILED, ERR_INVALID, ERR_UNSUPPORTED, ERR_RUNTIME, ERR_CUDA, ERR_NCCL, ERR_WORKSPACE = range(8)
STATUS_NAMES = ["OK", "ASSUMPTION_FAILED", "ERR_INVALID", "ERR_UNSUPPORTED", "ERR_RUNTIME",
                "ERR_CUDA", "ERR_NCCL", "ERR_WORKSPACE"]
PATH_GRAPH, PATH_IMPERATIVE = 0, 1
EV_HIT, EV_MISS, EV_ABORT, EV_IMPERATIVE_ENTRY = range(4)
EVENT_NAMES = ["HIT", "MISS", "ABORT", "IMPERATIVE_ENTRY"]
F32, BF16, I32, I64, U8 = range(5)


class JanusTensor(C.Structure):
    _fields_ = [("data", C.c_void_p), ("dtype", C.c_int32), ("ndim", C.c_int32),
                ("shape", C.c_int64 * 4), ("stride", C.c_int64 * 4)]


class JanusOp(C.Structure):
    _fields_ = [("kind", C.c_int32), ("func", C.c_int32), ("n_in", C.c_int32),
                ("in_node", C.c_int32 * 12), ("in_port", C.c_int32 * 12),
                ("iattr", C.c_int64 * 8), ("fattr", C.c_double * 2)]


class JanusAssumption(C.Structure):
    _fields_ = [("id", C.c_uint32), ("kind", C.c_int32), ("mode", C.c_int32), ("target", C.c_int32),
                ("dtype", C.c_int32), ("ndim", C.c_int32), ("dims", C.c_int64 * 4),
                ("lo", C.c_int64), ("hi", C.c_int64), ("value", C.c_int64),
                ("ref_arg", C.c_int32), ("ref_dim", C.c_int32)]


class JanusFailure(C.Structure):
    _fields_ = [("assumption_id", C.c_uint32), ("rank", C.c_int32), ("index", C.c_int64),
                ("observed", C.c_int64)]


class JanusBuildOpts(C.Structure):
    _fields_ = [("world_size", C.c_int32), ("rank", C.c_int32), ("nccl_id", C.c_uint8 * 128),
                ("gemm_dtype", C.c_int32), ("strip_asserts", C.c_int32),
                ("fail_assert_id", C.c_int32), ("serial_layers", C.c_int32), ("tree_grid", C.c_int32),
                ("force_dp", C.c_int32), ("no_dp_overlap", C.c_int32), ("fused_allreduce", C.c_int32)]


class JanusSessionOpts(C.Structure):
    _fields_ = [("fail_threshold", C.c_int32), ("cache_max", C.c_int32), ("reserved", C.c_int32 * 6)]


class JanusStepInfo(C.Structure):
    _fields_ = [("path", C.c_int32), ("event", C.c_int32), ("entry", C.c_int32), ("generated", C.c_int32),
                ("fail", JanusFailure), ("workspace_bytes", C.c_uint64)]


if not os.path.exists(LIB_PATH):
    raise ImportError(f"libjanus.so not built ({LIB_PATH}); run __graft_entry__.build()")
lib = C.CDLL(LIB_PATH)

EXPORTS = ["janus_graph_build", "janus_workspace_bytes", "janus_run", "janus_run_imperative",
           "janus_counters", "janus_describe", "janus_graph_destroy", "janus_status_str",
           "janus_abi_version", "janus_session_create", "janus_session_workspace_bytes",
           "janus_session_step", "janus_session_stats", "janus_session_destroy", "janus_relax",
           "janus_state_changed"]
DEV_EXPORTS = ["janus_dev_gemm_bf16", "janus_dev_gemm_bf16_splitk"]

_P = C.c_void_p
for _name, _res, _args in [
    ("janus_dev_gemm_bf16", C.c_int32, [C.c_int32, C.c_int32, C.c_int32, _P, C.c_int32, C.c_int32, _P,
                                        C.c_int32, C.c_int32, _P, C.c_int32, _P, _P, C.c_int32, _P]),
    ("janus_dev_gemm_bf16_splitk", C.c_int32, [C.c_int32, C.c_int32, C.c_int32, _P, C.c_int32, C.c_int32, _P,
                                               C.c_int32, C.c_int32, _P, C.c_int32, _P, _P, C.c_int32,
                                               C.c_int32, _P]),
]:
    if hasattr(lib, _name):
        f = getattr(lib, _name)
        f.restype, f.argtypes = _res, _args


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def dev_gemm_bf16(M, N, K, A, lda, a_mn, B, ldb, b_mn, Cout, ldc, bias_col=None, bias_row=None,
                  accumulate=False, stream=None):
    r = lib.janus_dev_gemm_bf16(M, N, K, _ptr(A), lda, int(a_mn), _ptr(B), ldb, int(b_mn), _ptr(Cout),
                                ldc, _ptr(bias_col), _ptr(bias_row), int(accumulate), _stream(stream))
    if r != 0:
        raise RuntimeError(f"janus_dev_gemm_bf16 failed with cuda error {r}")


def dev_gemm_bf16_splitk(M, N, K, A, lda, a_mn, B, ldb, b_mn, Cout, ldc, bias_col=None, bias_row=None,
                         accumulate=False, splits=0, stream=None):
    r = lib.janus_dev_gemm_bf16_splitk(M, N, K, _ptr(A), lda, int(a_mn), _ptr(B), ldb, int(b_mn), _ptr(Cout),
                                       ldc, _ptr(bias_col), _ptr(bias_row), int(accumulate), int(splits),
                                       _stream(stream))
    if r != 0:
        raise RuntimeError(f"janus_dev_gemm_bf16_splitk failed with cuda error {r}")


# ----------------------------------------------------------------------------------- step ABI
_sigs = {
    "janus_graph_build": (C.c_int, [C.POINTER(JanusOp), C.c_int32, C.POINTER(JanusAssumption), C.c_int32,
                                    C.POINTER(JanusBuildOpts), C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]),
    "janus_workspace_bytes": (C.c_int, [C.c_void_p, C.POINTER(C.c_size_t)]),
    "janus_run": (C.c_int, [C.c_void_p, C.POINTER(JanusTensor), C.c_int32, C.POINTER(JanusTensor), C.c_int32,
                            C.POINTER(JanusTensor), C.c_int32, JanusTensor, C.c_void_p, C.POINTER(JanusFailure)]),
    "janus_run_imperative": (C.c_int, [C.c_void_p, C.POINTER(JanusTensor), C.c_int32, C.POINTER(JanusTensor),
                                       C.c_int32, C.POINTER(JanusTensor), C.c_int32, JanusTensor, C.c_void_p]),
    "janus_counters": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "janus_describe": (C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t]),
    "janus_graph_destroy": (None, [C.c_void_p]),
    "janus_status_str": (C.c_char_p, [C.c_int]),
    "janus_abi_version": (C.c_int32, []),
    "janus_state_changed": (C.c_int, []),
    "janus_session_create": (C.c_int, [C.POINTER(JanusOp), C.c_int32, C.POINTER(JanusAssumption), C.c_int32,
                                       C.POINTER(JanusBuildOpts), C.POINTER(JanusSessionOpts),
                                       C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]),
    "janus_session_workspace_bytes": (C.c_int, [C.c_void_p, C.POINTER(C.c_size_t)]),
    "janus_session_step": (C.c_int, [C.c_void_p, C.POINTER(JanusTensor), C.c_int32, C.POINTER(JanusTensor),
                                     C.c_int32, C.POINTER(JanusTensor), C.c_int32, JanusTensor, C.c_void_p,
                                     C.POINTER(JanusStepInfo)]),
    "janus_session_stats": (C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t]),
    "janus_session_destroy": (None, [C.c_void_p]),
    "janus_relax": (C.c_int, [C.POINTER(JanusAssumption), C.POINTER(JanusTensor), C.POINTER(JanusAssumption),
                              C.POINTER(C.c_int32)]),
}
for _n, (_r, _a) in _sigs.items():
    _f = getattr(lib, _n)
    _f.restype, _f.argtypes = _r, _a

_TORCH_DT = None


def _dtcode(t):
    global _TORCH_DT
    import torch
    if _TORCH_DT is None:
        _TORCH_DT = {torch.float32: F32, torch.bfloat16: BF16, torch.int32: I32, torch.int64: I64,
                     torch.uint8: U8}
    return _TORCH_DT[t.dtype]


def to_jt(t):
    """torch tensor (cuda or pinned cpu) or numpy array -> JanusTensor (borrowed pointer)."""
    jt = JanusTensor()
    if isinstance(t, np.ndarray):
        assert t.flags["C_CONTIGUOUS"]
        jt.data = t.ctypes.data
        jt.dtype = {np.dtype(np.float32): F32, np.dtype(np.int32): I32, np.dtype(np.int64): I64,
                    np.dtype(np.uint8): U8}[t.dtype]
        shape, strides = t.shape, [s // t.itemsize for s in t.strides]
    else:
        assert t.is_contiguous()
        jt.data = t.data_ptr()
        jt.dtype = _dtcode(t)
        shape, strides = tuple(t.shape), t.stride()
    jt.ndim = len(shape)
    for k, (s, st) in enumerate(zip(shape, strides)):
        jt.shape[k] = s
        jt.stride[k] = st
    return jt


def _jt_array(ts):
    arr = (JanusTensor * max(1, len(ts)))()
    for k, t in enumerate(ts):
        arr[k] = to_jt(t)
    return arr


def marshal_ops(program):
    ops = (JanusOp * len(program.ops))()
    for k, o in enumerate(program.ops):
        j = ops[k]
        j.kind = pg.OP_CODE[o.kind]
        j.func = o.func
        j.n_in = len(o.ins)
        for m, (n, p) in enumerate(o.ins):
            j.in_node[m] = n
            j.in_port[m] = p
        for m, v in enumerate(o.i):
            j.iattr[m] = int(v)
        for m, v in enumerate(o.f):
            j.fattr[m] = float(v)
    return ops


def marshal_assumptions(program):
    arr = (JanusAssumption * max(1, len(program.assumptions)))()
    for k, a in enumerate(program.assumptions):
        j = arr[k]
        j.id = a.id
        j.kind = pg.ASM_CODE[a.kind]
        j.mode = a.mode
        j.target = a.target
        j.dtype = a.dtype
        j.ndim = len(a.dims)
        for m, d in enumerate(a.dims):
            j.dims[m] = d
        j.lo, j.hi, j.value = a.lo, a.hi, a.value
        j.ref_arg, j.ref_dim = a.ref_arg, a.ref_dim
    return arr


class JanusError(RuntimeError):
    pass


_seen_state = {}   # id(tensor) -> (weakref, _version) at the last library call


def _note_state(state):
    """janus_state_changed when a state tensor was written outside the library since the last
    call (torch bumps _version on every in-place write; a different tensor object counts too): the
    LM step then re-casts its bf16 operand copies instead of trusting the ones its commit refreshed."""
    changed = False
    for t in state:
        v = getattr(t, "_version", None)
        if v is None:
            changed = True
            continue
        e = _seen_state.get(id(t))
        if e is None or e[0]() is not t or e[1] != v:
            changed = True
            _seen_state[id(t)] = (weakref.ref(t), v)
    if changed:
        lib.janus_state_changed()
        if len(_seen_state) > 4096:
            for k in [k for k, e in _seen_state.items() if e[0]() is None]:
                del _seen_state[k]


class Graph:
    """A speculatively specialised graph (janus_graph_build) for one Program."""

    def __init__(self, program, gemm=None, world_size=1, rank=0, nccl_id=None, strip_asserts=False,
                 fail_assert_id=-1, **ablation):
        """ablation: serial_layers, tree_grid, force_dp, no_dp_overlap, fused_allreduce (janus_build_opts)."""
        self.program = program
        opts = _build_opts(program, gemm, world_size, rank, nccl_id, strip_asserts, fail_assert_id, **ablation)
        self._ops = marshal_ops(program)
        self._asms = marshal_assumptions(program)
        h = C.c_void_p()
        err = C.create_string_buffer(1024)
        r = lib.janus_graph_build(self._ops, len(program.ops), self._asms, len(program.assumptions),
                                  C.byref(opts), C.byref(h), err, 1024)
        if r not in (OK, ERR_UNSUPPORTED) or not h.value:
            raise JanusError(f"janus_graph_build: {STATUS_NAMES[r]}: {err.value.decode()}")
        self.h = h
        self.device_path = r == OK
        self.build_message = err.value.decode()
        n = C.c_size_t()
        lib.janus_workspace_bytes(self.h, C.byref(n))
        self.workspace_bytes = n.value

    def __del__(self):
        if getattr(self, "h", None) and lib is not None:  # (module globals are gone at interpreter exit)
            lib.janus_graph_destroy(self.h)
            self.h = None

    def new_workspace(self, device="cuda"):
        import torch
        return torch.zeros(max(16, self.workspace_bytes), dtype=torch.uint8, device=device)

    def run(self, args, state, workspace, outs=(), stream=None):
        """janus_run: returns (status, failure dict or None)."""
        _note_state(state)
        a, s, o = _jt_array(args), _jt_array(state), _jt_array(outs)
        f = JanusFailure()
        r = lib.janus_run(self.h, a, len(args), s, len(state), o, len(outs), to_jt(workspace),
                          _stream(stream), C.byref(f))
        fail = None
        if r == ASSUMPTION_FAILED:
            fail = dict(assumption_id=f.assumption_id, rank=f.rank, index=f.index, observed=f.observed)
        return r, fail

    def run_imperative(self, args, state, workspace, outs=(), stream=None):
        _note_state(state)
        a, s, o = _jt_array(args), _jt_array(state), _jt_array(outs)
        return lib.janus_run_imperative(self.h, a, len(args), s, len(state), o, len(outs),
                                        to_jt(workspace), _stream(stream))

    def counters(self):
        l, h, a = C.c_uint64(), C.c_uint64(), C.c_uint64()
        lib.janus_counters(self.h, C.byref(l), C.byref(h), C.byref(a))
        return dict(launches=l.value, host_syncs=h.value, aborts=a.value)

    def describe(self):
        buf = C.create_string_buffer(4096)
        lib.janus_describe(self.h, buf, 4096)
        return buf.value.decode()


# ----------------------------------------------------------------------------------- dev hooks
lib.janus_dev_profile.restype, lib.janus_dev_profile.argtypes = C.c_int32, [C.c_void_p, C.c_int32]
lib.janus_dev_phase_report.restype = C.c_int32
lib.janus_dev_phase_report.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t]


lib.janus_nccl_unique_id.restype = C.c_int32
lib.janus_nccl_unique_id.argtypes = [C.c_void_p]


def _build_opts(program, gemm=None, world_size=1, rank=0, nccl_id=None, strip_asserts=False, fail_assert_id=-1,
                serial_layers=False, tree_grid=0, force_dp=False, no_dp_overlap=False, fused_allreduce=False):
    opts = JanusBuildOpts()
    opts.fused_allreduce = int(fused_allreduce)
    opts.serial_layers, opts.tree_grid = int(serial_layers), int(tree_grid)
    opts.force_dp, opts.no_dp_overlap = int(force_dp), int(no_dp_overlap)
    opts.world_size, opts.rank = world_size, rank
    if nccl_id is not None:
        for k, b in enumerate(bytes(nccl_id)[:128]):
            opts.nccl_id[k] = b
    gemm = gemm or program.meta.get("gemm", "bf16")
    opts.gemm_dtype = F32 if gemm == "f32" else BF16
    opts.strip_asserts = int(strip_asserts)
    opts.fail_assert_id = fail_assert_id
    return opts


class Session:
    """Graph cache + relaxation driver (janus_session_*): every step dispatches to a cached
    specialised graph, falls back to the imperative executor on a miss or an AssertOp failure, and
    regenerates graphs whose assumptions repeatedly break. Owns a device workspace (torch) that
    grows when the library asks for more (JANUS_ERR_WORKSPACE)."""

    def __init__(self, program, gemm=None, fail_threshold=2, cache_max=0, strip_asserts=False,
                 fail_assert_id=-1, device="cuda"):
        self.program = program
        opts = _build_opts(program, gemm, strip_asserts=strip_asserts, fail_assert_id=fail_assert_id)
        so = JanusSessionOpts()
        so.fail_threshold, so.cache_max = fail_threshold, cache_max
        self._ops = marshal_ops(program)
        self._asms = marshal_assumptions(program)
        h = C.c_void_p()
        err = C.create_string_buffer(1024)
        r = lib.janus_session_create(self._ops, len(program.ops), self._asms, len(program.assumptions),
                                     C.byref(opts), C.byref(so), C.byref(h), err, 1024)
        if r not in (OK, ERR_UNSUPPORTED) or not h.value:
            raise JanusError(f"janus_session_create: {STATUS_NAMES[r]}: {err.value.decode()}")
        self.h = h
        self.device = device
        self.workspace = None

    def __del__(self):
        if getattr(self, "h", None) and lib is not None:
            lib.janus_session_destroy(self.h)
            self.h = None

    def workspace_bytes(self):
        n = C.c_size_t()
        lib.janus_session_workspace_bytes(self.h, C.byref(n))
        return n.value

    def step(self, args, state, outs=(), stream=None):
        """janus_session_step: returns (status, info dict)."""
        import torch
        _note_state(state)
        a, s, o = _jt_array(args), _jt_array(state), _jt_array(outs)
        info = JanusStepInfo()
        for _ in range(4):
            if self.workspace is None:
                self.workspace = torch.zeros(max(16, self.workspace_bytes()), dtype=torch.uint8, device=self.device)
            r = lib.janus_session_step(self.h, a, len(args), s, len(state), o, len(outs), to_jt(self.workspace),
                                       _stream(stream), C.byref(info))
            if r != ERR_WORKSPACE:
                break
            self.workspace = None   # grow (the library asked for info.workspace_bytes)
            self.workspace = torch.zeros(int(info.workspace_bytes), dtype=torch.uint8, device=self.device)
        f = info.fail
        return r, dict(path="graph" if info.path == PATH_GRAPH else "imperative", event=EVENT_NAMES[info.event],
                       entry=info.entry, generated=info.generated,
                       fail=dict(assumption_id=f.assumption_id, rank=f.rank, index=f.index, observed=f.observed),
                       workspace_bytes=int(info.workspace_bytes))

    def stats(self):
        import json
        buf = C.create_string_buffer(1 << 16)
        if lib.janus_session_stats(self.h, buf, 1 << 16) != OK:
            raise JanusError("janus_session_stats")
        return json.loads(buf.value.decode())


def relax(assumption, observed=None):
    """janus_relax on one programs.Assumption; observed = (dtype code, shape tuple) or None.
    Returns the relaxed JanusAssumption, or None when the assumption is dropped."""
    src = marshal_assumptions(type("P", (), {"assumptions": [assumption]}))
    jt = None
    if observed is not None:
        jt = JanusTensor()
        jt.dtype, shape = observed
        jt.ndim = len(shape)
        for k, d in enumerate(shape):
            jt.shape[k] = d
    out = JanusAssumption()
    dropped = C.c_int32()
    r = lib.janus_relax(src, C.byref(jt) if jt is not None else None, C.byref(out), C.byref(dropped))
    if r != OK:
        raise JanusError(f"janus_relax: {STATUS_NAMES[r]}")
    return None if dropped.value else out


def nccl_unique_id():
    buf = (C.c_uint8 * 128)()
    if lib.janus_nccl_unique_id(buf) != 0:
        raise JanusError("ncclGetUniqueId failed")
    return bytes(buf)


def broadcast_bytes(data, rank, src=0):
    """Broadcast a bytes object from `src` over the default torch.distributed group (any backend)."""
    import torch.distributed as dist
    obj = [data if rank == src else None]
    dist.broadcast_object_list(obj, src=src)
    return obj[0]


def nccl_unique_id_bcast(rank, world):
    """Rank 0 creates the NCCL unique id; torch.distributed carries it to every rank."""
    return broadcast_bytes(nccl_unique_id() if rank == 0 else None, rank)


lib.janus_dev_workspace_region.restype = C.c_int32
lib.janus_dev_workspace_region.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_size_t),
                                           C.POINTER(C.c_size_t)]


def dev_workspace_region(graph, workspace, name, dtype=np.int32):
    """Copy a named workspace region (see janus_dev.h) to a numpy array."""
    off, n = C.c_size_t(), C.c_size_t()
    if lib.janus_dev_workspace_region(graph.h, name.encode(), C.byref(off), C.byref(n)) != 0:
        raise KeyError(name)
    raw = workspace[off.value:off.value + n.value].cpu().numpy()
    return raw.view(dtype)


def dev_profile(graph, enable):
    lib.janus_dev_profile(graph.h, int(enable))


def dev_phase_report(graph):
    """{phase: (total_ms, launches)} since dev_profile(graph, True)."""
    buf = C.create_string_buffer(1 << 16)
    lib.janus_dev_phase_report(graph.h, buf, 1 << 16)
    out = {}
    for item in buf.value.decode().split(";"):
        if item:
            name, ms, cnt = item.rsplit(":", 2)
            out[name] = (float(ms), int(cnt))
    return out


# ------------------------------------------------------------------ DP protocol test hooks (CPU)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32)
lib.janus_dev_dp_set_host_collective.restype = C.c_int32
lib.janus_dev_dp_set_host_collective.argtypes = [C.c_void_p, ALLREDUCE_FN, C.c_void_p]
lib.janus_dev_dp_segments.restype = C.c_int32
lib.janus_dev_dp_segments.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.c_int32]
lib.janus_dev_dp_host_step.restype = C.c_int32
lib.janus_dev_dp_host_step.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(JanusFailure), C.c_int32,
                                       C.POINTER(JanusFailure), C.POINTER(C.c_int32)]


def dev_dp_set_host_collective(graph, allreduce):
    """Route the graph's protocol-test collectives through allreduce(ndarray, op) (in place; op
    0 sum, 1 min, 2 max). Keeps the ctypes callback alive on the graph."""
    def cb(ctx, buf, count, dtype, op):
        try:
            dt = {F32: np.float32, I64: np.int64}[dtype]
            arr = np.ctypeslib.as_array(C.cast(buf, C.POINTER(np.ctypeslib.as_ctypes_type(dt))), (count,))
            allreduce(arr, op)
            return 0
        except Exception:  # noqa: BLE001 — reported to the library as a transport failure
            import traceback
            traceback.print_exc()
            return 1
    graph._dp_cb = ALLREDUCE_FN(cb)
    if lib.janus_dev_dp_set_host_collective(graph.h, graph._dp_cb, None) != 0:
        raise JanusError("janus_dev_dp_set_host_collective: graph is not data-parallel")


def dev_dp_segments(graph):
    """[(communicator, byte offset, bytes)] of the step's arena allreduces, in issue order."""
    buf = (C.c_int64 * 48)()
    n = lib.janus_dev_dp_segments(graph.h, buf, 16)
    return [(buf[3 * i], buf[3 * i + 1], buf[3 * i + 2]) for i in range(n)]


def dev_dp_host_step(graph, ws_host, local=None, runtime_err=False):
    """One step's collective protocol on a host workspace copy (np.uint8 array, modified in place).
    local: None or (assumption_id, index, observed). Returns (status, failure dict or None)."""
    lf = None
    if local is not None:
        lf = JanusFailure(assumption_id=local[0], rank=0, index=local[1], observed=local[2])
    out, st = JanusFailure(), C.c_int32()
    r = lib.janus_dev_dp_host_step(graph.h, ws_host.ctypes.data_as(C.c_void_p),
                                   C.byref(lf) if lf is not None else None, int(runtime_err),
                                   C.byref(out), C.byref(st))
    if r != 0:
        raise JanusError(f"janus_dev_dp_host_step: {r}")
    f = None
    if st.value == ASSUMPTION_FAILED:
        f = dict(assumption_id=out.assumption_id, rank=out.rank, index=out.index, observed=out.observed)
    return st.value, f


def dev_workspace_region_bytes(graph, name):
    """(byte offset, bytes) of a named workspace region (janus_dev.h), without a workspace."""
    off, n = C.c_size_t(), C.c_size_t()
    if lib.janus_dev_workspace_region(graph.h, name.encode(), C.byref(off), C.byref(n)) != 0:
        raise KeyError(name)
    return off.value, n.value
