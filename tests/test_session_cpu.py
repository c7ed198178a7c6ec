"""Graph cache + relaxation driver, host side (no GPU): janus_relax against the SPEC lattice
examples and the Figure 4 hierarchy, session creation and its stats."""
import itertools

import numpy as np
import pytest

from workloads import programs as pg
from workloads.programs import Assumption, DISPATCH, RUNTIME

I32, I64 = 2, 3   # janus_dtype codes (include/janus.h)


def J():
    from paper_1812_01329_b200 import janus
    return janus


def _dims(a):
    return tuple(a.dims[k] for k in range(a.ndim))


def test_relax_shape_join_examples():
    janus = J()
    # S:246 join(Shape(4,8), Shape(3,8)) -> PartialShape(?,8)
    r = janus.relax(Assumption(4, "SHAPE_MATCH", DISPATCH, 0, dims=(4, 8)), (I32, (3, 8)))
    assert r is not None and r.kind == pg.ASM_CODE["SHAPE_MATCH"] and _dims(r) == (-1, 8) and r.id == 4
    # S:247 join(PartialShape(?,8), Shape(2,8)) -> PartialShape(?,8)
    r = janus.relax(Assumption(4, "SHAPE_MATCH", DISPATCH, 0, dims=(-1, 8)), (I32, (2, 8)))
    assert _dims(r) == (-1, 8)
    # S:248 rank mismatch -> kind level: the shape assumption is dropped
    assert janus.relax(Assumption(4, "SHAPE_MATCH", DISPATCH, 0, dims=(4, 8)), (I32, (4, 8, 2))) is None


def test_relax_control_flow_and_types():
    janus = J()
    # S:258 TripCount fails -> dynamic loop: a bounded device While (RANGE [1, n]) on the lengths
    r = janus.relax(Assumption(2, "TRIP_COUNT", RUNTIME, 2, value=35))
    assert r.kind == pg.ASM_CODE["RANGE"] and (r.lo, r.hi) == (1, 35) and r.target == 2 and r.mode == RUNTIME
    # the cache keys on argument types: a dtype failure re-specialises to the observed dtype
    r = janus.relax(Assumption(0, "DTYPE_EQ", DISPATCH, 0, dtype=I32), (I64, (64, 35)))
    assert r.dtype == I64 and r.kind == pg.ASM_CODE["DTYPE_EQ"]
    # single-arm branch / constant / tree-structure / range assumptions are dropped
    for a in (Assumption(3, "TYPE_TAG", RUNTIME, 9, value=1), Assumption(6, "VALUE_EQ", RUNTIME, 3, value=1),
              Assumption(7, "BRANCH_ARM", RUNTIME, 3, value=1),
              Assumption(8, "TREE_BINARY", RUNTIME, 0, hi=10, value=127),
              Assumption(2, "RANGE", RUNTIME, 2, lo=1, hi=35)):
        assert janus.relax(a) is None


def test_relax_is_a_least_upper_bound_brute_force():
    """For every pair of shapes of rank <= 3 over dims {1,2,3,?}: the relaxed assumption matches
    the observed shape and every shape the old one matched (upper bound), keeps every dim the two
    agree on (least), and relaxing again on a matching shape is a no-op (idempotent)."""
    janus = J()
    vals = [1, 2, 3, -1]

    def matches(dims, shape):
        return len(dims) == len(shape) and all(d == -1 or d == s for d, s in zip(dims, shape))

    for n in range(1, 4):
        for old in itertools.product(vals, repeat=n):
            for obs in itertools.product([1, 2, 3], repeat=n):
                r = janus.relax(Assumption(1, "SHAPE_MATCH", DISPATCH, 0, dims=old), (I32, obs))
                new = _dims(r)
                assert matches(new, obs)
                for shape in itertools.product([1, 2, 3], repeat=n):
                    if matches(old, shape):
                        assert matches(new, shape)
                assert all((d == o) if (o != -1 and o == s) else d == -1 for d, o, s in zip(new, old, obs))
                assert _dims(janus.relax(Assumption(1, "SHAPE_MATCH", DISPATCH, 0, dims=new), (I32, obs))) == new


def test_index_argument_dtypes_specialise_the_graph():
    """A graph specialised to int64 index arguments keeps its device program (it narrows them on
    the device, R10); any other index dtype has none (ERR_UNSUPPORTED: imperative only)."""
    janus = J()
    for dt, device in ((I64, True), (0, False)):
        prog = pg.lstm_lm_program(V=20, E=8, H=8, L=1, B=2, T=3, lr=0.1)
        for a in prog.assumptions:
            if a.kind == "DTYPE_EQ" and a.target == 0:
                a.dtype = dt
        g = janus.Graph(prog)
        assert g.device_path == device, g.build_message
        if not device:
            assert "int32 or int64" in g.build_message
        tp = pg.treelstm_program(V=20, E=8, H=8, C=2, B=2, lr=0.1)
        tp.assumptions[1].dtype = dt
        assert janus.Graph(tp).device_path == device


def test_session_create_and_stats_on_cpu():
    janus = J()
    prog = pg.lstm_lm_program(V=10000, E=650, H=650, L=2, B=64, T=35, lr=1.0)
    s = janus.Session(prog)
    st = s.stats()
    assert st["calls"] == st["graph_calls"] == st["imperative_calls"] == st["misses"] == 0
    assert st["aborts"] == {} and st["fail_threshold"] == 2
    assert len(st["entries"]) == 1 and st["entries"][0]["device"] and st["entries"][0]["active"]
    assert "2:TRIP_COUNT(2,35)" in st["entries"][0]["assumptions"]
    assert s.workspace_bytes() >= janus.Graph(prog).workspace_bytes
    # a program without a device lowering still makes a session (imperative-only initial entry)
    s2 = janus.Session(pg.running_sum_program(3))
    assert not s2.stats()["entries"][0]["device"]


def test_session_rejects_data_parallel_builds():
    import ctypes as C
    janus = J()
    prog = pg.lstm_lm_program(V=20, E=8, H=8, L=1, B=2, T=3, lr=0.1)
    opts = janus._build_opts(prog, world_size=2)
    h = C.c_void_p()
    err = C.create_string_buffer(256)
    ops, asms = janus.marshal_ops(prog), janus.marshal_assumptions(prog)
    r = janus.lib.janus_session_create(ops, len(prog.ops), asms, len(prog.assumptions), C.byref(opts), None,
                                       C.byref(h), err, 256)
    assert r == janus.ERR_UNSUPPORTED and not h.value and b"single-GPU" in err.value


def test_session_step_argument_errors_run_nothing():
    janus = J()
    s = janus.Session(pg.lstm_lm_program(V=20, E=8, H=8, L=1, B=2, T=3, lr=0.1))
    info = janus.JanusStepInfo()
    ws = janus.JanusTensor()   # NULL workspace: the step must refuse before touching anything
    a = janus._jt_array([np.zeros((2, 3), np.int32), np.zeros((2, 3), np.int32), np.full(2, 3, np.int32)])
    r = janus.lib.janus_session_step(s.h, a, 3, None, 5, None, 0, ws, None, None)
    assert r == janus.ERR_INVALID   # NULL state array with n_state > 0
    st = janus._jt_array([np.zeros(1, np.float32)])
    r = janus.lib.janus_session_step(s.h, a, 3, st, 1, None, 0, ws, None, info)
    assert r == janus.ERR_WORKSPACE and info.workspace_bytes > 0
    assert s.stats()["calls"] == 0
