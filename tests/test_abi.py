"""C ABI contract on the CPU (no GPU calls): the library loads, exports every symbol the headers
declare, validates op lists and lowers the paper's programs — or refuses them with the
documented status — without touching a device."""
import ctypes as C
import os
import re

import pytest

from workloads import programs as pg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def J():
    from paper_1812_01329_b200 import janus
    return janus


def _declared():
    names = set()
    for h in ("janus.h", "janus_dev.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(janus_\w+)\s*\(", src))
    return names


def test_library_exports_every_declared_symbol():
    janus = J()
    declared = _declared()
    assert {"janus_graph_build", "janus_run", "janus_run_imperative"} <= declared
    for name in declared:
        assert hasattr(janus.lib, name), name
    assert janus.lib.janus_abi_version() == 1
    assert janus.lib.janus_status_str(1) == b"ASSUMPTION_FAILED"


def test_struct_layouts_match_header():
    janus = J()
    assert C.sizeof(janus.JanusTensor) == 8 + 4 + 4 + 32 + 32
    assert C.sizeof(janus.JanusOp) == 12 + 48 + 48 + 4 + 64 + 16  # incl. 4 B padding before iattr
    assert C.sizeof(janus.JanusFailure) == 24
    assert C.sizeof(janus.JanusBuildOpts) == 4 + 4 + 128 + 4 * 8


@pytest.mark.parametrize("prog,kind", [
    (pg.lstm_lm_program(V=10000, E=650, H=650, L=2, B=64, T=35, lr=1.0), "tcgen05_bf16"),
    (pg.lstm_lm_program(V=32, E=16, H=16, L=1, B=4, T=8, lr=0.1, gemm="f32"), "fp32_single_cta"),
    (pg.lstm_lm_program(V=10000, E=650, H=650, L=2, B=64, T=35, lr=1.0, speculate="while", max_T=64), "while_width=64"),
    (pg.treelstm_program(V=20000, E=300, H=300, C=2, B=25, lr=0.05), "treelstm"),
])
def test_lowering_of_paper_programs(prog, kind):
    g = J().Graph(prog)
    assert g.device_path, g.build_message
    assert kind in g.describe()
    assert g.workspace_bytes > 0


def test_unspecialisable_graphs_keep_the_imperative_path():
    janus = J()
    for prog in (pg.running_sum_program(3),
                 pg.lstm_lm_program(V=20, E=8, H=8, L=1, B=2, T=3, lr=0.1, speculate="none"),
                 pg.treelstm_program(V=20, E=8, H=8, C=2, B=2, lr=0.1, speculate="none")):
        g = janus.Graph(prog)
        assert not g.device_path            # ERR_UNSUPPORTED: no device lowering...
        assert g.workspace_bytes > 0         # ...but a graph usable by janus_run_imperative
        assert "no device program" in g.describe()


def _corrupt(prog, fn):
    import copy
    p = copy.deepcopy(prog)
    fn(p)
    return p


def test_validation_rejects_malformed_op_lists():
    janus = J()
    base = pg.lstm_lm_program(V=20, E=8, H=8, L=1, B=2, T=3, lr=0.1)
    cases = {
        "bad arity": lambda p: p.ops[[o.kind for o in p.ops].index("LINEAR")].ins.pop(),
        "cycle": lambda p: p.ops.__setitem__(
            [o.kind for o in p.ops].index("EMBEDDING"),
            pg.Op("EMBEDDING", [(len(p.ops) - 1, 0), (len(p.ops) - 1, 0)])),
        "duplicate effect seq": lambda p: [o for o in p.ops if o.kind == "SGD_APPLY"][1].i.__setitem__(1, 1),
        "duplicate assumption id": lambda p: p.assumptions.append(pg.Assumption(0, "DTYPE_EQ", 0, 0, dtype=2)),
        "bad producer port": lambda p: p.ops[[o.kind for o in p.ops].index("LINEAR")].ins.__setitem__(0, (0, 5)),
    }
    for name, fn in cases.items():
        with pytest.raises(janus.JanusError, match="ERR_INVALID"):
            janus.Graph(_corrupt(base, fn))
