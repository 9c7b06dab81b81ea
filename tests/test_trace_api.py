"""The reference's Python trace surface (py_module.cpp:134-183, trace_io.cpp): generate_trace
-> Trace.to_jsonl is byte-identical to the UNMODIFIED reference's write_trace_jsonl, and
read_trace_jsonl round-trips it and rejects what the reference rejects (CPU: the generator is
host code). run_sim over a trace is checked on the GPU in test_gpu_trace_api.py."""
import pytest

import refshim
import paper_2605_27744_b200 as cb

pytestmark = pytest.mark.skipif(not refshim.available(), reason="oracle/_ref not built")

PRESETS = ["supervisor-a", "supervisor-b", "supervisor-c", "supervisor-d", "synthetic-chain"]


@pytest.mark.parametrize("name", PRESETS)
def test_to_jsonl_byte_identical(name):
    for sessions, seed in ((None, None), (7, 12345)):
        ref = refshim.preset_trace_jsonl(name, sessions=sessions, seed=seed)
        t = cb.generate_trace(name, sessions=sessions, seed=seed)
        assert t.to_jsonl() == ref
        assert t.turn_count == ref.count("\n") - 1 and t.name == name


def test_read_trace_jsonl_round_trip():
    ref = refshim.preset_trace_jsonl("supervisor-a", sessions=11)
    t = cb.read_trace_jsonl(ref)
    assert t.to_jsonl() == ref
    assert (t.rows == cb.generate_trace("supervisor-a", sessions=11).rows).all()


def test_read_trace_jsonl_errors():
    ref = refshim.preset_trace_jsonl("supervisor-a", sessions=2)
    lines = ref.splitlines()
    with pytest.raises(RuntimeError, match="line 1: missing header"):
        cb.read_trace_jsonl("")
    with pytest.raises(RuntimeError, match="line 1: expected header"):
        cb.read_trace_jsonl(lines[1] + "\n")
    bad = lines[1].replace('"agent":', '"agent":99,"x":')
    with pytest.raises(RuntimeError, match="line 2"):
        cb.read_trace_jsonl(lines[0] + "\n" + bad + "\n")
    with pytest.raises(RuntimeError, match="line 2"):
        cb.read_trace_jsonl(lines[0] + "\n{not json\n")
