"""run_sim(trace) on the GPU against the UNMODIFIED reference's run_sim(read_trace_jsonl(text))
(py_module.cpp:170-180): the same metrics dict, exact (integer fields equal, fp64 fields
bit-identical: the per-turn times are bit-exact and the sums run in the reference's order)."""
import pytest

import refshim
import paper_2605_27744_b200 as cb

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not refshim.available(), reason="oracle/_ref not built")]


@pytest.mark.parametrize("name,policy,kw", [
    ("supervisor-a", "cachesage", {}), ("supervisor-b", "lru", {}), ("synthetic-chain", "cachesage", {}),
    ("supervisor-c", "cachesage", {"budget": 60}), ("supervisor-d", "cachesage", {"prefetch": False}),
    ("supervisor-a", "cachesage", {"concurrency": 8}),
])
def test_run_sim_trace_matches_reference(name, policy, kw):
    text = refshim.preset_trace_jsonl(name)
    want = refshim.run_sim_jsonl(text, policy=policy, **kw)
    got = cb.run_sim(cb.read_trace_jsonl(text), policy=policy, **kw)
    assert got == want
