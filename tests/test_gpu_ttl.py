"""TtlPolicy (baselines.cpp:22-28) on the GPU against the UNMODIFIED reference's TTL runs
(oracle/_ref via tests/refshim.py): the same evictions in order, cached tokens per turn, hit rate
and completion times, bit-exact. (The device maps TTL onto the recency select: see cs_pool.cpp.)"""
import numpy as np
import pytest

import refshim

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not refshim.available(), reason="oracle/_ref not built")]


@pytest.mark.parametrize("name,kw", [("supervisor-a", {}), ("supervisor-b", {}), ("synthetic-chain", {}),
                                     ("supervisor-c", {"budget": 60}), ("supervisor-d", {"concurrency": 8})])
def test_ttl_matches_reference(name, kw):
    from paper_2605_27744_b200 import api, workloads

    spec = workloads.preset_by_name(name)
    ref = refshim.run(spec, policy="ttl", **kw)
    eng = api.Engine(spec, policy="ttl", agent_capacity=1024, **kw)
    try:
        res = eng.run()
        ev = eng.evictions()
        t = eng.turns()
    finally:
        eng.close()
    assert ev.size > 0
    assert np.array_equal(ev, ref["evictions"])
    assert np.array_equal(t["cached_tokens"], ref["cached_tokens"])
    assert np.array_equal(t["end_us"].view(np.uint64), ref["end_us"].view(np.uint64))
    assert res["hit_rate"] == ref["hit_rate"]
