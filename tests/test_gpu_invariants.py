"""Pool invariants after (and during) real runs: the packed scan word of every slot matches the
exact last_touch / agent / pin state (every writer keeps it in step), the resident
and pinned counts match the slots, and the block table maps every resident key to its slot."""
import json
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
RUNS = {(g["name"], g["kw"]["policy"]): g for g in json.load(open(os.path.join(GOLD, "runs.json")))["runs"]}

pytestmark = pytest.mark.gpu

ZERO = {"pk_mismatch": 0, "resident_delta": 0, "pinned_delta": 0, "table_mismatch": 0}
CASES = [("supervisor-a", "cachesage"), ("supervisor-a", "lru"), ("supervisor-a", "belady"),
         ("cfg1@128", "cachesage"), ("cfg1@4096", "cachesage"), ("oversized-mixed", "cachesage"),
         ("pins-defer", "lru"), ("supervisor-a-conc8", "cachesage"), ("cfg1@16384", "belady")]


@pytest.mark.parametrize("name,pol", CASES, ids=[f"{n}-{p}" for n, p in CASES])
@pytest.mark.parametrize("host_inputs", [False, True])
def test_invariants_through_a_run(name, pol, host_inputs):
    from paper_2605_27744_b200 import api

    g = RUNS[(name, pol)]
    kw = dict(g["kw"])
    kw.pop("policy")
    eng = api.Engine(g["spec"], policy=pol, agent_capacity=1024, host_inputs=host_inputs, **kw)
    try:
        for _ in range(3):
            eng.run_for(97)
            assert eng.check() == ZERO
        eng.run()
        assert eng.check() == ZERO
    finally:
        eng.close()


def test_invariants_on_a_restored_snapshot():
    """The bench's shape at 1M slots: an adversarial snapshot (40% agent-carrying, Zipf agents,
    0.01% pinned), then pipelined admissions with evictions."""
    import paper_2605_27744_b200 as cb
    from paper_2605_27744_b200 import workloads as W

    pool = 1 << 20
    spec = W.cfg4_mixed(sessions=2000, budget=pool, seed=2608)
    eng = cb.Engine(spec, policy="cachesage", budget=pool, agent_capacity=1024)
    try:
        keys, lt, agents, refs = W.pool_snapshot(pool, len(eng.agents()), seed=11, mode="adversarial")
        eng.restore(keys, lt, agents=agents, refs=refs)
        assert eng.check() == ZERO
        eng.run_for(150)
        assert eng.check() == ZERO
    finally:
        eng.close()


def test_tick_space_guard():
    """The packed scan word keeps 40 bits of last_touch: ticks at or past 2^40 - 1 are refused
    loudly (restore: invalid argument; an admission: capacity) instead of aliasing."""
    from paper_2605_27744_b200 import api

    p = api.Pool(64, policy="cachesage")
    try:
        with pytest.raises(Exception, match="2\\^40"):
            p.restore(np.array([5], np.uint64), np.array([(1 << 40) - 1], np.uint64))
        keys = np.arange(1, 4, dtype=np.uint64)
        with pytest.raises(Exception, match="tick space"):
            p.admit_pinned(keys, np.full(3, 16, np.int32), tick_base=(1 << 40) - 8)
        ev, pins = p.admit_pinned(keys, np.full(3, 16, np.int32), tick_base=(1 << 40) - 64)
        assert ev.size == 0 and pins.size == 3
    finally:
        p.close()
