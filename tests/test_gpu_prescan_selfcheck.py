"""Long-run self-check of the prescan pipeline at the bench's scale.

With CS_DEBUG_PRESCAN=1, CTA 0 brute-forces after every consumed prescan that each unpinned
agentless block older than the last listed entry of list E is in that list (debug_check_e,
csrc/cs_admit.cu). A stale TMA (async-proxy) read of the pool inside the persistent admission
server would show up here as a missing member. The run is 2,000 admissions of the bench's cfg4
trace on the realistic and the adversarial 16M-slot snapshots (1,400+ of them consume a
prescan); tests/test_gpu_scale_parity.py checks the same runs' decisions against the oracle.
"""
import ctypes as C

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.slow
@pytest.mark.parametrize("mode", ["realistic", "adversarial"])
def test_prescan_lists_complete_at_16m(mode, monkeypatch):
    monkeypatch.setenv("CS_DEBUG_PRESCAN", "1")  # read when the pool is created
    import paper_2605_27744_b200 as cb
    from paper_2605_27744_b200 import workloads as W
    from paper_2605_27744_b200._lib import lib

    pool = 16 << 20
    spec = W.cfg4_mixed(sessions=40000, budget=pool, seed=2608)
    eng = cb.Engine(spec, policy="cachesage", budget=pool, agent_capacity=1024, prefetch=spec.get("prefetch", True))
    try:
        keys, lt, agents, refs = W.pool_snapshot(pool, len(eng.agents()), seed=11, mode=mode)
        eng.restore(keys, lt, agents=agents, refs=refs)
        del keys, lt, agents, refs
        ps0 = eng.pool_stats()
        eng.run_for(2000)
        ps1 = eng.pool_stats()
        buf = (C.c_uint64 * (16 * 1024))()
        grid = C.c_int(0)
        assert lib().cs_pool_debug(lib().cs_engine_pool(eng.h), buf, 16 * 1024, C.byref(grid)) == 0
        missing = buf[16 * grid.value + 16]
        used = ps1["prescan_used"] - ps0["prescan_used"]
        assert missing == 0, f"{missing} true list-E members absent from the consumed prescan lists"
        # (admissions that evict nothing, or do not start, consume no prescan)
        assert used >= 1000, f"only {used} admissions were served by the prescan"
        assert eng.check() == {k: 0 for k in eng.check()}
    finally:
        eng.close()
