"""The reference's Policy / Runtime surface beyond the scoring loop, through the C ABI on the GPU:
Runtime::dispatch_event for every Event kind with its tick-regression check (runtime.cpp:59-69),
CacheSagePolicy::serialize_state().dump() byte for byte, predict / predict_next (the full MLE row,
fp64 bits) and poll_actions (cachesage_policy.cpp:50-153; baselines.cpp), and EngineSim::unpin by
BlockKey (engine.cpp:170-180).

The expected values are the UNMODIFIED reference's (tests/golden/policy_state.json, made by
tests/golden/make_policy_state.py through oracle/_ref).
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "policy_state.json")))
CASES = GOLD["cases"]
KINDS = {0: "block_touch", 1: "request_arrival", 2: "agent_dispatch", 3: "tool_return", 4: "turn_complete"}


def _pool(case):
    import paper_2605_27744_b200 as cb

    ids = [int(x, 16) for x in case["agents"]]
    pool = cb.Pool(64, agent_capacity=64, **case["kw"])
    # registration order is deliberately not first-seen order: the alphabet is note_agent's
    perm = list(np.random.default_rng(len(ids)).permutation(len(ids)))
    pool.register_agents([ids[i] for i in perm])
    idx = {ids[i]: k for k, i in enumerate(perm)}
    return pool, ids, idx


def _ranked(pool, forecast):
    return [[f"0x{i:016x}", p] for i, p, _ in forecast]


@pytest.mark.parametrize("case", [c for c in CASES if "checkpoints" in c], ids=lambda c: c["name"])
def test_event_stream_matches_reference(case):
    pool, ids, idx = _pool(case)
    id_of = {k: i for i, k in idx.items()}
    try:
        cps = iter(case["checkpoints"])
        drained = []
        for i, e in enumerate(case["events"]):
            agent = idx.get(e["agent"], -1) if e["kind"] in (1, 2, 3) else -1
            prev = idx[e["prev"]] if e.get("prev") is not None else None
            pool.dispatch_event(e["tick"], KINDS[e["kind"]], agent=agent, prev=prev, request=e["request"])
            if e["drain"]:
                t, k = pool.poll_actions()
                drained += [[f"0x{id_of[int(x)]:016x}", int(tk)] for x, tk in zip(t, k)]
            if e["ckpt"]:
                cp = next(cps)
                assert cp["i"] == i
                assert pool.serialize_state() == cp["state"], f"serialize_state differs after event {i}"
                assert drained == cp["drained"], f"drained warmups differ before event {i}"
                drained = []
                assert _ranked(pool, pool.predict(1)) == cp["predict"]
                for a_hex, row in cp["next"].items():
                    assert _ranked(pool, pool.predict(1, current=idx[int(a_hex, 16)])) == row, a_hex
                if case["kw"]["policy"] == "cachesage":
                    assert pool.state_bytes() == json.loads(cp["state"])["state_bytes"]
    finally:
        pool.close()


def test_tick_regression_is_a_runtime_error():
    case = next(c for c in CASES if c["name"] == "tick-regression")
    pool, ids, idx = _pool(case)
    try:
        for i, e in enumerate(case["events"]):
            agent = idx.get(e["agent"], -1) if e["kind"] in (1, 2, 3) else -1
            prev = idx[e["prev"]] if e.get("prev") is not None else None
            if i == case["fail_at"]:
                with pytest.raises(RuntimeError, match="tick regression"):
                    pool.dispatch_event(e["tick"], KINDS[e["kind"]], agent=agent, prev=prev)
                break
            pool.dispatch_event(e["tick"], KINDS[e["kind"]], agent=agent, prev=prev)
        else:
            pytest.fail("no regression in the stream")
        # observe_dispatch is the same Runtime entry point: equal ticks pass, lower ones fail
        last = case["events"][case["fail_at"] - 1]["tick"]
        pool.observe_dispatch(None, 0, last)
        with pytest.raises(RuntimeError, match="tick regression"):
            pool.observe_dispatch(0, 1, last - 1)
    finally:
        pool.close()


def test_unpin_by_key():
    """EngineSim::unpin (engine.cpp:170-180): refs drop per key; a key that is not resident throws
    logic_error (AssertionError in Python) after the keys before it were unpinned."""
    import paper_2605_27744_b200 as cb

    pool = cb.Pool(32, policy="lru")
    try:
        keys = np.arange(1, 9, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
        _, _ = pool.admit_pinned(keys, np.full(8, 16, np.int32), tick_base=0)
        _, _ = pool.admit_pinned(keys[:4], np.full(4, 16, np.int32), tick_base=8)  # keys 0..3 pinned twice
        assert pool.stats()["pinned"] == 8
        pool.unpin(keys[4:])
        assert pool.stats()["pinned"] == 4
        pool.unpin(keys[:4])
        assert pool.stats()["pinned"] == 4  # one pin left on each
        with pytest.raises(AssertionError, match="vanished"):  # logic_error (_lib.check)
            pool.unpin(np.array([keys[0], keys[1], 12345, keys[2]], np.uint64))
        assert pool.stats()["pinned"] == 2  # keys 0 and 1 were released before the throw
        with pytest.raises(AssertionError, match="vanished"):  # logic_error (_lib.check)
            pool.unpin(keys[5:6])  # resident but no pin left
        chk = np.zeros(4, np.int64)
        from paper_2605_27744_b200._lib import lib

        assert lib().cs_pool_check(pool.h, chk.ctypes.data) == 0 and not chk.any()
    finally:
        pool.close()


CELLS = GOLD["cells"]


def _fnv(a):
    import refshim

    return hex(refshim.fnv1a64(np.ascontiguousarray(a, dtype="<u8")))


@pytest.mark.parametrize("device_scheduler", [False, True], ids=["host", "devsched"])
@pytest.mark.parametrize("cell", CELLS, ids=lambda c: f"{c['name']}@{c['budget']}-{c['kw']['policy']}"
                         + ("-cost" if "cost" in c["kw"] else ""))
def test_engine_cell_state_and_cost_model(cell, device_scheduler):
    """A whole cell through the engine: bit-exact victims / cached tokens / completion times
    under the cell's CostModel (experiment.cpp:270-280; engine.cpp:302-305, 224-227), and the
    final serialize_state().dump() equal to the reference policy's at the end of the run."""
    from paper_2605_27744_b200 import api

    kw = dict(cell["kw"])
    pol = kw.pop("policy")
    cost = kw.pop("cost", None)
    cm = None if cost is None else dict(zip(("prefill_base_us", "prefill_per_token_us", "decode_per_token_us"), cost))
    eng = api.Engine(cell["spec"], policy=pol, budget=cell["budget"], cost_model=cm,
                     device_scheduler=device_scheduler, agent_capacity=1024, **kw)
    try:
        res = eng.run()
        t = eng.turns()
        ev = eng.evictions()
        assert repr(res["hit_rate"]) == cell["hit_rate"]
        assert ev.size == cell["evictions"] and _fnv(ev) == cell["evictions_fnv"]
        assert _fnv(t["cached_tokens"]) == cell["cached_fnv"]
        assert _fnv(t["end_us"].view(np.uint64)) == cell["end_us_fnv"]
        assert repr(res["sim_us"]) == cell["sim_us"]
        if not device_scheduler:
            assert eng.serialize_state() == cell["state"]
    finally:
        eng.close()


def test_cost_model_is_validated():
    from paper_2605_27744_b200 import api, workloads

    with pytest.raises(ValueError, match="cost model"):
        api.Engine(workloads.preset_by_name("supervisor-a"), cost_model={"prefill_base_us": 0.0})
