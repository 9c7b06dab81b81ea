"""Decision parity at the BASELINE scales (VERDICT r01 "N1"): the GPU engine against the fast
exact CPU oracle (oracle/cs_oracle.c, fast_evict) on the SURVEY §8d cfg2/cfg3/cfg4 traces and on
the bench's own configuration (the cfg4 trace on a 16M-slot pre-filled pool).

The fast oracle is the reference's evict_one restated with per-agent heaps (exact by the
class-head lemma); tests/test_oracle_fast.py pins it to the O(N) oracle and to the unmodified
reference (oracle/_ref) on every golden fixture before it is trusted here. The bar is
bit-exact: every victim key in order, per-turn cached tokens, fp64 completion times, and the
drained warmups (step, target, tick).
"""
import threading

import numpy as np
import pytest

from oracle import pyoracle as orc

pytestmark = pytest.mark.gpu


def _snap_for_oracle(eng_agents, keys, lt, agents, refs):
    has = agents != np.uint32(0xFFFFFFFF)
    ids = np.zeros(keys.size, np.uint64)
    ids[has] = eng_agents[agents[has]]
    return keys, lt, has.astype(np.int32), ids, None if refs is None else refs.astype(np.int32)


def _gpu_state(eng):
    res = eng.result()
    t = eng.turns()
    ws, wt, wk = eng.warmups()
    return {"evictions": eng.evictions(), "cached": t["cached_tokens"], "end_us": t["end_us"].view(np.uint64),
            "w_step": ws, "w_target": wt, "w_tick": wk, "steps": res["steps"], "hit_rate": res["hit_rate"],
            "admissions": res["admissions"], "completed": res["completed"]}


def _assert_same(g, o, completed_only=False):
    assert g["evictions"].size == o["evictions"].size, (g["evictions"].size, o["evictions"].size)
    if g["evictions"].size:
        first = int(np.argmax(g["evictions"] != o["evictions"])) if not np.array_equal(g["evictions"], o["evictions"]) else -1
        assert first < 0, f"first differing victim at eviction {first}"
    assert np.array_equal(g["cached"], o["cached_tokens"])
    assert np.array_equal(g["end_us"], o["end_us"].view(np.uint64))
    assert np.array_equal(g["w_step"], o["warmup_step"])
    assert np.array_equal(g["w_target"], o["warmup_target"])
    assert np.array_equal(g["w_tick"], o["warmup_tick"])
    assert g["steps"] == o["n_steps"]
    if not completed_only:
        assert repr(g["hit_rate"]) == repr(o["hit_rate"])


# ------------------------------------------------------------- (a) whole traces, ~200K requests

TRACE_CASES = [
    # (config, budget, policy): SURVEY §8d cfg2 (32 agents, prefetch off) / cfg3 (128) / cfg4 (256)
    ("cfg2", 2048, "cachesage"), ("cfg3", 2048, "cachesage"), ("cfg4", 2048, "cachesage"),
    ("cfg2", 16384, "cachesage"), ("cfg3", 16384, "cachesage"), ("cfg4", 16384, "cachesage"),
    ("cfg4", 2048, "lru"),
    ("cfg2", 1 << 20, "cachesage"), ("cfg3", 4 << 20, "cachesage"), ("cfg4", 1 << 20, "cachesage"),
    ("cfg4", 4 << 20, "cachesage"),
]


def _trace_spec(cfg, budget, sessions=20000):
    from paper_2605_27744_b200 import workloads as W

    return {"cfg2": W.cfg2_hierarchical, "cfg3": W.cfg3_swarm, "cfg4": W.cfg4_mixed}[cfg](sessions=sessions,
                                                                                     budget=budget)


@pytest.mark.slow
@pytest.mark.parametrize("cfg,budget,policy", TRACE_CASES, ids=[f"{c}@{b}-{p}" for c, b, p in TRACE_CASES])
def test_trace_matches_fast_oracle(cfg, budget, policy):
    import paper_2605_27744_b200 as cb

    spec = _trace_spec(cfg, budget)
    eng = cb.Engine(spec, policy=policy, agent_capacity=1024, prefetch=spec["prefetch"])
    try:
        eng.run()
        g = _gpu_state(eng)
        assert eng.check() == {"pk_mismatch": 0, "resident_delta": 0, "pinned_delta": 0, "table_mismatch": 0}
    finally:
        eng.close()
    o = orc.run(spec, policy=policy, prefetch=spec["prefetch"], fast=True)
    assert len(g["cached"]) > 190_000
    _assert_same(g, o)
    if budget <= 16384:
        assert g["evictions"].size > 100_000


# ------------------------------------------------------------- (b) the bench's configuration

BENCH_POOL = 16 << 20
BENCH_ADMISSIONS = 2000


def _bench_spec():
    from paper_2605_27744_b200 import workloads as W

    return W.cfg4_mixed(sessions=40_000, budget=BENCH_POOL, seed=2608)  # bench.py rank 0


_ORACLE_CACHE = {}


def _oracle_for(mode, eng_agents, keys, lt, agents, refs, steps):
    k = (mode, steps)
    if k not in _ORACLE_CACHE:
        _ORACLE_CACHE.clear()
        _ORACLE_CACHE[k] = orc.run(_bench_spec(), snapshot=_snap_for_oracle(eng_agents, keys, lt, agents, refs),
                                   max_steps=steps, policy="cachesage", fast=True)
    return _ORACLE_CACHE[k]


@pytest.mark.slow
@pytest.mark.parametrize("mode,host_inputs", [("realistic", False), ("realistic", True), ("adversarial", False)])
def test_bench_configuration_matches_fast_oracle(mode, host_inputs):
    """bench.py's exact workload (cfg4 trace, 16M-slot pool pre-filled with the seed-11 snapshot,
    the prescan pipeline on every full-pool admission), >= 2000 admissions, on the device-input
    (`value`) and host-input (`e2e`) paths."""
    import paper_2605_27744_b200 as cb
    from paper_2605_27744_b200 import workloads as W

    spec = _bench_spec()
    eng = cb.Engine(spec, policy="cachesage", budget=BENCH_POOL, host_inputs=host_inputs, agent_capacity=1024,
                    prefetch=True)
    try:
        ag = eng.agents()
        keys, lt, agents, refs = W.pool_snapshot(BENCH_POOL, len(ag), seed=11, mode=mode)
        eng.restore(keys, lt, agents=agents, refs=refs)
        eng.run_for(BENCH_ADMISSIONS)
        g = _gpu_state(eng)
        ps = eng.pool_stats()
        assert eng.check() == {"pk_mismatch": 0, "resident_delta": 0, "pinned_delta": 0, "table_mismatch": 0}
    finally:
        eng.close()
    assert g["admissions"] >= BENCH_ADMISSIONS
    assert ps["prescan_used"] > BENCH_ADMISSIONS // 2  # the pipelined path is what was checked
    o = _oracle_for(mode, ag, keys, lt, agents, refs, g["steps"])
    assert o["n_admissions"] == g["admissions"]
    assert g["evictions"].size > 10_000
    _assert_same(g, o, completed_only=True)


@pytest.mark.slow
@pytest.mark.parametrize("transport", ["local", "peer"])
def test_bench_configuration_four_shards_match_fast_oracle(transport):
    """The same 16M-slot configuration hash-sharded over 4 shards (threads sharing this GPU),
    checked against the oracle — not against the single pool — with the device-to-device copy
    exchange and with the fused peer-memory exchange."""
    from paper_2605_27744_b200 import api, shard, workloads as W

    spec = _bench_spec()
    world = 4
    comms = shard.local_group(world) if transport == "local" else shard.peer_group(world)
    out = [None] * world
    err = []
    snap = {}

    def work(r):
        try:
            eng = api.Engine(spec, policy="cachesage", budget=BENCH_POOL, agent_capacity=1024, comm=comms[r],
                             grid_ctas=148 // world - (4 if transport == "peer" else 0), prefetch=True)
            try:
                if r == 0:
                    snap["agents"] = eng.agents()
                keys, lt, agents, refs = W.pool_snapshot(BENCH_POOL, len(eng.agents()), seed=11, mode="realistic")
                eng.restore(keys, lt, agents=agents, refs=refs)  # each shard keeps the keys it owns
                del keys, lt, agents, refs
                eng.run_for(BENCH_ADMISSIONS // 4)
                out[r] = _gpu_state(eng)
            finally:
                eng.close()
        except Exception as e:  # noqa: BLE001
            err.append(e)

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for c in comms:
        c.close()
    if err:
        raise err[0]
    keys, lt, agents, refs = W.pool_snapshot(BENCH_POOL, len(snap["agents"]), seed=11, mode="realistic")
    o = orc.run(spec, snapshot=_snap_for_oracle(snap["agents"], keys, lt, agents, refs),
                max_steps=out[0]["steps"], policy="cachesage", fast=True)
    owners = set(shard.shard_owner(o["evictions"], world).tolist())
    assert len(owners) == world
    for g in out:
        _assert_same(g, o, completed_only=True)
