"""Pins the fast exact CPU oracle (cs_oracle.c fast_evict: per-agent heaps of unpinned blocks
ordered by last_touch + a heap of all resident blocks) before tests/test_gpu_scale_parity.py
trusts it at the BASELINE scales. CPU only.

It must reproduce (1) every reference fixture in tests/golden (the unmodified reference's runs),
(2) the O(N)-per-eviction oracle (the reference's argmin restated) on the cfg2/cfg3/cfg4
generators and on pre-filled snapshots, and (3) oracle/_ref itself on random specs.
"""
import json
import os
import sys

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2605_27744_b200 import workloads as W
import refshim

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
RUNS = [g for g in json.load(open(os.path.join(GOLD, "runs.json")))["runs"] if g["kw"]["policy"] != "belady"]


def fnv(a):
    return hex(refshim.fnv1a64(np.ascontiguousarray(a, dtype="<u8")))


@pytest.mark.parametrize("g", RUNS, ids=[g["name"] + "-" + g["kw"]["policy"] for g in RUNS])
def test_fast_oracle_reference_fixtures(g):
    r = O.run(g["spec"], fast=True, **g["kw"])
    assert repr(r["hit_rate"]) == g["hit_rate"]
    assert r["evictions"].size == g["evictions"]
    assert fnv(r["evictions"]) == g["evictions_fnv"]
    assert fnv(r["cached_tokens"].astype(np.int64)) == g["cached_fnv"]
    assert fnv(r["end_us"].view(np.uint64)) == g["end_us_fnv"]
    assert fnv(r["warmup_target"]) == g["warmups_fnv"]
    assert r["n_steps"] == g["steps"]
    assert repr(r["sim_us"]) == g["sim_us"]


def _same(a, b):
    for f in ("evictions", "cached_tokens", "warmup_step", "warmup_target", "warmup_tick", "completed"):
        assert np.array_equal(a[f], b[f]), f
    assert np.array_equal(a["end_us"].view(np.uint64), b["end_us"].view(np.uint64))
    for f in ("n_steps", "n_admissions", "truncated", "warmups_executed"):
        assert a[f] == b[f], f


def _spec(cfg, sessions, budget):
    from paper_2605_27744_b200 import workloads as W

    return {"cfg2": W.cfg2_hierarchical, "cfg3": W.cfg3_swarm, "cfg4": W.cfg4_mixed}[cfg](sessions=sessions,
                                                                                     budget=budget)


@pytest.mark.parametrize("cfg,policy", [("cfg2", "cachesage"), ("cfg3", "cachesage"), ("cfg4", "cachesage"),
                                        ("cfg4", "lru"), ("cfg4", "ttl")])
def test_fast_equals_scan_oracle_on_generators(cfg, policy):
    spec = _spec(cfg, 600, 512)
    kw = {"policy": policy, "prefetch": spec["prefetch"]}
    fast, slow = O.run(spec, fast=True, **kw), O.run(spec, fast=False, **kw)
    assert slow["evictions"].size > 10_000
    _same(fast, slow)


@pytest.mark.parametrize("mode", ["realistic", "adversarial"])
def test_fast_equals_scan_oracle_from_snapshot(mode):
    """A pre-filled pool (cfg5 composition, 0.01%..1% pinned) + the cfg4 trace, bounded steps."""
    from paper_2605_27744_b200 import workloads as W

    pool = 1 << 14
    spec = W.cfg4_mixed(sessions=200, budget=pool, seed=2608)
    keys, lt, agents, refs = W.pool_snapshot(pool, 256, seed=3, mode=mode, pinned_frac=0.01)
    ids = np.array([O.mix64(0xA6E + i) for i in range(256)], np.uint64)
    has = agents != np.uint32(0xFFFFFFFF)
    aid = np.where(has, ids[np.minimum(agents, 255)], 0).astype(np.uint64)
    snap = (keys, lt, has.astype(np.int32), aid, refs.astype(np.int32))
    fast = O.run(spec, snapshot=snap, max_steps=400, fast=True)
    slow = O.run(spec, snapshot=snap, max_steps=400, fast=False)
    assert fast["n_steps"] == 400 and slow["evictions"].size > 2000
    assert not fast["completed"].all()
    _same(fast, slow)


def test_snapshot_and_step_bound_semantics():
    """max_steps stops at a step boundary; a snapshot larger than the budget is rejected."""
    spec = _spec("cfg4", 50, 4096)
    full = O.run(spec, fast=True)
    part = O.run(spec, fast=True, max_steps=full["n_steps"] // 2)
    assert part["n_steps"] == full["n_steps"] // 2
    assert np.array_equal(part["evictions"], full["evictions"][:part["evictions"].size])
    done = part["completed"]
    assert np.array_equal(part["cached_tokens"][done], full["cached_tokens"][done])
    k = np.arange(1, 5000, dtype=np.uint64)
    with pytest.raises(RuntimeError, match="snapshot"):
        O.run(spec, snapshot=(k, k, np.zeros(k.size, np.int32), np.zeros(k.size, np.uint64), None), max_steps=1)


def test_cost_model_knobs():
    """CostModel (engine.hpp:20-24): non-default costs change completion times (and so pin
    release order); non-positive costs are invalid_argument (engine.cpp:60-63)."""
    spec = _spec("cfg4", 100, 1024)
    a = O.run(spec, fast=True)
    b = O.run(spec, fast=True, cost=(500.0, 20.0, 9000.0))
    assert not np.array_equal(a["end_us"], b["end_us"])
    with pytest.raises(RuntimeError, match="cost model"):
        O.run(spec, fast=True, cost=(-1.0, 50.0, 20000.0))


@pytest.mark.skipif(not refshim.available(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("seed", range(8))
def test_fast_oracle_vs_reference_random(seed):
    from test_oracle_golden import _random_spec

    rng = np.random.default_rng(5000 + seed)
    spec = _random_spec(rng, int(rng.integers(2, 9)))
    for pol in ("lru", "cachesage", "ttl"):
        kw = {"policy": pol, "window": int(rng.choice([8, 64, 1024])), "e_max": int(rng.integers(2, 10))}
        try:
            ref = refshim.run(spec, **kw)
        except RuntimeError:
            with pytest.raises(RuntimeError):
                O.run(spec, fast=True, **kw)
            continue
        mine = O.run(spec, fast=True, **kw)
        for f in ("cached_tokens", "evictions", "warmup_step", "warmup_target", "warmup_tick"):
            assert np.array_equal(np.asarray(ref[f]), np.asarray(mine[f])), f
        assert ref["n_steps"] == mine["n_steps"]


@pytest.mark.skipif(not refshim.available(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("cost", [(500.0, 20.0, 9000.0), (3000.0, 7.5, 41000.0)])
def test_cost_model_matches_reference(cost):
    """A non-default CostModel (experiment.cpp:270-280) moves completion times and so the pin
    release order: the oracle follows the reference bit for bit (end_us bits, victims)."""
    for name, budget in (("cfg1", 256), ("cfg1", 128), ("supervisor-a", 60)):
        spec = W.cfg1(budget) if name == "cfg1" else W.preset_by_name(name)
        ref = refshim.run(spec, policy="cachesage", budget=budget, cost=cost)
        mine = O.run(spec, fast=True, policy="cachesage", budget=budget, cost=cost)
        assert np.array_equal(ref["end_us"].view(np.uint64), mine["end_us"].view(np.uint64))
        assert np.array_equal(ref["evictions"], mine["evictions"])
        assert np.array_equal(ref["cached_tokens"], mine["cached_tokens"])


@pytest.mark.skipif(not refshim.available(), reason="oracle/_ref not built (needs /root/reference)")
def test_policy_state_fixture_is_the_reference():
    """tests/golden/policy_state.json (the GPU serialize_state / predict / event-stream parity
    fixture) is what the reference produces for the same streams today."""
    sys.path.insert(0, GOLD)
    import make_policy_state as M

    gold = json.load(open(os.path.join(GOLD, "policy_state.json")))["cases"]
    for (name, seed, na, ne, kw), g in zip(M.CASES, gold):
        _, ev = M.stream(seed, na, ne)
        cps, err = refshim.policy_events(ev, **kw)
        assert err is None and cps == g["checkpoints"], name
