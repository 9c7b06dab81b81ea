"""EXPERIMENTAL device-resident scheduler (`device_scheduler=True`): whole
EngineSim steps in one persistent cooperative launch. Checked against the reference fixtures
(tests/golden) bit-exactly, like the default per-admission path."""
import json
import os

import numpy as np
import pytest

import refshim

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
RUNS = json.load(open(os.path.join(GOLD, "runs.json")))["runs"]

pytestmark = pytest.mark.gpu

ENGINE_KW = ("budget", "concurrency", "block_size", "prefetch", "skip", "take")


def fnv(a):
    return hex(refshim.fnv1a64(np.ascontiguousarray(a, dtype="<u8")))


@pytest.mark.parametrize("g", RUNS, ids=[g["name"] + "-" + g["kw"]["policy"] for g in RUNS])
def test_device_scheduler_golden(g):
    from paper_2605_27744_b200 import api

    kw = dict(g["kw"])
    ekw = {k: kw.pop(k) for k in list(kw) if k in ENGINE_KW}
    pol = kw.pop("policy")
    eng = api.Engine(g["spec"], policy=pol, agent_capacity=1024, device_scheduler=True, **ekw, **kw)
    try:
        res = eng.run()
        t = eng.turns()
        ev = eng.evictions()
        ws, wt, wk = eng.warmups()
    finally:
        eng.close()
    assert repr(res["hit_rate"]) == g["hit_rate"]
    assert ev.size == g["evictions"]
    assert fnv(ev) == g["evictions_fnv"]
    assert fnv(t["cached_tokens"]) == g["cached_fnv"]
    assert fnv(t["end_us"].view(np.uint64)) == g["end_us_fnv"]
    assert fnv(wt) == g["warmups_fnv"]
    assert res["steps"] == g["steps"]
    assert repr(res["sim_us"]) == g["sim_us"]
