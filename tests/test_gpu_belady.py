"""The Belady baseline (BeladyPolicy, baselines.cpp:34-70) on the GPU pool: beyond the golden
runs in test_gpu_golden.py (every preset, tight budgets, oversized prompts, pins), the grid-wide
radix select on several CTAs, the hit-rate sandwich LRU <= CacheSage <= Belady (acceptance
criterion 2) on the reference's own fixtures, and the documented error paths.
"""
import json
import os

import numpy as np
import pytest

import refshim  # fnv1a64 only (pure Python)

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
RUNS = {(g["name"], g["kw"]["policy"]): g for g in json.load(open(os.path.join(GOLD, "runs.json")))["runs"]}

pytestmark = pytest.mark.gpu


def fnv(a):
    return hex(refshim.fnv1a64(np.ascontiguousarray(a, dtype="<u8")))


def _run(g, **extra):
    from paper_2605_27744_b200 import api

    kw = dict(g["kw"])
    pol = kw.pop("policy")
    eng = api.Engine(g["spec"], policy=pol, agent_capacity=1024, **kw, **extra)
    try:
        res = eng.run()
        return res, eng.evictions(), eng.turns()
    finally:
        eng.close()


@pytest.mark.parametrize("ctas", [2, 8, 37])
def test_belady_multi_cta_select(ctas, monkeypatch):
    """cfg1 at 16384 blocks: > kBelCand unpinned candidates, so every eviction pass runs the
    radix select; forcing several CTAs splits it over the grid (digits merged by global
    histograms, candidates compacted by atomics)."""
    monkeypatch.setenv("CS_BELADY_CTAS", str(ctas))
    g = RUNS[("cfg1@16384", "belady")]
    res, ev, t = _run(g)
    assert repr(res["hit_rate"]) == g["hit_rate"]
    assert ev.size == g["evictions"]
    assert fnv(ev) == g["evictions_fnv"]
    assert fnv(t["cached_tokens"]) == g["cached_fnv"]


@pytest.mark.parametrize("name", ["cfg1@128", "cfg1@256", "cfg1@4096", "supervisor-a", "supervisor-b",
                                  "supervisor-c", "supervisor-d", "synthetic-chain"])
def test_sandwich(name):
    """LRU <= CacheSage <= Belady on the same trace (acceptance_main.cpp crit. 2), all three from
    the GPU."""
    hr = {}
    for pol in ("lru", "cachesage", "belady"):
        g = RUNS[(name, pol)]
        res, ev, _ = _run(g)
        assert fnv(ev) == g["evictions_fnv"]
        hr[pol] = res["hit_rate"]
    assert hr["lru"] <= hr["cachesage"] <= hr["belady"]


def test_belady_host_inputs_multi_cta(monkeypatch):
    monkeypatch.setenv("CS_BELADY_CTAS", "4")
    g = RUNS[("cfg1@65536", "belady")]
    res, ev, t = _run(g, host_inputs=True)
    assert repr(res["hit_rate"]) == g["hit_rate"]
    assert fnv(ev) == g["evictions_fnv"]


def test_belady_needs_the_request_stream():
    from paper_2605_27744_b200 import api

    p = api.Pool(64, policy="belady")
    try:
        keys = np.arange(1, 5, dtype=np.uint64)
        with pytest.raises(Exception, match="request stream"):
            p.admit_pinned(keys, np.full(4, 16, np.int32), tick_base=0)
    finally:
        p.close()
