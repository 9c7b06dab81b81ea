"""GPU path (through the C ABI) against the fixtures the UNMODIFIED reference produced
(tests/golden, made by tests/golden/make_golden.py over oracle/_ref). Bit-exact: evicted keys in
order, cached tokens per turn, completion times (fp64 bits), warmups, hit rate (repr), and
policy scores (fp64 bits).
"""
import json
import os

import numpy as np
import pytest

import refshim  # fnv1a64 only (pure Python)

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
RUNS = json.load(open(os.path.join(GOLD, "runs.json")))["runs"]
HASH = json.load(open(os.path.join(GOLD, "hashing.json")))
POL = json.load(open(os.path.join(GOLD, "policy.json")))

pytestmark = pytest.mark.gpu

ENGINE_KW = ("budget", "concurrency", "block_size", "prefetch", "skip", "take")


def fnv(a):
    return hex(refshim.fnv1a64(np.ascontiguousarray(a, dtype="<u8")))


def _engine(g):
    from paper_2605_27744_b200 import api

    kw = dict(g["kw"])
    ekw = {k: kw.pop(k) for k in list(kw) if k in ENGINE_KW}
    pol = kw.pop("policy")
    return api.Engine(g["spec"], policy=pol, agent_capacity=1024, **ekw, **kw)


@pytest.mark.parametrize("g", RUNS, ids=[g["name"] + "-" + g["kw"]["policy"] for g in RUNS])
def test_engine_run_golden(g):
    eng = _engine(g)
    try:
        res = eng.run()
        t = eng.turns()
        ev = eng.evictions()
        ws, wt, wk = eng.warmups()
    finally:
        eng.close()
    assert t["cached_tokens"].size == g["turns"]
    assert repr(res["hit_rate"]) == g["hit_rate"]
    assert ev.size == g["evictions"]
    assert [hex(int(x)) for x in ev[:16]] == g["first_evictions"]
    assert fnv(ev) == g["evictions_fnv"]
    assert fnv(t["cached_tokens"]) == g["cached_fnv"]
    assert fnv(t["end_us"].view(np.uint64)) == g["end_us_fnv"]
    assert ws.size == g["n_warmups"]
    assert fnv(wt) == g["warmups_fnv"]
    assert [[int(a), hex(int(b)), int(c)] for a, b, c in zip(ws, wt, wk)][:200] == g["warmups"]
    assert res["steps"] == g["steps"]
    assert res["truncated"] == g["truncated"]
    assert res["warmups_executed"] == g["warmups_executed"]
    assert repr(res["sim_us"]) == g["sim_us"]


def test_hash_golden_on_device():
    from paper_2605_27744_b200 import api

    by_bs = {}
    for c in HASH["block_keys"]:
        by_bs.setdefault(c["block_size"], []).append(c)
    for bs, cases in by_bs.items():
        ks, cs, _ = api.hash_prompts([c["tokens"] for c in cases], block_size=bs)
        for c, k, n in zip(cases, ks, cs):
            assert [hex(int(x)) for x in k] == c["keys"]
            assert [int(x) for x in n] == c["counts"]


def test_identity_golden_on_device():
    """derive_agent_identity over device-hashed prompts, via the reference's identity of the
    same keys (the golden identity cases take arbitrary keys; here the keys come from K1)."""
    from paper_2605_27744_b200 import api
    from oracle import pyoracle as O

    rng = np.random.default_rng(7)
    prompts = [rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32).tolist()
               for n in (1, 40, 64, 65, 80, 128, 129, 300)]
    for skip, take in ((4, 4), (0, 1), (2, 6)):
        ks, _, ag = api.hash_prompts(prompts, block_size=16, skip=skip, take=take)
        for k, a in zip(ks, ag):
            assert int(a) == O.identity(k, skip, take)


@pytest.mark.parametrize("p", POL, ids=[str(p["seed"]) for p in POL])
def test_policy_trace_golden_on_device(p):
    from paper_2605_27744_b200 import api

    ids = [int(x, 16) for x in p["agents"]]
    kw = dict(p["kw"])
    pool = api.Pool(64, policy="cachesage", agent_capacity=64, **kw)
    try:
        first = pool.register_agents(ids)
        idx = {a: first + i for i, a in enumerate(ids)}
        rid = {v: k for k, v in idx.items()}
        prev = None
        for i, a in enumerate(p["next"]):
            pool.observe_dispatch(prev, idx[ids[a]], i + 1)
            prev = idx[ids[a]]
            t, _ = pool.poll_actions(64)
            got = rid[int(t[-1])] if len(t) else 0
            assert hex(got) == p["warm"][i], i
        hops = pool.hops(first + len(ids))[first:]
        assert hops.tolist() == p["hops"]
        b = p["blocks"]
        keys = np.array([int(x, 16) for x in b["keys"]], np.uint64)
        ags = np.array([idx[int(a, 16)] if h else 0xFFFFFFFF for a, h in zip(b["agents"], b["has_agent"])],
                       np.uint32)
        pool.restore(keys, np.array(b["touch"], np.uint64), agents=ags)
        k, s = pool.score_snapshot(b["now"])
        got = {int(kk): hex(int(v)) for kk, v in zip(k, s.view(np.uint64))}
        for kk, want in zip(keys, p["scores_bits"]):
            assert got[int(kk)] == want
    finally:
        pool.close()


HOST_INPUT_RUNS = [g for g in RUNS if g["name"] in ("supervisor-a", "synthetic-chain", "cfg1@128", "oversized-mixed",
                                                    "supervisor-a-conc8", "pins-defer")]


@pytest.mark.parametrize("g", HOST_INPUT_RUNS, ids=[g["name"] + "-" + g["kw"]["policy"] for g in HOST_INPUT_RUNS])
def test_engine_host_inputs_golden(g):
    """The end-to-end path bench.py times (prompt blocks H2D per admission from pinned memory,
    the victims D2H behind each admission kernel) gives the reference's run bit-exactly."""
    from paper_2605_27744_b200 import api

    kw = dict(g["kw"])
    ekw = {k: kw.pop(k) for k in list(kw) if k in ENGINE_KW}
    pol = kw.pop("policy")
    eng = api.Engine(g["spec"], policy=pol, agent_capacity=1024, host_inputs=True, **ekw, **kw)
    try:
        res = eng.run()
        t = eng.turns()
        ev = eng.evictions()
        ws, wt, wk = eng.warmups()
        r = eng.result()
    finally:
        eng.close()
    assert repr(res["hit_rate"]) == g["hit_rate"]
    assert fnv(ev) == g["evictions_fnv"]
    assert fnv(t["cached_tokens"]) == g["cached_fnv"]
    assert fnv(wt) == g["warmups_fnv"]
    assert r["h2d_bytes"] > 0 and r["d2h_bytes"] > 0
