"""Pins the CPU oracle (oracle/cs_oracle.c) to the reference (CPU-only, no GPU).

Three anchors, strongest first:
  1. tests/golden/*.json — produced by the UNMODIFIED reference compiled in place
     (tests/golden/make_golden.py over oracle/_ref); always available, also on the GPU box.
  2. SURVEY.md Appendix A numbers (hit rates / eviction FNVs of the shipped presets).
  3. oracle/_ref itself on randomised specs, when it is built in this container.
Mirrors the reference's own test themes: test_hashing.cpp (KATs, block splits, identity
fallbacks), test_workload.cpp (determinism), test_reachability.cpp / test_cachesage_policy.cpp
(hops, gate, warmups), test_engine.cpp / test_integration.cpp (run summaries).
"""
import json
import os

import numpy as np
import pytest

from oracle import pyoracle as O
import refshim

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def fnv(a):
    return hex(refshim.fnv1a64(np.ascontiguousarray(a, dtype="<u8")))


RUNS = _load("runs.json")["runs"]
HASH = _load("hashing.json")
GEN = _load("generator.json")
POL = _load("policy.json")


# ------------------------------------------------------------------ hashing (K1)

def test_hash_kats():
    assert hex(O.chain_hash(None, [1, 2, 3])) == HASH["kats"]["chain_hash_123"]
    assert hex(O.chain_hash(0x1234, [5])) == HASH["kats"]["chain_hash_parent"]


@pytest.mark.parametrize("i", range(len(HASH["block_keys"])))
def test_block_keys_golden(i):
    c = HASH["block_keys"][i]
    k, n = O.block_keys(np.array(c["tokens"], np.uint32), c["block_size"])
    assert [hex(int(x)) for x in k] == c["keys"]
    assert [int(x) for x in n] == c["counts"]


def test_identity_golden():
    for c in HASH["identity"]:
        keys = np.array([int(x, 16) for x in c["keys"]], np.uint64)
        assert hex(O.identity(keys, c["skip"], c["take"])) == c["identity"], c


def test_block_keys_empty_prompt():
    k, n = O.block_keys(np.zeros(0, np.uint32), 16)
    assert len(k) == 0 and len(n) == 0


# ------------------------------------------------------------------ generator

@pytest.mark.parametrize("g", GEN, ids=[g["name"] for g in GEN])
def test_generator_golden(g):
    t = O.generate(g["spec"])
    assert t.shape[0] == g["n"]
    assert fnv(t.astype(np.uint64).reshape(-1)) == g["fnv"]
    assert t[:20].tolist() == g["head"]


def test_generator_deterministic():
    s = GEN[0]["spec"]
    assert np.array_equal(O.generate(s), O.generate(s))


# ------------------------------------------------------------------ full runs (observe->score->select->act)

def _check_run(r, g):
    assert r["cached_tokens"].size == g["turns"]
    assert repr(r["hit_rate"]) == g["hit_rate"]
    assert r["evictions"].size == g["evictions"]
    assert [hex(int(x)) for x in r["evictions"][:16]] == g["first_evictions"]
    assert fnv(r["evictions"]) == g["evictions_fnv"]
    assert fnv(r["cached_tokens"].astype(np.int64)) == g["cached_fnv"]
    assert fnv(r["end_us"].view(np.uint64)) == g["end_us_fnv"]
    assert r["warmup_step"].size == g["n_warmups"]
    assert fnv(r["warmup_target"]) == g["warmups_fnv"]
    w = [[int(s), hex(int(t)), int(k)] for s, t, k in zip(r["warmup_step"], r["warmup_target"], r["warmup_tick"])]
    assert w[:200] == g["warmups"]
    assert r["n_steps"] == g["steps"]
    assert r["truncated"] == g["truncated"]
    assert r["warmups_executed"] == g["warmups_executed"]
    assert repr(r["sim_us"]) == g["sim_us"]


@pytest.mark.parametrize("g", RUNS, ids=[g["name"] + "-" + g["kw"]["policy"] for g in RUNS])
def test_oracle_run_golden(g):
    if g["kw"]["policy"] == "belady" and g["kw"].get("budget", 0) >= 4096:
        pytest.skip("O(N) per eviction at N >= 4096 takes minutes on CPU; the GPU tests check these fixtures")
    _check_run(O.run(g["spec"], **g["kw"]), g)


# SURVEY.md Appendix A.1 (hit rates of the five presets under the two policies)
SURVEY_A1 = {
    ("supervisor-a", "cachesage"): 0.41240476693085648,
    ("supervisor-a", "belady"): 0.42184651403788215,
    ("supervisor-b", "belady"): 0.48052231635950737,
}


def test_survey_appendix_anchor():
    for (name, pol), hr in SURVEY_A1.items():
        g = next(x for x in RUNS if x["name"] == name and x["kw"]["policy"] == pol)
        assert float(g["hit_rate"]) == hr


# ------------------------------------------------------------------ policy (K3/K4/K6)

@pytest.mark.parametrize("p", POL, ids=[str(p["seed"]) for p in POL])
def test_policy_trace_golden(p):
    ids = [int(x, 16) for x in p["agents"]]
    kw = dict(p["kw"])
    e_max = kw.get("e_max", 8)
    eng = O.Engine(budget=64, agent_cap=len(ids) + 1, policy="cachesage", **kw)
    try:
        for i, a in enumerate(p["next"]):
            eng.dispatch(ids[a])
            t, _ = eng.poll_into(64)
            want = int(p["warm"][i], 16)
            got = int(t[-1]) if len(t) else 0
            assert got == want, (i, hex(got), p["warm"][i])
        hops = eng.hops(np.array(ids, np.uint64))
        assert hops.tolist() == p["hops"]
        for h, s in zip(hops, p["survival"]):
            if h < 0:
                continue
            surv = 1.0 - min(int(h), e_max) / e_max
            assert repr(surv) == s
        # CacheSagePolicy::score over explicit blocks: restore them at tick `now`
        b = p["blocks"]
        keys = [int(x, 16) for x in b["keys"]]
        ags = [int(a, 16) if h else None for a, h in zip(b["agents"], b["has_agent"])]
        eng.restore(keys, b["touch"], agents=ags, tick=b["now"])
        k, s = eng.scores()
        got = {int(kk): hex(int(v)) for kk, v in zip(k, s.view(np.uint64))}
        for kk, want in zip(keys, p["scores_bits"]):
            assert got[kk] == want
    finally:
        eng.close()


# ------------------------------------------------------------------ live reference on random specs

def _random_spec(rng, n_agents):
    T = rng.random((n_agents, n_agents))
    T[rng.random((n_agents, n_agents)) < 0.5] = 0.0
    for i in range(n_agents):
        T[i, (i + 1) % n_agents] += 0.5
    T = T / T.sum(1, keepdims=True)
    return {"name": "rand", "anchor_tokens": [int(x) for x in rng.integers(32, 300, n_agents)],
            "transition": T.tolist(), "supervisor": int(rng.integers(0, n_agents)) if rng.random() < 0.5 else None,
            "turns_min": 2, "turns_max": int(rng.integers(3, 9)), "sessions": int(rng.integers(5, 60)),
            "task_tokens": int(rng.integers(16, 200)), "history_growth": int(rng.integers(0, 64)),
            "decode_tokens": 16, "template_tokens": int(rng.integers(0, 40)),
            "concurrency": int(rng.integers(1, 6)), "budget_blocks": int(rng.integers(24, 400)),
            "seed": int(rng.integers(0, 2**31))}


@pytest.mark.skipif(not refshim.available(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("seed", range(12))
def test_oracle_vs_reference_random(seed):
    rng = np.random.default_rng(1000 + seed)
    spec = _random_spec(rng, int(rng.integers(2, 9)))
    for pol in ("lru", "cachesage"):
        kw = {"policy": pol, "window": int(rng.choice([8, 64, 1024])), "e_max": int(rng.integers(2, 10))}
        try:
            ref = refshim.run(spec, **kw)
        except RuntimeError as ex:  # e.g. an all-pinned pool: the oracle must fail the same way
            with pytest.raises(RuntimeError):
                O.run(spec, **kw)
            assert "pinned" in str(ex) or "stall" in str(ex)
            continue
        mine = O.run(spec, **kw)
        for f in ("cached_tokens", "prompt_tokens", "evictions", "warmup_step", "warmup_target", "warmup_tick"):
            assert np.array_equal(np.asarray(ref[f]), np.asarray(mine[f])), f
        assert np.array_equal(ref["end_us"].view(np.uint64), mine["end_us"].view(np.uint64))
        for f in ("hit_rate", "truncated", "warmups_executed", "n_steps", "sim_us"):
            assert ref[f] == mine[f], f
