"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle and the reference
goldens. Bit-exact for every integer/index decision and every fp64 score (no tolerance: the
reference's score arithmetic is reproduced operation by operation)."""
import numpy as np
import pytest

import paper_2605_27744_b200 as cb
from oracle import pyoracle as orc
from paper_2605_27744_b200 import workloads as W

pytestmark = pytest.mark.gpu


def fnv1a64(keys):
    h = 1469598103934665603
    for byte in np.ascontiguousarray(keys, dtype="<u8").tobytes():
        h ^= byte
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


# ------------------------------------------------------------------ K1 hashing

def test_hash_known_answers():
    # SURVEY.md Appendix A.1, produced by the compiled reference
    assert cb.chain_hash(None, [1, 2, 3]) == 0x00C88D3A7850FA3D
    keys, counts = cb.block_keys_for(list(range(35)), 16)
    assert [int(k) for k in keys] == [0x316AFA7F10D3948D, 0xB306231F587B8829, 0x9902B6FEE6B545AE]
    assert list(counts) == [16, 16, 3]


def test_hash_random_prompts_match_oracle():
    rng = np.random.default_rng(7)
    prompts = [rng.integers(0, 2**32, size=int(n), dtype=np.uint64).astype(np.uint32)
               for n in rng.integers(1, 700, size=300)]
    for bs in (16, 7, 1):
        ks, cs, ag = cb.hash_prompts(prompts, block_size=bs, skip=4, take=4)
        for p, k, c, a in zip(prompts, ks, cs, ag):
            ok, oc = orc.block_keys(p, bs)
            assert np.array_equal(k, ok) and np.array_equal(c, oc)
            assert int(a) == orc.identity(ok, 4, 4)


def test_hash_rejects_empty_prompt():
    with pytest.raises(ValueError):
        cb.hash_prompts([[1, 2], []])


# ------------------------------------------------------------------ full engine runs

def _compare_runs(spec, policy, budget=None, prefetch=True):
    eng = cb.Engine(spec, policy=policy, budget=budget, prefetch=prefetch)
    try:
        res = eng.run()
        t = eng.turns()
        ev = eng.evictions()
        wst, wtg, wtk = eng.warmups()
    finally:
        eng.close()
    o = orc.run(spec, policy=policy, budget=budget, prefetch=prefetch)
    assert ev.size == o["evictions"].size
    assert np.array_equal(ev, o["evictions"])
    assert np.array_equal(t["cached_tokens"], o["cached_tokens"])
    assert np.array_equal(t["end_us"], o["end_us"])
    assert np.array_equal(wtg, o["warmup_target"])
    assert np.array_equal(wst, o["warmup_step"])
    assert np.array_equal(wtk, o["warmup_tick"])
    assert res["hit_rate"] == o["hit_rate"]
    assert res["steps"] == o["n_steps"]
    return res, ev


@pytest.mark.parametrize("name", W.preset_names())
@pytest.mark.parametrize("policy", ["lru", "cachesage"])
def test_presets_match_oracle(name, policy):
    _compare_runs(W.preset_by_name(name), policy)


# SURVEY.md Appendix A.2 (compiled reference): (hit_rate, evictions, fnv, warmups)
PRESET_GOLDENS = {
    ("supervisor-a", "lru"): (0.2722754226717074, 19088, 0x666D98380814C7C2),
    ("supervisor-a", "cachesage"): (0.41240476693085648, 14666, 0x765F27528F338DE6),
    ("supervisor-b", "lru"): (0.32819460214865925, 15488, 0xF0789EDF46701806),
    ("supervisor-b", "cachesage"): (0.476198794654555, 12015, 0xBE24A88438B51D38),
    ("supervisor-c", "lru"): (0.25840050053365721, 20299, 0x3376C49A1889C30F),
    ("supervisor-c", "cachesage"): (0.39325015641676786, 16172, 0x330C120001240365),
    ("supervisor-d", "lru"): (0.26296087976880855, 19106, 0x345C182A5D399D22),
    ("supervisor-d", "cachesage"): (0.38581043076863397, 15202, 0xBDE71FF663322F96),
    ("synthetic-chain", "lru"): (0.030494031479981691, 54816, 0x2202B3DCBDDBBAD1),
    ("synthetic-chain", "cachesage"): (0.23648720025353007, 50572, 0x3C20B4A646CF8F12),
}


@pytest.mark.parametrize("key", sorted(PRESET_GOLDENS))
def test_presets_match_reference_goldens(key):
    name, policy = key
    hit, n_ev, fnv = PRESET_GOLDENS[key]
    eng = cb.Engine(W.preset_by_name(name), policy=policy)
    res = eng.run()
    ev = eng.evictions()
    eng.close()
    assert res["hit_rate"] == hit
    assert res["evictions"] == n_ev
    assert fnv1a64(ev) == fnv


CFG1_GOLDENS = {  # SURVEY.md Appendix A.2, BASELINE cfg1
    (128, "lru"): (0.3564942747417032, 156981, 0x177BE4DA7DC86C66),
    (128, "cachesage"): (0.48797872495264472, 125366, 0x5BCAD5F614FB8A03),
    (65536, "lru"): (0.72966426095617121, 1837, 0x115F3A1A488E57D9),
    (65536, "cachesage"): (0.72966426095617121, 1839, 0xC65A36B1237BEB51),
}


@pytest.mark.parametrize("key", sorted(CFG1_GOLDENS))
def test_cfg1_matches_reference_goldens(key):
    budget, policy = key
    hit, n_ev, fnv = CFG1_GOLDENS[key]
    eng = cb.Engine(W.cfg1(budget), policy=policy)
    res = eng.run()
    ev = eng.evictions()
    eng.close()
    assert res["hit_rate"] == hit
    assert res["evictions"] == n_ev
    assert fnv1a64(ev) == fnv


# ------------------------------------------------------------------ admission-level parity

def _snapshot(rng, n, n_agents, pinned_frac=0.0, agent_frac=0.4):
    keys = rng.choice(2**62, size=n, replace=False).astype(np.uint64) + np.uint64(7)
    lt = (rng.permutation(n) + 1000).astype(np.uint64)
    has = rng.random(n) < agent_frac
    ag = rng.integers(0, n_agents, size=n)
    refs = (rng.random(n) < pinned_frac).astype(np.int32)
    return keys, lt, has, ag, refs


@pytest.mark.parametrize("seed,n,n_agents,pinned,policy", [
    (1, 3000, 6, 0.0, "cachesage"),
    (2, 5000, 12, 0.05, "cachesage"),
    (3, 20000, 40, 0.01, "cachesage"),
    (4, 4000, 8, 0.02, "lru"),
    (5, 700, 5, 0.3, "cachesage"),
])
def test_admissions_on_snapshots_match_oracle(seed, n, n_agents, pinned, policy):
    rng = np.random.default_rng(seed)
    keys, lt, has, ag, refs = _snapshot(rng, n, n_agents, pinned)
    agent_ids = [orc.mix64(0xA6E47 + i) for i in range(n_agents)]
    g = cb.Pool(n, policy=policy)
    g.register_agents(agent_ids)
    g.restore(keys, lt, agents=np.where(has, ag, 0xFFFFFFFF).astype(np.uint32), refs=refs)
    o = orc.Engine(n, agent_cap=n_agents + 1, policy=policy)
    o.restore(keys, lt, agents=[agent_ids[a] if h else None for h, a in zip(has, ag)], refs=refs,
              tick=int(lt.max()))
    tick = int(lt.max())
    prev = None
    pins_g = []
    for step in range(40):
        a = int(rng.integers(0, n_agents))
        # dispatch through the policy, then a prompt mixing resident and new blocks
        w = g.observe_dispatch(prev, a, tick + 1)
        o.dispatch(agent_ids[a])
        tick += 1
        prev = a
        L = int(rng.integers(1, 160))
        resident_pick = rng.choice(keys, size=min(L // 3, keys.size), replace=False)
        fresh = rng.choice(2**62, size=L - resident_pick.size).astype(np.uint64) + np.uint64(2**62)
        prompt = np.concatenate([resident_pick, fresh]).astype(np.uint64)
        counts = np.full(prompt.size, 16, np.int32)
        anchor = int(rng.integers(0, L + 1))
        cached, fm = g.lookup(prompt, counts, tick)
        oc, ofm = o.lookup(prompt, counts)
        assert (cached, fm) == (oc, ofm)
        tick += fm
        ev, pins = g.admit_pinned(prompt, counts, agent=a, anchor=anchor, tick_base=tick)
        o.admit_pinned(prompt, counts, agent=agent_ids[a], anchor=anchor)
        tick += prompt.size
        assert tick == o.tick
        assert np.array_equal(ev, o.evictions()[-ev.size:] if ev.size else ev)
        pins_g.append((pins, prompt))
        if len(pins_g) > 3:  # complete the oldest flight
            pslots, pkeys = pins_g.pop(0)
            if step % 2:  # EngineSim::unpin by BlockKey (cs_unpin) and by slot (cs_unpin_slots)
                g.unpin(pkeys)
            else:
                g.unpin_slots(pslots)
            o.unpin(pkeys)
        if w is not None:
            tg, _ = g.poll_actions()
            ot, _ = o.poll_into()
            assert [agent_ids[t] for t in tg] == [int(x) for x in ot]
        st = g.stats()
        assert st["resident"] == o.resident and st["pinned"] == o.pinned
    gk, gs = g.score_snapshot(tick)
    ok, os_ = o.scores()
    gi, oi = np.argsort(gk), np.argsort(ok)
    assert np.array_equal(gk[gi], ok[oi])
    assert np.array_equal(gs[gi], os_[oi])  # bit-equal fp64 scores
    g.close()
    o.close()


def test_all_pinned_raises_runtime_error():
    g = cb.Pool(4)
    keys = np.arange(1, 5, dtype=np.uint64)
    g.restore(keys, keys + 10, refs=np.ones(4, np.uint32))
    with pytest.raises(cb.CacheSageError, match="all resident blocks are pinned"):
        g.admit_pinned(np.array([99], np.uint64), np.array([16], np.int32), tick_base=100)
    g.close()


def test_large_pool_admissions_match_oracle():
    """A 1M-slot snapshot (multi-CTA scan, many trims) against the oracle's O(N) argmin."""
    rng = np.random.default_rng(11)
    n, n_agents = 1 << 20, 64
    keys, lt, has, ag, refs = _snapshot(rng, n, n_agents, 0.001, agent_frac=0.4)
    agent_ids = [orc.mix64(0xBEEF + i) for i in range(n_agents)]
    g = cb.Pool(n)
    g.register_agents(agent_ids)
    g.restore(keys, lt, agents=np.where(has, ag, 0xFFFFFFFF).astype(np.uint32), refs=refs)
    o = orc.Engine(n, agent_cap=n_agents + 1)
    o.restore(keys, lt, agents=[agent_ids[a] if h else None for h, a in zip(has, ag)], refs=refs,
              tick=int(lt.max()))
    tick = int(lt.max())
    prev = None
    for step in range(3):
        a = int(rng.integers(0, n_agents))
        g.observe_dispatch(prev, a, tick + 1)
        o.dispatch(agent_ids[a])
        tick += 1
        prev = a
        prompt = (rng.choice(2**62, size=64).astype(np.uint64) + np.uint64(2**62))
        counts = np.full(64, 16, np.int32)
        ev, _ = g.admit_pinned(prompt, counts, agent=a, anchor=8, tick_base=tick)
        o.admit_pinned(prompt, counts, agent=agent_ids[a], anchor=8)
        tick += 64
        assert np.array_equal(ev, o.evictions()[-64:])
    g.close()
    o.close()


@pytest.mark.parametrize("task,budget,policy", [(2600, 700, "cachesage"), (2600, 700, "lru"), (4200, 1500, "cachesage")])
def test_long_prompts_multi_chunk_match_oracle(task, budget, policy):
    """Prompts of 170-300 blocks: admissions span several 128-block chunks (the prescan feeds the
    first chunk, the later chunks rescan), against the C oracle, bit-exact."""
    spec = dict(W.preset_by_name("supervisor-a"))
    spec["task_tokens"], spec["sessions"] = task, 40
    res, ev = _compare_runs(spec, policy, budget=budget)
    assert ev.size > 0
