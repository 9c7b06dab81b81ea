"""Regenerates the golden fixtures in tests/golden from the UNMODIFIED reference.

Needs oracle/_ref/libcachesage_ref.so (built by `make -C oracle ref` from /root/reference). The
fixtures are committed; the GPU box and the CPU test suite only read them.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import refshim  # noqa: E402
from paper_2605_27744_b200 import workloads as W  # noqa: E402


def fnv(arr) -> str:
    return hex(refshim.fnv1a64(np.ascontiguousarray(arr, dtype="<u8")))


def tiny_spec(agents=2, sessions=4, seed=5):
    """helpers.hpp tiny_spec (test fixture restated): 2-agent cycle, budget 64."""
    T = [[1.0 if j == (i + 1) % agents else 0.0 for j in range(agents)] for i in range(agents)]
    return {"name": "tiny", "anchor_tokens": [160] * agents, "transition": T, "supervisor": 0,
            "turns_min": 4, "turns_max": 6, "sessions": sessions, "task_tokens": 96, "history_growth": 16,
            "decode_tokens": 8, "template_tokens": 16, "concurrency": 1, "budget_blocks": 64, "seed": seed}


def run_cases():
    cases = []
    for s in W.preset_workloads():
        for pol in ("lru", "cachesage"):
            cases.append((s["name"], s, {"policy": pol}))
    for b in (128, 256, 4096, 65536):
        for pol in ("lru", "cachesage"):
            cases.append((f"cfg1@{b}", W.cfg1(b), {"policy": pol, "budget": b}))
    # engine edge cases (test_engine.cpp themes): tight budgets, oversized prompts, prefetch off,
    # concurrency, identity windows, policy knobs
    t = tiny_spec(2, 6, 21)
    t["budget_blocks"] = 40
    t["turns_min"] = t["turns_max"] = 6
    cases.append(("tiny-alternation-lru", t, {"policy": "lru", "prefetch": False}))
    cases.append(("tiny-alternation-cachesage", t, {"policy": "cachesage", "prefetch": False}))
    o = tiny_spec(1, 1, 9)
    o["turns_min"] = o["turns_max"] = 1
    o["task_tokens"] = 512
    o["history_growth"] = 0
    o["budget_blocks"] = 10
    cases.append(("oversized-solo", o, {"policy": "lru"}))
    o2 = tiny_spec(1, 3, 9)
    o2["task_tokens"] = 512
    o2["history_growth"] = 16
    o2["budget_blocks"] = 30
    o2["concurrency"] = 2
    cases.append(("oversized-mixed", o2, {"policy": "cachesage"}))
    p = tiny_spec(1, 2, 9)
    p["turns_min"] = p["turns_max"] = 1
    p["task_tokens"] = 256 - 16 - 160
    p["history_growth"] = 0
    p["concurrency"] = 2
    p["budget_blocks"] = 16
    cases.append(("pins-defer", p, {"policy": "lru"}))
    sa = W.preset_by_name("supervisor-a")
    cases.append(("supervisor-a-noprefetch", sa, {"policy": "cachesage", "prefetch": False}))
    cases.append(("supervisor-a-conc8", sa, {"policy": "cachesage", "concurrency": 8}))
    cases.append(("supervisor-a-budget60", sa, {"policy": "cachesage", "budget": 60}))
    cases.append(("supervisor-a-emax3", sa, {"policy": "cachesage", "e_max": 3}))
    cases.append(("supervisor-a-emax14", sa, {"policy": "cachesage", "e_max": 14}))
    cases.append(("supervisor-a-wpred0.5", sa, {"policy": "cachesage", "w_pred": 0.5}))
    cases.append(("supervisor-a-wpred3", sa, {"policy": "cachesage", "w_pred": 3.0}))
    cases.append(("supervisor-a-tau0.2", sa, {"policy": "cachesage", "tau": 0.2}))
    cases.append(("supervisor-a-gate", sa, {"policy": "cachesage", "min_confidence": 0.3, "min_row_count": 2,
                                             "budget_per_step": 3}))
    cases.append(("supervisor-a-window16", sa, {"policy": "cachesage", "window": 16}))
    cases.append(("supervisor-a-skip2take6", sa, {"policy": "cachesage", "skip": 2, "take": 6}))
    cases.append(("supervisor-a-bs8", sa, {"policy": "cachesage", "block_size": 8}))
    ch = W.preset_by_name("synthetic-chain")
    cases.append(("chain-budget120", ch, {"policy": "cachesage", "budget": 120}))
    # the Belady baseline (baselines.cpp:34-70) on the same pool: every preset, tight budgets,
    # oversized prompts, pins, concurrency
    for s in W.preset_workloads():
        cases.append((s["name"], s, {"policy": "belady"}))
    for b in (128, 256, 4096, 16384, 65536):  # (the last two run the radix select over > kBelCand slots)
        cases.append((f"cfg1@{b}", W.cfg1(b), {"policy": "belady", "budget": b}))
    cases.append(("tiny-alternation-belady", t, {"policy": "belady", "prefetch": False}))
    cases.append(("oversized-solo", o, {"policy": "belady"}))
    cases.append(("oversized-mixed", o2, {"policy": "belady"}))
    cases.append(("pins-defer", p, {"policy": "belady"}))
    cases.append(("supervisor-a-conc8", sa, {"policy": "belady", "concurrency": 8}))
    cases.append(("supervisor-a-budget60", sa, {"policy": "belady", "budget": 60}))
    cases.append(("chain-budget120", ch, {"policy": "belady", "budget": 120}))
    return cases


def main():
    assert refshim.available(), "build oracle/_ref first: make -C oracle ref"
    out = {"source": "oracle/_ref (unmodified reference compiled in place)", "runs": []}
    for name, spec, kw in run_cases():
        r = refshim.run(spec, **kw)
        out["runs"].append({
            "name": name, "spec": spec, "kw": kw,
            "turns": int(r["cached_tokens"].size), "hit_rate": repr(r["hit_rate"]),
            "evictions": int(r["evictions"].size), "evictions_fnv": fnv(r["evictions"]),
            "first_evictions": [hex(int(x)) for x in r["evictions"][:16]],
            "cached_fnv": fnv(r["cached_tokens"].astype(np.int64)),
            "end_us_fnv": fnv(r["end_us"].view(np.uint64)),
            "warmups": [[int(s), hex(int(t)), int(k)] for s, t, k in
                        zip(r["warmup_step"], r["warmup_target"], r["warmup_tick"])][:200],
            "n_warmups": int(r["warmup_step"].size),
            "warmups_fnv": fnv(r["warmup_target"]),
            "steps": int(r["n_steps"]), "truncated": int(r["truncated"]),
            "warmups_executed": int(r["warmups_executed"]), "sim_us": repr(r["sim_us"]),
        })
    with open(os.path.join(HERE, "runs.json"), "w") as f:
        json.dump(out, f, indent=1)

    # K1: chain_hash / block_keys_for / derive_agent_identity
    rng = np.random.default_rng(2605)
    hashes = []
    for n in (1, 2, 3, 15, 16, 17, 35, 64, 100, 257):
        toks = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
        for bs in (1, 7, 16):
            k, c = refshim.block_keys(toks, bs)
            hashes.append({"tokens": [int(x) for x in toks], "block_size": bs, "keys": [hex(int(x)) for x in k],
                           "counts": [int(x) for x in c]})
    idents = []
    for n in (1, 3, 4, 5, 7, 8, 9, 20):
        keys = rng.integers(0, 2**63, size=n, dtype=np.uint64)
        for skip, take in ((4, 4), (0, 1), (2, 6)):
            idents.append({"keys": [hex(int(x)) for x in keys], "skip": skip, "take": take,
                           "identity": hex(refshim.identity(keys, skip, take))})
    kats = {"chain_hash_123": hex(refshim.chain_hash(None, [1, 2, 3])),
            "chain_hash_parent": hex(refshim.chain_hash(0x1234, [5]))}
    with open(os.path.join(HERE, "hashing.json"), "w") as f:
        json.dump({"kats": kats, "block_keys": hashes, "identity": idents}, f, indent=1)

    # generator: per preset / cfg1 the turn table FNV + head
    gens = []
    for s in W.preset_workloads() + [W.cfg1()]:
        t = refshim.generate(s)
        gens.append({"name": s["name"], "spec": s, "n": int(t.shape[0]), "fnv": fnv(t.astype(np.uint64).reshape(-1)),
                     "head": t[:20].tolist()})
    with open(os.path.join(HERE, "generator.json"), "w") as f:
        json.dump(gens, f, indent=1)

    # policy traces: dispatch streams -> rebuild flags, warmup targets, hops, survival, row totals
    pol = []
    for seed, n_agents, n_ev, kw in ((1, 4, 200, {}), (2, 12, 600, {}), (3, 40, 3000, {"window": 64}),
                                     (4, 6, 400, {"tau": 0.3, "e_max": 3}), (5, 9, 500, {"min_confidence": 0.2})):
        r = np.random.default_rng(seed)
        ids = [int(x) for x in r.integers(1, 2**63, size=n_agents, dtype=np.uint64)]
        nxt = r.integers(0, n_agents, size=n_ev)
        # a biased walk so that some rows clear the prefetch gate
        for i in range(1, n_ev):
            if r.random() < 0.6:
                nxt[i] = (nxt[i - 1] + 1) % n_agents
        has_prev = np.ones(n_ev, np.int32)
        has_prev[0] = 0
        prev = np.array([0] + [ids[x] for x in nxt[:-1]], np.uint64)
        nx = np.array([ids[x] for x in nxt], np.uint64)
        drain = np.ones(n_ev, np.uint8)
        cfg = refshim.run_cfg(**kw)
        rebuilt = np.zeros(n_ev, np.int32)
        warm = np.zeros(n_ev, np.uint64)
        q = np.array(ids, np.uint64)
        hops = np.zeros(n_agents, np.int32)
        surv = np.zeros(n_agents, np.float64)
        tot = np.zeros(n_agents, np.uint64)
        sb = np.zeros(1, np.uint64)
        nb = 8
        bk = r.integers(1, 2**63, size=nb, dtype=np.uint64)
        bha = (np.arange(nb) % 2).astype(np.int32)
        bag = np.array([ids[i % n_agents] for i in range(nb)], np.uint64)
        btouch = np.uint64(n_ev) + np.arange(10, 10 + nb, dtype=np.uint64) * 7  # past the event ticks
        sc = np.zeros(nb, np.float64)
        P = lambda a: a.ctypes.data_as(refshim.C.c_void_p)  # noqa: E731
        rc = refshim.lib().ref_policy_trace(refshim.C.byref(cfg), n_ev, P(has_prev), P(prev), P(nx), P(drain),
                                            P(rebuilt), P(warm), n_agents, P(q), P(hops), P(surv), P(tot), nb,
                                            P(bk), P(bha), P(bag), P(btouch), int(btouch.max()) + 50,
                                            int(btouch.min()), P(sc), P(sb))
        assert rc == 0, refshim._err()
        pol.append({"seed": seed, "kw": kw, "agents": [hex(x) for x in ids], "next": nxt.tolist(),
                    "rebuilt": rebuilt.tolist(), "warm": [hex(int(x)) for x in warm], "hops": hops.tolist(),
                    "survival": [repr(float(x)) for x in surv], "row_total": [int(x) for x in tot],
                    "blocks": {"keys": [hex(int(x)) for x in bk], "has_agent": bha.tolist(),
                               "agents": [hex(int(x)) for x in bag], "touch": btouch.tolist(),
                               "now": int(btouch.max()) + 50, "oldest": int(btouch.min())},
                    "scores_bits": [hex(int(x)) for x in sc.view(np.uint64)], "state_bytes": int(sb[0])})
    with open(os.path.join(HERE, "policy.json"), "w") as f:
        json.dump(pol, f, indent=1)
    print("wrote", len(out["runs"]), "runs,", len(hashes), "hash cases,", len(gens), "generator cases,",
          len(pol), "policy traces")


if __name__ == "__main__":
    main()
