"""Fixtures for the Policy / Runtime surface beyond the scoring loop: Runtime::dispatch_event over
every Event kind, CacheSagePolicy::serialize_state().dump(), predict / predict_next and
poll_actions (runtime.cpp:59-90, cachesage_policy.cpp:50-153, baselines.cpp). Produced by the
UNMODIFIED reference (oracle/_ref through tests/refshim.py::policy_events), written to
tests/golden/policy_state.json. Run here (needs oracle/_ref): python tests/golden/make_policy_state.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import refshim  # noqa: E402


def stream(seed, n_agents, n_events):
    """A mixed observe stream: arrivals, tool returns, touches, completions and dispatches whose
    successor follows a skewed transition matrix (so the prefetch gate fires), nondecreasing ticks
    (with repeats), drains and checkpoints at random points."""
    rng = np.random.default_rng(seed)
    ids = [int(x) for x in rng.integers(1, 2**63, size=n_agents, dtype=np.int64)]
    trans = rng.dirichlet(np.full(n_agents, 0.3), size=n_agents)
    for a in range(n_agents):  # one dominant successor per agent
        trans[a] *= 0.3
        trans[a, (a * 7 + 3) % n_agents] += 0.7
    ev = []
    tick = 0
    cur = None
    for i in range(n_events):
        tick += int(rng.choice([0, 1, 1, 2]))
        r = rng.random()
        e = {"tick": tick, "request": int(rng.integers(0, 10**6))}
        if r < 0.55:
            nxt = int(rng.choice(n_agents, p=trans[cur])) if cur is not None else int(rng.integers(n_agents))
            e.update(kind=2, agent=ids[nxt], prev=None if (cur is None or rng.random() < 0.03) else ids[cur])
            cur = nxt
        elif r < 0.70:
            e.update(kind=1, agent=ids[int(rng.integers(n_agents))])
        elif r < 0.78:
            e.update(kind=3, agent=ids[int(rng.integers(n_agents))])
        elif r < 0.90:
            e.update(kind=0, agent=ids[int(rng.integers(n_agents))])
        else:
            e.update(kind=4, agent=0)
        e["drain"] = bool(rng.random() < 0.3)
        e["ckpt"] = bool(rng.random() < 0.015) or i == n_events - 1
        ev.append(e)
    return ids, ev


CASES = [
    ("default-12", 1, 12, 400, {"policy": "cachesage"}),
    ("window16-emax3", 2, 9, 500, {"policy": "cachesage", "window": 16, "e_max": 3}),
    ("gate-loose-budget2", 3, 6, 300, {"policy": "cachesage", "min_confidence": 0.3, "min_row_count": 2,
                                       "budget_per_step": 2}),
    ("tau0.2-40", 4, 40, 900, {"policy": "cachesage", "tau": 0.2, "window": 64}),
    ("wpred3-emax14", 5, 20, 600, {"policy": "cachesage", "w_pred": 3.0, "e_max": 14}),
    ("lru", 6, 5, 120, {"policy": "lru"}),
    ("ttl", 7, 5, 120, {"policy": "ttl"}),
]


def main():
    out = []
    for name, seed, na, ne, kw in CASES:
        ids, ev = stream(seed, na, ne)
        cps, err = refshim.policy_events(ev, **kw)
        assert err is None, (name, err)
        out.append({"name": name, "kw": kw, "agents": [hex(x) for x in ids], "events": ev, "checkpoints": cps})
        print(name, len(ev), "events", len(cps), "checkpoints", sum(len(c["drained"]) for c in cps), "warmups")
    # a tick regression: the reference throws runtime_error at that event (runtime.cpp:59-64)
    ids, ev = stream(8, 4, 60)
    ev[40]["tick"] = ev[39]["tick"] - 1
    for e in ev[41:]:
        e["tick"] = max(e["tick"], ev[39]["tick"])
    cps, err = refshim.policy_events(ev, policy="cachesage")
    assert err is not None and err[0] == 40, err
    out.append({"name": "tick-regression", "kw": {"policy": "cachesage"}, "agents": [hex(x) for x in ids],
                "events": ev, "fail_at": err[0], "error": err[1]})
    with open(os.path.join(HERE, "policy_state.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_policy_state.py", "cases": out, "cells": cells()}, f, indent=0)


CELLS = [  # whole simulation cells: the final serialize_state() and a non-default CostModel
    ("supervisor-a", None, {"policy": "cachesage"}),
    ("cfg1", 128, {"policy": "cachesage"}),
    ("synthetic-chain", 120, {"policy": "cachesage", "window": 16}),
    ("supervisor-a", None, {"policy": "cachesage", "cost": [500.0, 20.0, 9000.0]}),
    ("cfg1", 256, {"policy": "cachesage", "cost": [3000.0, 7.5, 41000.0]}),
    ("supervisor-a", 60, {"policy": "lru", "cost": [100.0, 90.0, 15000.0]}),
]


def cells():
    from paper_2605_27744_b200 import workloads as W

    out = []
    for name, budget, kw in CELLS:
        spec = W.cfg1(budget) if name == "cfg1" else W.preset_by_name(name)
        rkw = dict(kw)
        if budget:
            rkw["budget"] = budget
        if "cost" in rkw:
            rkw["cost"] = tuple(rkw["cost"])
        r = refshim.run(spec, **rkw)
        f = lambda a: hex(refshim.fnv1a64(np.ascontiguousarray(a, dtype="<u8")))  # noqa: E731
        out.append({"name": name, "budget": budget, "kw": kw, "spec": spec, "hit_rate": repr(r["hit_rate"]),
                    "evictions": int(r["evictions"].size), "evictions_fnv": f(r["evictions"]),
                    "end_us_fnv": f(r["end_us"].view(np.uint64)), "cached_fnv": f(r["cached_tokens"].astype(np.int64)),
                    "sim_us": repr(r["sim_us"]), "state": refshim.last_state()})
        print("cell", name, budget, kw, out[-1]["hit_rate"], out[-1]["evictions"])
    return out


if __name__ == "__main__":
    main()
