"""The LRU <= CacheSage <= Belady sandwich at scale (acceptance criterion 2) on the
GPU engine: the SURVEY cfg2 (hierarchical, 32 agents, prefetch off), cfg3 (swarm, 128 agents) and
cfg4 (mixed, 256 agents) traces, ~200K requests each, at pool budgets where eviction choices
matter (at 1M+ blocks these traces' reusable working set fits and all three policies tie).
Prints one JSON line per (config, budget, policy): hit rate, evictions, admissions/s.

    python tools/sandwich_scale.py [sessions] [budgets, comma-separated]
"""
import json
import sys
import time

sys.path.insert(0, ".")
import paper_2605_27744_b200 as cb  # noqa: E402
from paper_2605_27744_b200 import workloads as W  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
budgets = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["2048", "16384"])]
cases = []
for b in budgets:
    cases += [("cfg2-hierarchical", W.cfg2_hierarchical(sessions=S, budget=b), {"prefetch": False}),
              ("cfg3-swarm", W.cfg3_swarm(sessions=S, budget=b), {}),
              ("cfg4-mixed", W.cfg4_mixed(sessions=S, budget=b), {})]
for name, spec, kw in cases:
    for pol in ("lru", "cachesage", "belady"):
        t = time.time()
        eng = cb.Engine(spec, policy=pol, agent_capacity=1024, **kw)
        t_build = time.time() - t
        t = time.time()
        res = eng.run()
        dt = time.time() - t
        r = eng.result()
        eng.close()
        print(json.dumps({"config": name, "policy": pol, "budget": spec["budget_blocks"], "sessions": S,
                          "turns": r["turns"], "hit_rate": res["hit_rate"], "evictions": r["evictions"],
                          "admissions": r["admissions"], "run_s": round(dt, 2),
                          "admissions_per_s": round(r["admissions"] / dt, 1), "build_s": round(t_build, 2)}), flush=True)
