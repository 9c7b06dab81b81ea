"""Debug aid: the bench configuration with an adversarial snapshot, N admissions (argv: pool, n)."""
import sys
sys.path.insert(0, ".")
import paper_2605_27744_b200 as cb
from paper_2605_27744_b200 import workloads as W
pool = int(sys.argv[1]); n = int(sys.argv[2]); mode = sys.argv[3] if len(sys.argv) > 3 else "adversarial"
spec = W.cfg4_mixed(sessions=40000, budget=pool, seed=2608)
eng = cb.Engine(spec, policy="cachesage", budget=pool, agent_capacity=1024, prefetch=True)
keys, lt, agents, refs = W.pool_snapshot(pool, len(eng.agents()), seed=11, mode=mode)
eng.restore(keys, lt, agents=agents, refs=refs)
done = 0
step = int(sys.argv[4]) if len(sys.argv) > 4 else 50
try:
    while done < n:
        eng.run_for(step)
        done += step
except Exception as e:
    print("FAILED after", done, "admissions:", e, eng.pool_stats() if False else "")
    raise
print("ok", eng.result()["admissions"], eng.pool_stats()["prescan_fallbacks"], eng.check())
