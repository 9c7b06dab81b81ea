"""Belady admission rate on the GPU engine (cfg4 mixed trace, 3000 sessions) at three budgets."""
import sys, time
sys.path.insert(0, ".")
import paper_2605_27744_b200 as cb
from paper_2605_27744_b200 import workloads as W
for b in (4096, 16384, 65536):
    spec = W.cfg4_mixed(sessions=3000, budget=b)
    eng = cb.Engine(spec, policy="belady", agent_capacity=1024)
    t = time.time(); res = eng.run(); dt = time.time() - t
    r = eng.result(); eng.close()
    print(b, res["hit_rate"], r["admissions"] / dt, "adm/s")
