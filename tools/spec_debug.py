"""Finds the first admission whose evictions differ from the oracle (GPU triage tool)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2605_27744_b200 as cb
from paper_2605_27744_b200 import workloads as W
from oracle import pyoracle as orc

name, pol = sys.argv[1], sys.argv[2]
budget = int(sys.argv[3]) if len(sys.argv) > 3 else None
spec = W.cfg1(budget) if name == "cfg1" else W.preset_by_name(name)
o = orc.run(spec, policy=pol, budget=budget)
oe = o["evictions"]
e = cb.Engine(spec, policy=pol, budget=budget)
prev_ev = 0
prev_ph = np.zeros(16)
k = 0
while True:
    done = e.run_for(1)
    ev = e.evictions()
    st = e.result()
    ph = np.array(cb.Pool.stats.__get__(None) if False else [0] * 16, dtype=np.float64)
    m = min(ev.size, oe.size)
    bad = ev.size > oe.size or not np.array_equal(ev[:m], oe[:m])
    if bad:
        d = np.nonzero(ev[:m] != oe[:m])[0]
        f = int(d[0]) if d.size else m
        print(f"first bad admission #{k}: evictions before {prev_ev}, now {ev.size}; first bad index {f}")
        print("gpu :", [hex(int(x)) for x in ev[max(prev_ev, f - 2):f + 4]])
        print("ref :", [hex(int(x)) for x in oe[max(prev_ev, f - 2):f + 4]])
        print("result:", {kk: st[kk] for kk in ("admissions", "steps", "scans", "turns", "completed", "truncated")})
        break
    prev_ev = ev.size
    k += 1
    if done:
        print("no divergence", ev.size, oe.size)
        break
