"""Quick GPU-vs-oracle triage: runs each preset/policy and reports the first divergence."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2605_27744_b200 as cb
from paper_2605_27744_b200 import workloads as W
from oracle import pyoracle as orc

def run(spec, policy, budget=None):
    t = time.time()
    e = cb.Engine(spec, policy=policy, budget=budget, timing=True)
    r = e.run(); ev = e.evictions(); tt = e.turns(); st, tg, tk = e.warmups(); e.close()
    g_t = time.time() - t
    t = time.time(); o = orc.run(spec, policy=policy, budget=budget); o_t = time.time() - t
    ok = ev.size == o["evictions"].size and np.array_equal(ev, o["evictions"])
    first = None
    if not ok:
        m = min(ev.size, o["evictions"].size)
        d = np.nonzero(ev[:m] != o["evictions"][:m])[0]
        first = int(d[0]) if d.size else m
    okc = np.array_equal(tt["cached_tokens"], o["cached_tokens"])
    okw = np.array_equal(tg, o["warmup_target"])
    print(f"{spec['name']:28s} {policy:9s} ev={ev.size}/{o['evictions'].size} ev_ok={ok} first_bad={first} "
          f"cached_ok={okc} warm_ok={okw} hit={r['hit_rate']:.6f}/{o['hit_rate']:.6f} "
          f"scans={r['scans']} adm={r['admissions']} gpu_s={g_t:.2f} cpu_s={o_t:.2f} admit_ms={r['admit_ms']:.1f} scan_ms={r['scan_ms']:.1f}",
          flush=True)
    return ok and okc and okw

allok = True
for name in W.preset_names():
    for pol in ("lru", "cachesage"):
        allok &= run(W.preset_by_name(name), pol)
for b in (128, 65536):
    for pol in ("lru", "cachesage"):
        allok &= run(W.cfg1(b), pol, budget=b)
print("ALL_OK" if allok else "MISMATCH")
