"""Diagnostic: where the device scheduler's eviction sequence departs from the host one."""
import os, subprocess, sys, json
import numpy as np
sys.path.insert(0, ".")
name, pol = sys.argv[1], sys.argv[2]
if len(sys.argv) > 3:
    import paper_2605_27744_b200 as cb
    eng = cb.Engine(cb.preset_by_name(name), policy=pol, agent_capacity=1024)
    if sys.argv[3] == "steps":
        bounds = []
        while not eng.run_for(1):
            bounds.append(int(eng.evictions().size))
        bounds.append(int(eng.evictions().size))
        np.save("/tmp/bounds.npy", np.array(bounds))
    else:
        eng.run()
    np.save(sys.argv[4], eng.evictions())
    sys.exit(0)
for mode, env, how in [("host", "0", "full"), ("dev", "1" if not os.environ.get("CMP_HOST_FULLGRID") else "0", "full"), ("host", "0", "steps")]:
    subprocess.run([sys.executable, __file__, name, pol, how, f"/tmp/ev_{mode}_{how}.npy"],
                   env=dict(os.environ, CS_DEVICE_SCHED=env, CS_PRESCAN=os.environ.get("DEV_PRESCAN", "1") if env == "1" else "1",
                            CS_SPECULATE=os.environ.get("DEV_SPEC", "1") if env == "1" else "1",
                            CS_USE_PRESCAN=os.environ.get("DEV_USE", "1"), CS_FULL_GRID="1" if (mode == "dev" and os.environ.get("CMP_HOST_FULLGRID")) else "0"), check=True)
h = np.load("/tmp/ev_host_full.npy"); d = np.load("/tmp/ev_dev_full.npy"); b = np.load("/tmp/bounds.npy")
n = min(h.size, d.size)
diff = np.nonzero(h[:n] != d[:n])[0]
print("sizes", h.size, d.size, "ndiff", diff.size)
if diff.size:
    i = int(diff[0])
    adm = int(np.searchsorted(b, i, side="right"))
    lo = int(b[adm - 1]) if adm else 0
    print("first diff at eviction", i, "admission", adm, "its evictions", lo, "..", int(b[adm]))
    print("host", [hex(int(x)) for x in h[lo:min(lo + 12, h.size)]])
    print("dev ", [hex(int(x)) for x in d[lo:min(lo + 12, d.size)]])
    print("same multiset in that admission:", sorted(h[lo:b[adm]].tolist()) == sorted(d[lo:b[adm]].tolist()))
