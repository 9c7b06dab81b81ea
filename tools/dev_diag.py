"""Diagnostic: first divergence of the eviction sequence between scheduler modes."""
import os, subprocess, sys, json
import numpy as np
sys.path.insert(0, ".")
name, pol = sys.argv[1], sys.argv[2]
if len(sys.argv) > 3:
    import paper_2605_27744_b200 as cb
    spec = cb.preset_by_name(name)
    eng = cb.Engine(spec, policy=pol, agent_capacity=1024)
    eng.run()
    np.save(sys.argv[3], eng.evictions())
    r = eng.result()
    print(json.dumps({k: r[k] for k in ("hit_rate", "evictions", "admissions", "steps", "scans")}))
    sys.exit(0)
outs = {}
for mode, env in [("host", {"CS_DEVICE_SCHED": "0"}), ("dev", {"CS_DEVICE_SCHED": "1"}),
                  ("dev_nopre", {"CS_DEVICE_SCHED": "1", "CS_PRESCAN": "0"}), ("host_nopre", {"CS_DEVICE_SCHED": "0", "CS_PRESCAN": "0"})]:
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, __file__, name, pol, f"/tmp/ev_{mode}.npy"], env=e, capture_output=True, text=True)
    print(mode, r.stdout.strip(), r.stderr.strip()[-300:])
    outs[mode] = np.load(f"/tmp/ev_{mode}.npy")
base = outs["host"]
for m, v in outs.items():
    n = min(len(v), len(base))
    d = np.nonzero(v[:n] != base[:n])[0]
    print(m, len(v), "first diff", int(d[0]) if d.size else None, "ndiff", d.size)
