"""Diagnostic: first admission where the device scheduler diverges from the host scheduler."""
import os, subprocess, sys, json
import numpy as np
sys.path.insert(0, ".")
name, pol = sys.argv[1], sys.argv[2]
if len(sys.argv) > 3 and sys.argv[3] == "child":
    import paper_2605_27744_b200 as cb
    spec = cb.preset_by_name(name)
    eng = cb.Engine(spec, policy=pol, agent_capacity=1024)
    rows = []
    prev = 0
    for k in range(int(sys.argv[4])):
        d = eng.run_for(1)
        ev = eng.evictions()
        r = eng.result()
        rows.append([int(r["admissions"]), int(ev.size), int(ev[prev:].astype(np.uint64).sum() & 0xFFFFFFFF) if ev.size > prev else 0,
                     int(r["tick"]), int(r["scans"])])
        prev = ev.size
        if d:
            break
    print(json.dumps(rows))
    sys.exit(0)
res = {}
for mode, env in [("host", {"CS_DEVICE_SCHED": "0"}), ("dev", {"CS_DEVICE_SCHED": "1"})]:
    r = subprocess.run([sys.executable, __file__, name, pol, "child", "400"], env=dict(os.environ, **env),
                       capture_output=True, text=True)
    res[mode] = json.loads(r.stdout.strip().splitlines()[-1]) if r.stdout.strip() else r.stderr[-500:]
h, d = res["host"], res["dev"]
if isinstance(d, str) or isinstance(h, str):
    print(res)
    sys.exit(0)
for i, (a, b) in enumerate(zip(h, d)):
    if a[:4] != b[:4]:
        print("first divergence at step", i, "host", a, "dev", b, "prev", h[i - 1] if i else None)
        break
else:
    print("no divergence in", len(h), "steps")
