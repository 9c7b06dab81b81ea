"""cfg5 stress sweep: the bench engine (the admission server, one prescan pass per
admission) against pre-filled pools of 1M-64M slots, in the realistic and the adversarial (40%
agent-carrying, Zipf) composition, over the agent count A. A = 256 runs the bench's cfg4 mixed
trace; any other A runs the cfg5 stress trace (4 Dirichlet successors per agent,
workloads.cfg5_stress). Prints one JSON line per point: slots scored per second, per-admission
device time and its roofline fraction, evictions/s, prescan reuse, CTA 0's phase-0 time (probe,
unpins, learner record, BFS, lookup) per admission.

  python tools/stress_sweep.py --pools 1048576,16777216 --agents 8,32,128,256,512,1024
"""
import argparse
import json
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2605_27744_b200 as cb  # noqa: E402
from paper_2605_27744_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--pools", default="1048576,4194304,16777216,67108864")
ap.add_argument("--modes", default="realistic,adversarial")
ap.add_argument("--agents", default="256")
ap.add_argument("--steps", type=int, default=5)
args = ap.parse_args()
pools = [int(x) for x in args.pools.split(",")]
peak, _ = bench.measured_peak()
for mode in args.modes.split(","):
    for A in [int(x) for x in args.agents.split(",")]:
        for pool in pools:
            t = time.time()
            spec = (W.cfg4_mixed(sessions=40000, budget=pool, seed=2608) if A == 256 else
                    W.cfg5_stress(A, sessions=40000, budget=pool))
            eng = cb.Engine(spec, policy="cachesage", budget=pool, timing=True, agent_capacity=max(1024, A))
            keys, lt, agents, refs = W.pool_snapshot(pool, len(eng.agents()), seed=11, mode=mode)
            eng.restore(keys, lt, agents=agents, refs=refs)
            del keys, lt, agents, refs
            build_s = time.time() - t
            eng.run_timed(96)
            r0, p0 = eng.result(), eng.pool_stats()
            ms = sum(eng.run_timed(32)[0] for _ in range(args.steps))
            r1, p1 = eng.result(), eng.pool_stats()
            scans = r1["scan_launches"] - r0["scan_launches"]
            avg = (r1["scan_ms"] - r0["scan_ms"]) / max(scans, 1) / 1e3
            ph = bench._phases(p0["phase_ns"], p1["phase_ns"], scans)
            line = {"mode": mode, "agents": A, "trace": spec["name"], "pool": pool,
                    "value_slots_per_s": (r1["scanned_slots"] - r0["scanned_slots"]) / (ms / 1e3),
                    "ms_per_step": ms / args.steps, "avg_admission_us": avg * 1e6,
                    "frac": 16 * pool / avg / 1e9 / peak if scans else None,
                    "evictions_per_s": (r1["evictions"] - r0["evictions"]) / (ms / 1e3),
                    "admissions_per_s": (r1["admissions"] - r0["admissions"]) / (ms / 1e3),
                    "prescan_used": p1["prescan_used"] - p0["prescan_used"],
                    "prescan_fallbacks": p1["prescan_fallbacks"] - p0["prescan_fallbacks"],
                    "phase0_us": ph.get("phase0"), "build_s": round(build_s, 1)}
            print(json.dumps(line), flush=True)
            eng.close()
