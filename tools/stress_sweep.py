"""cfg5-style stress sweep: the bench engine (cfg4 mixed 256-agent trace, the
pipelined per-admission launch) against pre-filled pools of 1M-64M slots in the realistic and the
adversarial (40% agent-carrying, Zipf) composition. Prints one JSON line per point: slots scored
per second, roofline fraction of the scoring launches, evictions/s, prescan reuse."""
import json
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2605_27744_b200 as cb  # noqa: E402
from paper_2605_27744_b200 import workloads as W  # noqa: E402

pools = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1048576", "4194304", "16777216", "67108864"])]
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["realistic", "adversarial"]
peak, _ = bench.measured_peak()
for mode in modes:
    for pool in pools:
        t = time.time()
        spec = W.cfg4_mixed(sessions=40000, budget=pool, seed=2608)
        eng = cb.Engine(spec, policy="cachesage", budget=pool, timing=True, agent_capacity=1024)
        keys, lt, agents, refs = W.pool_snapshot(pool, len(eng.agents()), seed=11, mode=mode)
        eng.restore(keys, lt, agents=agents, refs=refs)
        del keys, lt, agents, refs
        build_s = time.time() - t
        eng.run_timed(96)
        r0, p0 = eng.result(), eng.pool_stats()
        ms = sum(eng.run_timed(32)[0] for _ in range(5))
        r1, p1 = eng.result(), eng.pool_stats()
        scans = r1["scan_launches"] - r0["scan_launches"]
        avg = (r1["scan_ms"] - r0["scan_ms"]) / max(scans, 1) / 1e3
        line = {"mode": mode, "pool": pool, "value_slots_per_s": (r1["scanned_slots"] - r0["scanned_slots"]) / (ms / 1e3),
                "ms_per_step": ms / 5, "avg_scan_launch_us": avg * 1e6,
                "frac": 16 * pool / avg / 1e9 / peak if scans else None,
                "evictions_per_s": (r1["evictions"] - r0["evictions"]) / (ms / 1e3),
                "prescan_used": p1["prescan_used"] - p0["prescan_used"],
                "prescan_fallbacks": p1["prescan_fallbacks"] - p0["prescan_fallbacks"],
                "prescan_unusable": p1["prescan_unusable"] - p0["prescan_unusable"],
                "rescans": None, "build_s": round(build_s, 1)}
        print(json.dumps(line), flush=True)
        eng.close()
