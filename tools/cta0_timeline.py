"""CTA-0 serial chain of the admission kernel on the bench workload (cfg4, 16M pool): mean
%globaltimer offsets (us) of the sub-phase stamps (pstamp) over steady-state scoring launches,
plus the prescan CTAs' stream end."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2605_27744_b200 import workloads as W  # noqa: E402
from paper_2605_27744_b200._lib import lib  # noqa: E402

NAMES = {0: "p0 start", 1: "table queue", 2: "unpins", 3: "probe", 13: "record", 14: "bfs", 4: "observe",
         5: "phase0 end", 6: "prologue", 7: "lists seen", 8: "validate", 9: "consume end", 10: "replay_apply",
         11: "epilogue", 12: "status"}
pool = 16 << 20
spec, seed = bench.rank_workload(40000, pool, 0)
eng = bench.build_engine(W, spec, pool, 0, False, seed)
eng.run_timed(int(sys.argv[1]) if len(sys.argv) > 1 else 100)
rows = []
wr = []
fnd = []
dsub = []
svc = []
ends = []
for it in range(40):
    eng.run_timed(1)
    buf = (C.c_uint64 * (16 * 1024))()
    grid = C.c_int(0)
    rc = lib().cs_pool_debug(lib().cs_engine_pool(eng.h), buf, 16 * 1024, C.byref(grid))
    assert rc == 0, (rc, lib().cs_last_error())
    g = grid.value
    d = np.array(buf[:16 * g + 64], dtype=np.int64)
    ent = d[9]  # CTA 0 kernel entry
    st = d[16 * g:16 * g + 16]
    rows.append((st - ent) / 1e3)
    per = d[:16 * g].reshape(g, 16)
    # service CTAs: 1 = table queue (start, done), 2 = list service (start, gathered, published)
    dsub.append(((per[0, 10:16] - ent) / 1e3))
    if os.environ.get("CS_DEBUG_WARPS"):
        full = np.array(buf[:16 * g + 256], dtype=np.int64)
        fnd.append([(full[16 * g + 100 + 4 * w + k] - ent) / 1e3 for w in range(3) for k in range(4)])
        wr.append(np.concatenate([(full[16 * g + 48:16 * g + 65] - ent) / 1e3, (full[16 * g + 72:16 * g + 89] - ent) / 1e3]))
    svc.append([(per[1, 6] - ent) / 1e3, (per[1, 7] - ent) / 1e3, (per[2, 6] - ent) / 1e3, (per[2, 7] - ent) / 1e3,
                (per[2, 8] - ent) / 1e3] + [(per[3, c] - ent) / 1e3 for c in (6, 7, 8, 9)])
    # streaming CTAs 4..: start, stream end, writeout end (= verdict wait start), verdict seen
    ends.append([((per[4:, c] - ent) / 1e3).max() for c in (0, 1, 4, 5)])
# the admission server's trace ring over runs of 8 consecutive admissions (one server launch)
srv = []
for it in range(10):
    eng.run_timed(8)
    buf = (C.c_uint64 * (16 * 1024))()
    grid = C.c_int(0)
    lib().cs_pool_debug(lib().cs_engine_pool(eng.h), buf, 16 * 1024, C.byref(grid))
    g = grid.value
    ring = np.array(buf[16 * g + 192:16 * g + 256], dtype=np.int64).reshape(8, 8)
    order = np.argsort(ring[:, 0])
    ring = ring[order]
    for k in range(7):
        a, b = ring[k], ring[k + 1]
        if a[0] <= 0 or b[0] <= a[0]:
            continue
        srv.append([(a[1] - a[0]) / 1e3, (a[2] - a[0]) / 1e3, (a[3] - a[0]) / 1e3, (a[4] - a[0]) / 1e3,
                    (a[5] - a[0]) / 1e3, (a[6] - a[0]) / 1e3, (b[0] - a[0]) / 1e3])
r = np.median(np.array(rows), axis=0)
ds = np.median(np.array(dsub), axis=0)
if wr:
    w = np.median(np.array(wr), axis=0)
    print("phase 0 round 1, per warp end (us):", " ".join("%.1f" % x for x in w[:17]))
    print("phase 0 round 2, per warp end (us):", " ".join("%.1f" % x for x in w[17:]))
    f = np.array(fnd)
    print("finds (lane 0 of warps 0-2): start / key loaded / found / found again (us):")
    for k in range(3):
        print("  warp %d: %.2f %.2f %.2f %.2f" % (k, np.median(f[:, 4 * k]), np.median(f[:, 4 * k + 1]),
                                                np.median(f[:, 4 * k + 2]), np.median(f[:, 4 * k + 3])))
print("replay_apply sub-phases (us from CTA 0 entry): start %.2f lists %.2f bulk decided %.2f prep %.2f victim keys %.2f end %.2f"
      % tuple(ds))
for k in [0, 1, 2, 3, 13, 14, 4, 5, 6, 7, 9, 10, 11, 12]:
    print(f"{NAMES[k]:>14}: {r[k]:8.2f} us")
e = np.median(np.array(ends), axis=0)
print("streaming CTAs (max over CTAs): start %.2f stream end %.2f writeout %.2f verdict seen %.2f us" % tuple(e))
sv = np.median(np.array(svc), axis=0)
print("service CTA 1 (table queue): start %.2f done %.2f us; CTA 2 (lists): start %.2f gathered %.2f published %.2f us"
      % tuple(sv[:5]))
print("learner service CTA 3: start %.2f window loaded %.2f BFS done %.2f published %.2f us" % tuple(sv[5:]))
if srv:
    v = np.median(np.array(srv), axis=0)
    print("admission server, us after the pickup (median over %d consecutive pairs):" % len(srv))
    for name, x in zip(["admit_body entry", "phase 0 end", "early status ready (CTA 0)", "status published (CTA 1)",
                        "CTA 0 done", "streamers saw the verdict", "NEXT admission picked up"], v):
        print("  %28s: %8.2f" % (name, x))
ps = eng.pool_stats()
if ps["host_turnarounds"]:
    print("host turnaround (status seen -> next post): %.2f us mean over %d" % (
        ps["host_turnaround_ns"] / ps["host_turnarounds"] / 1e3, ps["host_turnarounds"]))
res = eng.result()
print("admit_ms per launch", res["admit_ms"] / max(res["admissions"], 1) * 1e3)
