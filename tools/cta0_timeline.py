"""CTA-0 serial chain of the admission kernel on the bench workload (cfg4, 16M pool): mean
%globaltimer offsets (us) of the sub-phase stamps (pstamp) over steady-state scoring launches,
plus the prescan CTAs' stream end."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2605_27744_b200 import workloads as W  # noqa: E402
from paper_2605_27744_b200._lib import lib  # noqa: E402

NAMES = {0: "p0 start", 1: "table queue", 2: "unpins", 3: "probe", 13: "record", 14: "bfs", 4: "observe",
         5: "phase0 end", 6: "prologue", 7: "U set", 8: "validate", 9: "consume end", 10: "replay_apply",
         11: "epilogue", 12: "status"}
pool = 16 << 20
spec, seed = bench.rank_workload(40000, pool, 0)
eng = bench.build_engine(W, spec, pool, 0, False, seed)
eng.run_timed(int(sys.argv[1]) if len(sys.argv) > 1 else 100)
rows = []
fin = []
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
    fin.append([(per[1, c] - ent) / 1e3 for c in (6, 7, 8, 4, 11)])
    ends.append([((per[1:, c] - ent) / 1e3).max() for c in (0, 1, 2, 3, 4, 5)] + [((per[1:3, 4] - ent) / 1e3).max()])
r = np.median(np.array(rows), axis=0)
for k in [0, 1, 2, 3, 13, 14, 4, 5, 6, 7, 8, 9, 10, 11, 12]:
    print(f"{NAMES[k]:>14}: {r[k]:8.2f} us")
e = np.median(np.array(ends), axis=0)
print("prescan CTAs (max over CTAs): start %.2f stream end %.2f writeout %.2f barrier %.2f finish %.2f (finalizers %.2f) verdict %.2f us"
      % (e[0], e[1], e[2], e[3], e[4], e[6], e[5]))
res = eng.result()
print("admit_ms per launch", res["admit_ms"] / max(res["admissions"], 1) * 1e3)

f = np.median(np.array(fin), axis=0)
print("finalizer CTA 1: arrivals seen %.2f staged %.2f ranked %.2f published %.2f us; table queue applied %.2f us" % tuple(f))
