"""Per-CTA timeline of the last scoring launch of the bench engine (cfg4, 16M pool)."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2605_27744_b200 import workloads as W  # noqa: E402
from paper_2605_27744_b200._lib import lib  # noqa: E402

pool = 16 << 20
spec, seed = bench.rank_workload(40000, pool, 0)
eng = bench.build_engine(W, spec, pool, 0, False, seed)
eng.run_timed(200)
for it in range(6):
    r0 = eng.result()
    eng.run_timed(1)
    r1 = eng.result()
    if r1["scan_launches"] == r0["scan_launches"]:
        continue
    buf = (C.c_uint64 * (16 * 1024))()
    grid = C.c_int(0)
    lib().cs_pool_debug(lib().cs_engine_pool(eng.h), buf, 16 * 1024, C.byref(grid))
    d = np.array(buf[:16 * grid.value], dtype=np.int64).reshape(grid.value, 16)
    t0 = d[:, 9].min()  # kernel entry
    rel = (d - t0) / 1e3
    o = rel[1:]
    print(f"launch: {(r1['admit_ms'] - r0['admit_ms']) * 1e3:.1f} us (events); entry spread {rel[:, 9].max():.1f}; "
          f"scan start med {np.median(o[:, 0]):.1f}; stream end med/max {np.median(o[:, 1]):.1f}/{o[:, 1].max():.1f}; "
          f"flush end max {o[:, 2].max():.1f}; writeout max {o[:, 3].max():.1f}; barrier exit {rel[:, 4].max():.1f}; "
          f"cta0 scan start {rel[0, 0]:.1f} flush end {rel[0, 2]:.1f} writeout {rel[0, 3]:.1f}; staged med {np.median(d[1:, 5]):.0f} "
          f"max {d[1:, 5].max()}; fast {bool(d[1, 8])}")
