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
    b = d[:, 4].max()
    print("  after barrier (us): finalize end cta1/cta0 %.1f/%.1f" % tuple((np.array([d[1, 10], d[1, 11]]) - b) / 1e3))
    c = d[0, 10:16].astype(np.float64)
    f = d[2, 10:15].astype(np.float64)
    mhz = 1965.0
    print("  replay (us from start, SM clock): lists %.2f checks-start %.2f checks-end %.2f bulk %.2f setup-end %.2f "
          "vkeys %.2f apply-end %.2f" % ((c[1] - c[0]) / mhz, (d[3, 10] - c[0]) / mhz, (d[3, 11] - c[0]) / mhz,
                                         (c[2] - c[0]) / mhz, (c[3] - c[0]) / mhz, (c[4] - c[0]) / mhz, (c[5] - c[0]) / mhz))
    print("  finalize E by CTA0 (us): minima %.2f filter %.2f rank %.2f finish %.2f; mf %d m %d" % (
        (f[1] - f[0]) / mhz, (f[2] - f[0]) / mhz, (f[3] - f[0]) / mhz, (f[4] - f[0]) / mhz, d[2, 15] & 0xffffffff, d[2, 15] >> 32))
