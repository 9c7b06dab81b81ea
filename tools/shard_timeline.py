"""Sharded admission at N=1 on the bench workload (cfg4, 16M shard, peer exchange): mean
%globaltimer offsets (us, from the probe kernel's entry) of the phase stamps (shstamp in
csrc/cs_shard.cuh) over steady-state admissions that scanned."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2605_27744_b200 import shard  # noqa: E402
from paper_2605_27744_b200 import workloads as W  # noqa: E402
from paper_2605_27744_b200._lib import lib  # noqa: E402

NAMES = ["probe entry", "table queue", "unpins", "probe end", "decide entry", "decide end", "scan entry",
         "scan pass+barrier", "finalize+barrier", "scan end", "replay entry", "prologue", "merge",
         "replay loop", "apply", "replay end"]
pool = 16 << 20
spec, seed = bench.rank_workload(40000, pool, 0)
comm = shard.PeerComm(0, 1, 0, lambda b: [b])
eng = bench.build_engine(W, spec, pool, 0, False, seed, comm=comm)
eng.run_timed(int(sys.argv[1]) if len(sys.argv) > 1 else 100)
rows = []
cta = []
loop = []
for it in range(60):
    eng.run_timed(1)
    buf = (C.c_uint64 * (16 * 1024))()
    grid = C.c_int(0)
    rc = lib().cs_pool_debug(lib().cs_engine_pool(eng.h), buf, 16 * 1024, C.byref(grid))
    assert rc == 0, (rc, lib().cs_last_error())
    g = grid.value
    d = np.array(buf[:16 * g], dtype=np.int64).reshape(g, 16)
    st = np.concatenate([d[8, 10:16], d[9, 10:16], d[10, 10:16]])[:16]
    if st[6] <= st[0] or st[10] <= st[6]:
        continue  # an admission that did not scan
    rows.append((st - st[0]) / 1e3)
    loop.append([d[10, 14], d[10, 15] & ((1 << 48) - 1), d[10, 15] >> 48, d[0, 14] if False else 0])
    # scanning CTAs: stream start / stream end / flushed / published (us from scan entry), fast pass
    cta.append([((d[:, c] - st[6]) / 1e3).max() for c in (0, 1, 2, 3)] + [d[:, 8].mean(), d[:, 5].mean()])
r = np.array(rows)
print(f"{len(rows)} scanning admissions of a sharded pool at N=1 (16M-slot shard); us from probe entry")
for k, n in enumerate(NAMES):
    print(f"  {k:2d} {n:20s} {np.mean(r[:, k]):8.2f}  (median {np.median(r[:, k]):8.2f})")
c = np.array(cta)
print("scan CTAs (max over CTAs, us from scan entry): stream start %.2f, stream end %.2f, flushed %.2f, "
      "published %.2f; fast-pass fraction %.2f; staged candidates per CTA %.1f" % tuple(np.mean(c, axis=0)))
lp = np.array(loop, dtype=np.float64)
print("replay loop: %.0f SM cycles, of which %.0f in evict_one loops; %.1f evictions per admission"
      % (lp[:, 1].mean(), lp[:, 0].mean(), lp[:, 2].mean()))
