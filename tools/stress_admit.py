"""cfg5-style stress driver: a pre-filled pool snapshot, then admissions of k fresh blocks
(each evicts k victims) through the C ABI. Prints the per-phase device time of the admission
kernel; used under ncu to capture the scan. Not part of the product path."""
import argparse
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2605_27744_b200 as cb  # noqa: E402
from paper_2605_27744_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--pool", type=int, default=16 << 20)
ap.add_argument("--agents", type=int, default=256)
ap.add_argument("--k", type=int, default=64)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--mode", default="realistic")
ap.add_argument("--policy", default="cachesage")
args = ap.parse_args()

g = cb.Pool(args.pool, policy=args.policy)
ids = [int(x) for x in W._splitmix(np.arange(args.agents, dtype=np.uint64) + np.uint64(77))]
g.register_agents(ids)
t = time.time()
keys, lt, agents, refs = W.pool_snapshot(args.pool, args.agents, seed=3, mode=args.mode)
g.restore(keys, lt, agents=agents, refs=refs)
print(f"restore {args.pool} slots: {time.time() - t:.2f}s", flush=True)
tick = int(lt.max())
rng = np.random.default_rng(1)
prev = None
times = []
st0 = g.stats()
for it in range(args.iters):
    a = int(rng.integers(0, args.agents))
    g.observe_dispatch(prev, a, tick + 1)
    tick += 1
    prev = a
    prompt = (rng.choice(2**62, size=args.k).astype(np.uint64) + np.uint64(2**62))
    t0 = time.perf_counter()
    ev, pins = g.admit_pinned(prompt, np.full(args.k, 16, np.int32), agent=a, anchor=8, tick_base=tick)
    times.append(time.perf_counter() - t0)
    tick += args.k
    g.unpin_slots(pins)
st1 = g.stats()
ph = np.array(st1["phase_ns"], dtype=np.float64) - np.array(st0["phase_ns"], dtype=np.float64)
n = args.iters
names = ["probe/observe/lookup", "prep+barrier", "scan+barrier", "select+barrier", "replay(rest)", "epilogue",
         "replay-setup", "replay-loop", "apply", "cta0-flush", "cta0-flushes(x1e3)",
         "fast-evictions", "evictions", "rescans", "bulk-chunks", "-"]
print("per admission (us, CTA-0 globaltimer): " + ", ".join(
    f"{nm}={(v / n if k >= 10 else v / n / 1e3):.1f}" for k, (nm, v) in enumerate(zip(names, ph))))
print(f"host wall per admit call: median {np.median(times) * 1e6:.0f} us; scans={st1['scans'] - st0['scans']}")
print(f"scan roofline at 16 B/slot: {16 * args.pool / (ph[2] / n * 1e-9) / 1e9:.0f} GB/s over the scan phase")

# per-CTA timeline of the last scan (instrumentation buffer)
import ctypes as C
from paper_2605_27744_b200._lib import lib
buf = (C.c_uint64 * (16 * 1024))()
grid = C.c_int(0)
lib().cs_pool_debug(g.h, buf, 16 * 1024, C.byref(grid))
d = np.array(buf[:16 * grid.value], dtype=np.int64).reshape(grid.value, 16)
t0 = d[:, 0].min()
rel = (d[:, :5] - t0) / 1e3
print(f"CTAs={grid.value}: scan start spread {rel[:,0].max():.1f} us; stream end min/med/max "
      f"{rel[:,1].min():.1f}/{np.median(rel[:,1]):.1f}/{rel[:,1].max():.1f}; final flush end max {rel[:,2].max():.1f}; "
      f"writeout end max {rel[:,3].max():.1f}; barrier exit {rel[:,4].max():.1f} us")
ent = (d[:, 9] - t0) / 1e3
print(f"kernel entry rel. to first scan start: min/max {ent.min():.1f}/{ent.max():.1f} us; "
      f"scan start after entry med {np.median(rel[:,0]-ent):.1f} us")
print(f"staged at stream end: med {np.median(d[:,5]):.0f} max {d[:,5].max()}")
mhz = d[:, 6] / ((d[:, 1] - d[:, 0]) / 1e3)
print(f"SM clock during the stream (clock64 / globaltimer): med {np.median(mhz):.0f} MHz (min {mhz.min():.0f})")
print("stream time per CTA (us): min/med/max", np.round(np.percentile(rel[:,1]-rel[:,0],[0,50,100]),1))
nt = 0
print("last scan ran fast (warp-specialized):", bool(d[0, 8]))
