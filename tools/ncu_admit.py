"""Driver for ncu captures of the admission kernel in the bench workload (cfg4, 16M pool):
runs `--skip` admissions, then `--n` more (the ones a `ncu -k regex:admit_kernel -s SKIP`
capture sees). Not part of the product path."""
import argparse
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2605_27744_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--skip", type=int, default=250)
ap.add_argument("--n", type=int, default=3)
ap.add_argument("--pool", type=int, default=16 << 20)
args = ap.parse_args()
spec, seed = bench.rank_workload(40000, args.pool, 0)
eng = bench.build_engine(W, spec, args.pool, 0, False, seed)
eng.run_for(args.skip + args.n)
r = eng.result()
print("admissions", r["admissions"], "scans", r["scans"], "launches", r["gpu_launches"])
