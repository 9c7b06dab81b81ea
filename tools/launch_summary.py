"""Per-kernel median duration of an ncu launch list (gpu__time_duration.sum, --csv)."""
import collections
import csv
import sys

rows = [ln for ln in open(sys.argv[1]) if ln.startswith('"')]
d = collections.defaultdict(list)
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
for r in csv.DictReader(rows):
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    d[r["Kernel Name"].split("(")[0]].append(float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1.0))
for k, v in d.items():
    v = sorted(v)
    print(f"{k:40s} n={len(v):4d} median={v[len(v) // 2]:8.2f} us  max={v[-1]:8.2f} us")
