"""Turns the ncu launch list of tools/kernel_sweep.py (CSV: gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum per launch) and the sweep's PLAN line into a per-kernel
summary: K1 tokens/s, K2 ns per probe, K3/K3b/K6 microseconds per call over A, each with its
achieved DRAM GB/s.

  python tools/ncu_kernels.py gpurun_out/kernels.csv gpurun_out/kernel_sweep.out > profiles/r02_kernels.json
"""
import csv
import json
import sys
from collections import OrderedDict

UNIT = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "nsecond": 1e-9, "msecond": 1e-3, "ms": 1e-3, "s": 1.0,
        "second": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def launches(path):
    rows = OrderedDict()
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        k = r["ID"]
        d = rows.setdefault(k, {"name": r["Kernel Name"], "grid": r.get("Grid Size"), "block": r.get("Block Size")})
        v = float(r["Metric Value"].replace(",", "")) * UNIT.get(r["Metric Unit"], 1.0)
        d[r["Metric Name"]] = v
    return list(rows.values())


def main():
    ls = launches(sys.argv[1])
    plan = None
    with open(sys.argv[2]) as f:
        for ln in f:
            if ln.startswith("PLAN "):
                plan = json.loads(ln[5:])
    cursor = {}
    out = []
    for p in plan:
        name = p["kernel"]
        mine = [i for i, l in enumerate(ls) if name in l["name"]]
        start = cursor.get(name, 0)
        skip = 1 if p["section"] == "K3" else 0  # the untimed first record_many per A
        idx = mine[start + skip:start + skip + p["reps"]]
        cursor[name] = start + skip + p["reps"]
        t = sorted(ls[i]["gpu__time_duration.sum"] for i in idx)
        byt = sorted(ls[i]["dram__bytes_read.sum"] + ls[i]["dram__bytes_write.sum"] for i in idx)
        med_t = t[len(t) // 2]
        med_b = byt[len(byt) // 2]
        e = dict(p)
        e.update({"launches": len(idx), "device_us_median": med_t * 1e6, "dram_bytes_median": med_b,
                  "achieved_dram_gbs": med_b / med_t / 1e9 if med_t else None})
        if p["section"] == "K1":
            e["tokens_per_s"] = p["tokens_per_call"] / med_t
            e["algorithmic_bytes"] = 4 * p["tokens_per_call"] + 12 * p["blocks_per_call"]
            e["algorithmic_gbs"] = e["algorithmic_bytes"] / med_t / 1e9
        if p["section"] == "K2":
            e["ns_per_probe"] = med_t / p["probes_per_call"] * 1e9
            e["probes_per_s"] = p["probes_per_call"] / med_t
        if p["section"] == "K3":
            e["transitions_per_s"] = p["transitions_per_call"] / med_t
        out.append(e)
    print(json.dumps({"source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                                "--clock-control none (cold, serialized launches) of tools/kernel_sweep.py",
                      "kernels": out}, indent=1))


if __name__ == "__main__":
    main()
