"""Summaries of the committed ncu evidence for the dominant kernel (profiles/).

  python tools/ncu_summarize.py full  <rep.ncu-rep> <launches.csv> > profiles/ncu_admit_summary.json

`full`: one `ncu --set full` capture of admit_kernel (the admission body the server runs, launched
per admission under CS_SERVER=0 so ncu can replay it) plus the launch list of the bench command
(gpu__time_duration + DRAM bytes per launch). The summary records the sha256 prefix of the
libcachesage_b200.so it was taken on: bench.py uses its DRAM bytes per launch as
roofline.traffic only for that same build.
"""
import csv
import hashlib
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
        "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "%": 1.0, "": 1.0}


def lib_sha16():
    with open(os.path.join(ROOT, "paper_2605_27744_b200", "libcachesage_b200.so"), "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()[:16]


def src_sha16():
    sys.path.insert(0, ROOT)
    from paper_2605_27744_b200.build import src_sha16 as f

    return f()


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    return {n: (v[i], u[i]) for i, n in enumerate(h)}


def launch_list(path, kernel="admit_kernel"):
    rows = {}
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if kernel not in r["Kernel Name"]:
            continue
        d = rows.setdefault(r["ID"], {})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * UNIT.get(r["Metric Unit"], 1.0)
    return list(rows.values())


def main():
    rep, lcsv = sys.argv[2], sys.argv[3]
    m = raw_metrics(rep)

    def val(name):
        x, unit = m[name]
        return float(x.replace(",", "")) * UNIT.get(unit, 1.0)

    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    pool = 16 << 20
    ll = launch_list(lcsv)
    # scoring launches only (a launch that streams the pool reads > 64 MB)
    scan = [x for x in ll if x.get("dram__bytes_read.sum", 0) > 64e6]
    keep = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
            "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
            "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second",
            "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio"]
    out = {
        "kernel": "csb::admit_kernel(DevPool, AdmitArgs)",
        "so_sha16": lib_sha16(),
        "src_sha16": src_sha16(),
        "round": 2,
        "command": "CS_SERVER=0 ncu --set full --import-source on --clock-control none -k regex:admit_kernel -s 1600 -c 1 "
                   "python tools/ncu_admit.py --skip 1600 --n 2",
        "launch_list_command": "CS_SERVER=0 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                               "--clock-control none -k regex:admit_kernel -c 400 --csv python bench.py --steps 2 "
                               "--warmup 3 --no-cpu-baseline",
        "workload": "cfg4", "pool_blocks": pool, "algorithmic_bytes_per_launch": 16 * pool,
        "dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
        "traffic_over_algorithmic": (rd + wr) / (16 * pool), "streamed_bytes_per_launch": 8 * pool,
        "traffic_over_streamed": (rd + wr) / (8 * pool),
        "note": "admit_body is the same code in admit_kernel (one cooperative launch per admission) and in the "
                "persistent server_kernel the engine uses; ncu cannot replay the server (it waits on the host's "
                "mailbox), so the captures run the per-admission launch (CS_SERVER=0). Cold-cache, serialized replays: "
                "the DRAM bytes per launch are the evidence, the absolute times are not the bench's.",
        "metrics": {k: " ".join(m[k]) for k in keep if k in m},
        "launch_list": {"file": os.path.relpath(lcsv, ROOT), "launches": len(ll), "scoring_launches": len(scan),
                        "median_us": statistics.median(x["gpu__time_duration.sum"] for x in scan) * 1e6 if scan else None,
                        "dram_read_median_bytes": statistics.median(x["dram__bytes_read.sum"] for x in scan) if scan else None,
                        "dram_write_median_bytes": statistics.median(x["dram__bytes_write.sum"] for x in scan) if scan else None},
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
