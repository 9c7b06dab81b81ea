"""Regenerates tests/golden/outputs.json from the UNMODIFIED reference's experiment driver
(oracle/_ref/ref_experiment = run_experiment over a config, experiment.cpp:380-495): per cell the
sha256 and size of metrics.json, turns.csv and events.jsonl (and metrics.json in full), so the
GPU tests can check the output writers byte for byte without the reference on the box.

    make -C oracle ref && python tests/golden/make_outputs.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import refshim  # noqa: E402

FILES = ("metrics.json", "turns.csv", "events.jsonl")

# (preset, policy, engine overrides, prefetch)
CELLS = [
    ("supervisor-a", "cachesage", {}, True),
    ("supervisor-a", "lru", {}, True),
    ("supervisor-a", "ttl", {}, True),
    ("supervisor-a", "belady", {}, True),
    ("supervisor-b", "cachesage", {}, True),
    ("supervisor-c", "cachesage", {}, True),
    ("synthetic-chain", "cachesage", {}, True),
    ("supervisor-a", "cachesage", {"budget_blocks": 60}, True),
    ("supervisor-a", "cachesage", {"concurrency": 8}, True),
    ("supervisor-a", "cachesage", {}, False),
]


def main():
    out = {"source": "oracle/_ref/ref_experiment (unmodified reference run_experiment)", "cells": []}
    for preset, policy, engine, prefetch in CELLS:
        d = tempfile.mkdtemp()
        cfg = {"workload": preset, "policies": [policy], "output": {"dir": d, "events": True},
               "policy": {"prefetch": prefetch}}
        if engine:
            cfg["engine"] = engine
        refshim.run_experiment(cfg)
        cell = os.path.join(d, preset, policy)
        rec = {"preset": preset, "policy": policy, "engine": engine, "prefetch": prefetch, "files": {}}
        for f in FILES:
            b = open(os.path.join(cell, f), "rb").read()
            rec["files"][f] = {"sha256": hashlib.sha256(b).hexdigest(), "size": len(b)}
        rec["metrics_json"] = open(os.path.join(cell, "metrics.json")).read()
        rec["events_head"] = open(os.path.join(cell, "events.jsonl")).read().splitlines()[:40]
        out["cells"].append(rec)
    with open(os.path.join(HERE, "outputs.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", len(out["cells"]), "cells")


if __name__ == "__main__":
    main()
