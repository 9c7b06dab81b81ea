"""Output writers (acceptance criterion 10): the GPU engine's metrics.json,
turns.csv and events.jsonl against the reference experiment driver's files for the same cell
(tests/golden/outputs.json, made by tests/golden/make_outputs.py from oracle/_ref), byte for byte.
"""
import hashlib
import json
import os

import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CELLS = json.load(open(os.path.join(GOLD, "outputs.json")))["cells"]

pytestmark = pytest.mark.gpu


def _id(c):
    extra = "-".join(f"{k}{v}" for k, v in c["engine"].items())
    return f"{c['preset']}-{c['policy']}" + (f"-{extra}" if extra else "") + ("" if c["prefetch"] else "-noprefetch")


def _run_cell(c, out_dir, **kw):
    from paper_2605_27744_b200 import api
    from paper_2605_27744_b200 import workloads as W

    spec = W.preset_by_name(c["preset"])
    eng = api.Engine(spec, policy=c["policy"], budget=c["engine"].get("budget_blocks"),
                     concurrency=c["engine"].get("concurrency"), prefetch=c["prefetch"], agent_capacity=1024, **kw)
    try:
        eng.record_events()
        eng.run()
        eng.write_outputs(out_dir)
    finally:
        eng.close()


@pytest.mark.parametrize("c", CELLS, ids=[_id(c) for c in CELLS])
def test_cell_outputs_byte_identical(c, tmp_path):
    _run_cell(c, tmp_path)
    got = (tmp_path / "metrics.json").read_text()
    assert got == c["metrics_json"]
    for f, want in c["files"].items():
        b = (tmp_path / f).read_bytes()
        if f == "events.jsonl" and hashlib.sha256(b).hexdigest() != want["sha256"]:
            assert b.decode().splitlines()[:40] == c["events_head"]
        assert (len(b), hashlib.sha256(b).hexdigest()) == (want["size"], want["sha256"]), f


def test_outputs_through_host_inputs(tmp_path):
    """The end-to-end path (host-resident prompt blocks) writes the same files."""
    c = CELLS[0]
    _run_cell(c, tmp_path, host_inputs=True)
    for f, want in c["files"].items():
        b = (tmp_path / f).read_bytes()
        assert hashlib.sha256(b).hexdigest() == want["sha256"], f


def test_events_need_recording(tmp_path):
    from paper_2605_27744_b200 import api
    from paper_2605_27744_b200 import workloads as W

    eng = api.Engine(W.preset_by_name("supervisor-a"), policy="lru", agent_capacity=1024)
    try:
        eng.run()
        with pytest.raises(Exception, match="not recorded"):
            eng.write_outputs(tmp_path)
        eng.write_outputs(tmp_path, events=False)  # metrics + turns only
        assert (tmp_path / "metrics.json").read_text() == next(
            x for x in CELLS if x["preset"] == "supervisor-a" and x["policy"] == "lru")["metrics_json"]
        with pytest.raises(Exception, match="before the first step"):
            eng.record_events()
    finally:
        eng.close()
