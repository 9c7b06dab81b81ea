"""Multi-process (world_size 2, gloo on CPU) coverage of bench.py's N>1 logic: the replicas
partition the job (distinct traces and snapshots per rank, no data-path collective), the
whole-job value is the sum of units over the max of device times, and the reference arm
prints from rank 0 only.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import bench

    d = bench.Dist(world, rank, rank, backend="gloo")
    try:
        d.barrier()
        ms = [1.0 + rank, 2.0]          # rank 1 is the slow one: 4 ms total
        value, tot = bench.aggregate(d, ms, 1000 * (rank + 1))
        spec, snap = bench.rank_workload(50, 4096, rank)
        q.put((rank, value, tot, spec["seed"], snap))
    finally:
        d.close()


def test_gloo_world2_aggregation_and_partition():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
        assert p.exitcode == 0
    out = sorted(q.get() for _ in range(world))
    for rank, value, tot, seed, snap in out:
        assert tot == 4.0                       # max over ranks of the per-rank device time
        assert value == 3000 / 4e-3             # units of all ranks / slowest rank's time
    assert out[0][3] != out[1][3] and out[0][4] != out[1][4]  # disjoint trace partitions


def test_rank_partitions_generate_different_traces():
    import bench
    from paper_2605_27744_b200 import api

    a, _ = bench.rank_workload(30, 4096, 0)
    b, _ = bench.rank_workload(30, 4096, 1)
    ta, tb = api.generate_trace_rows(a), api.generate_trace_rows(b)
    assert not (ta.shape == tb.shape and np.array_equal(ta, tb))


def test_reference_arm_rank_nonzero_is_silent(tmp_path):
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "3", "--pool", "4096"], env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0
    assert r.stdout.strip() == ""


def test_reference_arm_line_small_pool():
    env = dict(os.environ, RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "3", "--pool", "4096"], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    if "unavailable" in line:
        return
    for k in ("metric", "value", "unit", "higher_is_better", "cpu_baseline", "e2e", "config"):
        assert k in line
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["value"] > 0
