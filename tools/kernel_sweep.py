"""Per-kernel measurements the survey asks for beside the dominant admission kernel:
K1 hashing (tokens/s), K2 block-table probes (ns per probe), and the latency-bound policy kernels
K3 learner record, K3b reachability BFS, K6 argmax over A in {8, 32, 128, 512, 1024}.

Run it under ncu's launch list for the device-side numbers (every kernel's duration and DRAM
bytes; tools/ncu_kernels.py turns the CSV into profiles/*_kernels.json):

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file gpurun_out/kernels.csv python tools/kernel_sweep.py

Each section repeats its call REPS times in a fixed order and prints a JSON plan (section,
parameters, kernel, repetitions, work units per call) that the parser matches to the launch
list in order. Without ncu it prints host wall times per call (sync included) instead."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2605_27744_b200 as cb  # noqa: E402
from paper_2605_27744_b200 import api  # noqa: E402
from paper_2605_27744_b200 import workloads as W  # noqa: E402

REPS = 5
plan = []


def timed(fn):
    t = time.perf_counter()
    fn()
    return (time.perf_counter() - t) * 1e6


# ---- K1: chained prefix hashing + identity fold (hash_prompts_kernel), 128-bit token loads
rng = np.random.default_rng(1)
n_prompts, toks_per = 16384, 1024
prompts = [rng.integers(0, 1 << 31, toks_per, dtype=np.uint32) for _ in range(n_prompts)]
pool = api.Pool(1 << 16)
us = [timed(lambda: api.hash_prompts(prompts, pool=pool)) for _ in range(REPS)]
plan.append({"section": "K1", "kernel": "hash_prompts_kernel", "reps": REPS, "prompts": n_prompts,
             "tokens_per_call": n_prompts * toks_per, "blocks_per_call": n_prompts * toks_per // 16,
             "host_us_median": float(np.median(us))})
pool.close()

# ---- K2: block-table probes on a 16M-slot pool (1 GiB table, misses L2): half the keys resident
N = 16 << 20
pool = api.Pool(N)
keys, lt, agents, refs = W.pool_snapshot(N, 256, seed=11, mode="realistic")
pool.register_agents(np.arange(1, 257, dtype=np.uint64))
pool.restore(keys, lt, agents=agents, refs=refs)
n_probe = 1 << 20
probe = np.concatenate([keys[rng.integers(0, N, n_probe // 2)], rng.integers(1, 1 << 62, n_probe // 2, dtype=np.uint64)])
del keys, lt, agents, refs
us = [timed(lambda: pool.probe_needed(probe)) for _ in range(REPS)]
plan.append({"section": "K2", "kernel": "probe_kernel", "reps": REPS, "probes_per_call": int(n_probe),
             "resident_fraction": 0.5, "pool_slots": N, "host_us_median": float(np.median(us))})
pool.close()

# ---- K3 / K3b / K6 over the agent count A: learner record (B transitions), BFS rebuild, argmax
for A in (8, 32, 128, 512, 1024):
    L = api.TransitionLearner(window=1024, agent_capacity=max(A, 8))
    ids = np.arange(1, A + 1, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
    # 4 successors per agent with random weights (cfg5), a walk of B transitions
    succ = rng.integers(0, A, (A, 4))
    B = 4096
    walk = np.zeros(B + 1, np.int64)
    for i in range(B):
        walk[i + 1] = succ[walk[i], rng.integers(0, 4)]
    prev, nxt = ids[walk[:-1]], ids[walk[1:]]
    L.record_many(prev, nxt)  # learn the alphabet (untimed)
    us_r = [timed(lambda: L.record_many(prev, nxt)) for _ in range(REPS)]
    us_b = [timed(lambda: L.rebuild_reachability(int(ids[0]))) for _ in range(REPS)]
    us_a = [timed(lambda: L.argmax_row(int(ids[0]))) for _ in range(REPS)]
    plan.append({"section": "K3", "kernel": "learner_record_kernel", "agents": A, "reps": REPS,
                 "transitions_per_call": B, "host_us_median": float(np.median(us_r))})
    plan.append({"section": "K3b", "kernel": "learner_bfs_kernel", "agents": A, "reps": REPS,
                 "host_us_median": float(np.median(us_b))})
    plan.append({"section": "K6", "kernel": "learner_argmax_kernel", "agents": A, "reps": REPS,
                 "host_us_median": float(np.median(us_a))})
    L.close()

print("PLAN " + json.dumps(plan), flush=True)
