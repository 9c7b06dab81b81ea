"""Workload specs: the reference's bundled presets, BASELINE.json cfg1, and the widened
large-scale traces cfg2-cfg4.

Specs are plain dicts with the WorkloadSpec fields of workload.hpp:21-42 (+ anchor_stride /
hist_pos_bits of the widened token scheme). The preset values restate
presets.cpp:14-124 (data, not code).
"""
from __future__ import annotations

import copy

SUPERVISOR_AGENTS = ["supervisor", "planner", "researcher", "coder", "tester", "critic"]


def _supervisor_base(name, seed):
    # presets.cpp:14-33
    return {
        "name": name,
        "labels": list(SUPERVISOR_AGENTS),
        "anchor_tokens": [176, 176, 176, 176, 160, 160],
        "supervisor": 0,
        "turns_min": 6, "turns_max": 14, "sessions": 100,
        "task_tokens": 160, "history_growth": 8, "decode_tokens": 32, "template_tokens": 16,
        "concurrency": 4, "budget_blocks": 120, "seed": seed,
    }


def preset_workloads():
    """The five bundled workloads (presets.cpp:37-130)."""
    a = _supervisor_base("supervisor-a", 101)
    a["task_tokens"] = 176
    a["transition"] = [
        [0.00, 0.25, 0.25, 0.25, 0.15, 0.10],
        [0.15, 0.00, 0.70, 0.15, 0.00, 0.00],
        [0.15, 0.15, 0.00, 0.70, 0.00, 0.00],
        [0.15, 0.00, 0.00, 0.00, 0.70, 0.15],
        [0.15, 0.55, 0.00, 0.00, 0.00, 0.30],
        [0.60, 0.25, 0.00, 0.15, 0.00, 0.00],
    ]
    b = _supervisor_base("supervisor-b", 102)
    b["task_tokens"] = 160
    b["transition"] = [
        [0.000, 0.35, 0.15, 0.300, 0.10, 0.10],
        [0.200, 0.00, 0.65, 0.150, 0.00, 0.00],
        [0.200, 0.00, 0.00, 0.650, 0.15, 0.00],
        [0.200, 0.00, 0.00, 0.000, 0.70, 0.10],
        [0.025, 0.95, 0.00, 0.025, 0.00, 0.00],
        [0.650, 0.20, 0.00, 0.000, 0.15, 0.00],
    ]
    c = _supervisor_base("supervisor-c", 103)
    c["anchor_tokens"][0] = 144
    c["task_tokens"] = 200
    c["transition"] = [
        [0.00, 0.30, 0.30, 0.20, 0.10, 0.10],
        [0.15, 0.00, 0.70, 0.15, 0.00, 0.00],
        [0.15, 0.15, 0.00, 0.70, 0.00, 0.00],
        [0.15, 0.00, 0.15, 0.00, 0.70, 0.00],
        [0.30, 0.70, 0.00, 0.00, 0.00, 0.00],
        [0.65, 0.20, 0.00, 0.00, 0.15, 0.00],
    ]
    d = _supervisor_base("supervisor-d", 104)
    d["anchor_tokens"][0] = 192
    d["task_tokens"] = 192
    d["transition"] = [
        [0.00, 0.22, 0.22, 0.22, 0.17, 0.17],
        [0.12, 0.00, 0.76, 0.12, 0.00, 0.00],
        [0.12, 0.00, 0.00, 0.76, 0.12, 0.00],
        [0.12, 0.00, 0.00, 0.00, 0.76, 0.12],
        [0.38, 0.50, 0.00, 0.00, 0.00, 0.12],
        [0.55, 0.33, 0.00, 0.12, 0.00, 0.00],
    ]
    n = 12
    chain = {
        "name": "synthetic-chain",
        "labels": [f"step-{i + 1:02d}" for i in range(n)],
        "anchor_tokens": [208] * n,
        "transition": [[1.0 if j == (i + 1) % n else 0.0 for j in range(n)] for i in range(n)],
        "supervisor": 0,
        "turns_min": 12, "turns_max": 28, "sessions": 50,
        "task_tokens": 352, "history_growth": 32, "decode_tokens": 32, "template_tokens": 16,
        "concurrency": 1, "budget_blocks": 250, "seed": 105,
    }
    return [a, b, c, d, chain]


def preset_names():
    return [s["name"] for s in preset_workloads()]


def preset_by_name(name):
    for s in preset_workloads():
        if s["name"] == name:
            return s
    raise ValueError(f"unknown workload preset '{name}' (valid: {', '.join(preset_names())})")


def cfg1(budget=65536):
    """BASELINE cfg1: synthetic supervisor -> 4-specialist trace, ~10k requests."""
    return {
        "name": "cfg1-supervisor-4specialist",
        "labels": ["supervisor", "planner", "researcher", "coder", "tester"],
        "anchor_tokens": [176, 176, 176, 176, 160],
        "transition": [
            [0.00, 0.30, 0.30, 0.25, 0.15],
            [0.15, 0.00, 0.70, 0.15, 0.00],
            [0.15, 0.15, 0.00, 0.70, 0.00],
            [0.15, 0.00, 0.00, 0.00, 0.85],
            [0.40, 0.60, 0.00, 0.00, 0.00],
        ],
        "supervisor": 0,
        "turns_min": 6, "turns_max": 14, "sessions": 1000,
        "task_tokens": 160, "history_growth": 8, "decode_tokens": 32, "template_tokens": 16,
        "concurrency": 4, "budget_blocks": budget, "seed": 2605,
    }


def cfg2_hierarchical(sessions=100_000, budget=1 << 20):
    """cfg2: hierarchical org, 32 agents (root -> 3 directors -> 9 managers -> 18 ICs + reviewer).
    0.8 down (uniform over children) / 0.2 up; leaves 0.7 parent / 0.3 sibling. Prefetch off."""
    A = 32
    T = [[0.0] * A for _ in range(A)]
    root, reviewer = 0, 31
    directors = [1, 2, 3]
    managers = list(range(4, 13))
    ics = list(range(13, 31))
    for d in directors:
        T[root][d] = 0.8 / 3
    T[root][reviewer] = 0.2
    for k, d in enumerate(directors):
        for m in managers[3 * k:3 * k + 3]:
            T[d][m] = 0.8 / 3
        T[d][root] = 0.2
    for k, m in enumerate(managers):
        d = directors[k // 3]
        for ic in ics[2 * k:2 * k + 2]:
            T[m][ic] = 0.4
        T[m][d] = 0.2
    for k, ic in enumerate(ics):
        m = managers[k // 2]
        sib = ics[k ^ 1]
        T[ic][m] = 0.7
        T[ic][sib] = 0.3
    T[reviewer][root] = 1.0
    return {
        "name": "cfg2-hierarchical-32",
        "anchor_tokens": [176] * A,
        "transition": T, "supervisor": 0,
        "turns_min": 6, "turns_max": 14, "sessions": sessions,
        "task_tokens": 160, "history_growth": 8, "decode_tokens": 32, "template_tokens": 16,
        "concurrency": 4, "budget_blocks": budget, "seed": 2606,
        "anchor_stride": 0x10000, "hist_pos_bits": 11, "prefetch": False,
    }


def cfg3_swarm(sessions=100_000, budget=4 << 20):
    """cfg3: swarm handoff, 128 agents, successors {i+1, i+7, i+31} w.p. {0.6, 0.3, 0.1}."""
    A = 128
    T = [[0.0] * A for _ in range(A)]
    for i in range(A):
        T[i][(i + 1) % A] += 0.6
        T[i][(i + 7) % A] += 0.3
        T[i][(i + 31) % A] += 0.1
    return {
        "name": "cfg3-swarm-128",
        "anchor_tokens": [176] * A,
        "transition": T, "supervisor": 0,
        "turns_min": 6, "turns_max": 14, "sessions": sessions,
        "task_tokens": 160, "history_growth": 8, "decode_tokens": 32, "template_tokens": 16,
        "concurrency": 4, "budget_blocks": budget, "seed": 2607,
        "anchor_stride": 0x10000, "hist_pos_bits": 11, "prefetch": True,
    }


def scaled(spec, **kw):
    s = copy.deepcopy(spec)
    s.update(kw)
    return s
