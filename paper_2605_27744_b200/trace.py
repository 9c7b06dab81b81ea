"""The reference's Python trace surface (py_module.cpp:134-183, trace_io.cpp): Trace,
generate_trace(preset, sessions, seed), Trace.to_jsonl(), read_trace_jsonl(text) and
run_sim(trace, ...) -> the metrics dict of run_cell (experiment.cpp:355-379, engine.cpp:394-410).

The JSONL text is byte-identical to the reference's write_trace_jsonl (nlohmann ordered_json,
compact), so traces move between the two implementations both ways; run_sim replays a Trace
through the GPU engine (cs_engine_create_from_turns) and aggregates exactly as the reference
(aggregate_metrics, metrics.cpp:5-25, summation in turn-id order).
"""
from __future__ import annotations

import copy
import ctypes as C
import json

import numpy as np

from . import workloads
from ._lib import EngineCfg, check, lib

SCHEMA = "cachesage-trace/v1"
_FIELDS = ("session", "turn", "agent", "anchor", "history", "prompt", "decode")


def _dumps(obj):
    return json.dumps(obj, separators=(",", ":"), ensure_ascii=False)


class Trace:
    """A workload spec and its turns (rows: session, turn_index, agent, anchor_tokens,
    history_tokens, prompt_tokens, decode_tokens), like the reference's Trace."""

    def __init__(self, spec, rows):
        self.spec = spec
        self.rows = np.ascontiguousarray(rows, dtype=np.int64).reshape(-1, 7)

    @property
    def name(self):
        return self.spec["name"]

    @property
    def turn_count(self):
        return int(self.rows.shape[0])

    def _spec_json(self):  # spec_to_json (trace_io.cpp:18-43), key order included
        s = self.spec
        j = {"name": s["name"],
             "agents": [{"label": lab, "anchor_tokens": int(a)} for lab, a in zip(s["labels"], s["anchor_tokens"])],
             "transition": [[float(p) for p in row] for row in s["transition"]],
             "turns_min": int(s["turns_min"]), "turns_max": int(s["turns_max"]), "sessions": int(s["sessions"]),
             "task_tokens": int(s["task_tokens"]), "history_growth": int(s["history_growth"]),
             "decode_tokens": int(s["decode_tokens"]), "template_tokens": int(s["template_tokens"]),
             "concurrency": int(s["concurrency"]), "budget_blocks": int(s["budget_blocks"]), "seed": int(s["seed"])}
        if s.get("supervisor") is not None:
            j["supervisor"] = int(s["supervisor"])
        return j

    def to_jsonl(self):
        """write_trace_jsonl (trace_io.cpp:74-85)."""
        for k in ("anchor_stride", "hist_pos_bits", "start_dist"):
            if self.spec.get(k):
                raise ValueError(f"to_jsonl: the trace schema has no '{k}' (widened generator spec)")
        labels = self.spec["labels"]
        out = [_dumps({"schema": SCHEMA, "spec": self._spec_json()})]
        for r in self.rows.tolist():
            out.append(_dumps({"session": r[0], "turn": r[1], "agent": r[2], "label": labels[r[2]], "anchor": r[3],
                               "history": r[4], "prompt": r[5], "decode": r[6]}))
        return "\n".join(out) + "\n"

    def __repr__(self):
        return f"Trace(name={self.name!r}, turn_count={self.turn_count})"


def _validate(spec):
    """WorkloadSpec::validate (workload.cpp:70-106) through the device library's generator (a
    one-session copy), so both implementations reject the same specs."""
    from .api import spec_struct

    s = dict(spec)
    s["sessions"] = 1
    st = spec_struct(s)
    check(lib().cs_generate_trace(C.byref(st), None, 0))


def generate_trace(preset, sessions=None, seed=None):
    """generate_trace (py_module.cpp:134-146): a named preset (or a spec dict), optionally with
    another session count or seed."""
    from .api import generate_trace_rows

    spec = workloads.preset_by_name(preset) if isinstance(preset, str) else copy.deepcopy(preset)
    if sessions is not None:
        spec["sessions"] = int(sessions)
    if seed is not None:
        spec["seed"] = int(seed)
    return Trace(spec, generate_trace_rows(spec))


def read_trace_jsonl(text):
    """read_trace_jsonl (trace_io.cpp:87-136): errors name the line (RuntimeError)."""
    spec, rows = None, []
    for no, line in enumerate(text.split("\n"), start=1):
        if not line:
            continue
        try:
            j = json.loads(line)
        except json.JSONDecodeError as e:
            raise RuntimeError(f"trace line {no}: {e}") from None
        try:
            if spec is None:
                if not isinstance(j, dict) or j.get("schema") != SCHEMA:
                    raise RuntimeError(f"expected header with schema '{SCHEMA}'")
                sj = j["spec"]
                spec = {"name": sj["name"], "labels": [a["label"] for a in sj["agents"]],
                        "anchor_tokens": [int(a["anchor_tokens"]) for a in sj["agents"]],
                        "transition": [[float(p) for p in row] for row in sj["transition"]],
                        "supervisor": sj.get("supervisor")}
                for k in ("turns_min", "turns_max", "sessions", "task_tokens", "history_growth", "decode_tokens",
                          "template_tokens", "concurrency", "budget_blocks", "seed"):
                    spec[k] = int(sj[k])
                _validate(spec)
                continue
            row = [int(j[f]) for f in _FIELDS]
            if not 0 <= row[2] < len(spec["labels"]):
                raise RuntimeError("agent index out of range")
            rows.append(row)
        except (KeyError, TypeError, ValueError, RuntimeError) as e:
            raise RuntimeError(f"trace line {no}: {e}") from None
    if spec is None:
        raise RuntimeError("trace line 1: missing header line")
    return Trace(spec, np.array(rows, np.int64).reshape(-1, 7))


def run_sim(trace, policy="cachesage", budget=None, concurrency=None, block_size=16, prefetch=True, **kw):
    """run_sim (py_module.cpp:170-180): one (trace, policy) cell on the GPU engine; the metrics
    dict of metrics_to_py (py_module.cpp:48-63). `trace` may also be a preset name or spec."""
    from .api import Engine, spec_struct

    if not isinstance(trace, Trace):
        trace = generate_trace(trace)
    eng = Engine.__new__(Engine)
    cfg = EngineCfg()
    lib().cs_engine_cfg_default(C.byref(cfg))
    from .api import pool_cfg

    cfg.pool = pool_cfg(budget or 0, policy=policy, **kw)
    cfg.concurrency = concurrency or 0
    cfg.block_size = block_size
    cfg.prefetch = 1 if prefetch else 0
    eng._spec = spec_struct(trace.spec)
    eng.comm = None
    h = C.c_void_p()
    rows = np.ascontiguousarray(trace.rows, dtype=np.int64)
    check(lib().cs_engine_create_from_turns(C.byref(cfg), C.byref(eng._spec), rows.ctypes.data_as(C.c_void_p),
                                            rows.shape[0], C.byref(h)))
    eng.h = h
    try:
        res = eng.run()
        t = eng.turns()
        arr = np.zeros(max(res["turns"], 1), np.float64)
        check(lib().cs_engine_turn_arrivals(eng.h, arr.ctypes.data_as(C.c_void_p), res["turns"]))
    finally:
        eng.close()
    n = int(res["turns"])
    ttft_sum = latency_sum = 0.0
    for c, p, e, a in zip(t["cached_tokens"].tolist(), t["prompt_tokens"].tolist(), t["end_us"].tolist(),
                          arr[:n].tolist()):
        ttft_sum += 1000.0 + 50.0 * float(p - c)  # CostModel defaults (engine.cpp:302-304)
        latency_sum += e - a
    sim = float(res["sim_us"])
    return {"hit_rate": res["hit_rate"], "mean_ttft_ms": (ttft_sum / n if n else 0.0) / 1000.0,
            "mean_latency_ms": (latency_sum / n if n else 0.0) / 1000.0,
            "throughput_turns_per_s": n / (sim / 1e6) if sim > 0.0 else 0.0, "sim_duration_ms": sim / 1000.0,
            "turns": n, "total_prompt_tokens": int(res["total_prompt_tokens"]),
            "total_cached_tokens": int(res["total_cached_tokens"]), "evictions": int(res["evictions"]),
            "truncated_admissions": int(res["truncated"]), "warmups_executed": int(res["warmups_executed"]),
            "warmup_prompt_tokens": int(res["warmup_prompt_tokens"])}
