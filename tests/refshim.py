"""ctypes binding of oracle/_ref/libcachesage_ref.so — the UNMODIFIED reference compiled in place.

TEST INFRASTRUCTURE ONLY (also used by bench.py's reference arm). Available when the library was
built (``make -C oracle ref`` in the container that has /root/reference; the .so then travels to
the GPU box). ``available()`` is False otherwise and callers skip.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(os.path.dirname(_HERE), "oracle", "_ref", "libcachesage_ref.so")

_lib = None


class RefSpec(C.Structure):
    _fields_ = [
        ("n_agents", C.c_int),
        ("anchor_tokens", C.POINTER(C.c_int)),
        ("transition", C.POINTER(C.c_double)),
        ("supervisor", C.c_int),
        ("turns_min", C.c_int), ("turns_max", C.c_int), ("sessions", C.c_int),
        ("task_tokens", C.c_int), ("history_growth", C.c_int), ("decode_tokens", C.c_int),
        ("template_tokens", C.c_int), ("concurrency", C.c_int), ("budget_blocks", C.c_int),
        ("seed", C.c_ulonglong),
    ]


class RefRunCfg(C.Structure):
    _fields_ = [
        ("policy", C.c_int), ("budget_blocks", C.c_int), ("concurrency", C.c_int),
        ("block_size", C.c_int), ("prefetch", C.c_int), ("skip", C.c_int), ("take", C.c_int),
        ("tau", C.c_double), ("e_max", C.c_int), ("w_pred", C.c_double), ("window", C.c_long),
        ("min_confidence", C.c_double), ("min_row_count", C.c_ulonglong),
        ("budget_per_step", C.c_int), ("prefill_base_us", C.c_double),
        ("prefill_per_token_us", C.c_double), ("decode_per_token_us", C.c_double),
    ]


class RefRunOut(C.Structure):
    _fields_ = [
        ("n_turns", C.c_long), ("cached_tokens", C.POINTER(C.c_long)),
        ("prompt_tokens", C.POINTER(C.c_long)), ("start_us", C.POINTER(C.c_double)),
        ("end_us", C.POINTER(C.c_double)), ("n_evictions", C.c_long),
        ("evictions", C.POINTER(C.c_ulonglong)), ("n_warmups", C.c_long),
        ("warmup_step", C.POINTER(C.c_long)), ("warmup_target", C.POINTER(C.c_ulonglong)),
        ("warmup_tick", C.POINTER(C.c_ulonglong)), ("hit_rate", C.c_double),
        ("truncated", C.c_long), ("warmups_executed", C.c_long), ("warmups_dropped", C.c_long),
        ("sim_us", C.c_double), ("n_steps", C.c_long), ("events", C.c_long),
    ]


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(LIB_PATH)
        _lib.ref_chain_hash.restype = C.c_ulonglong
        _lib.ref_chain_hash.argtypes = [C.c_int, C.c_ulonglong, C.c_void_p, C.c_size_t]
        _lib.ref_block_keys.restype = C.c_long
        _lib.ref_block_keys.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_void_p, C.c_void_p]
        _lib.ref_identity.restype = C.c_int
        _lib.ref_identity.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_void_p]
        _lib.ref_preset_spec.restype = C.c_int
        _lib.ref_preset_spec.argtypes = [C.c_char_p, C.POINTER(RefSpec)]
        _lib.ref_generate.restype = C.c_long
        _lib.ref_generate.argtypes = [C.POINTER(RefSpec), C.c_void_p, C.c_long]
        _lib.ref_turn_tokens.restype = C.c_long
        _lib.ref_turn_tokens.argtypes = [C.POINTER(RefSpec), C.c_long, C.c_void_p, C.c_long]
        _lib.ref_run.restype = C.c_int
        _lib.ref_run.argtypes = [C.POINTER(RefSpec), C.POINTER(RefRunCfg), C.POINTER(RefRunOut)]
        _lib.ref_free_run.argtypes = [C.POINTER(RefRunOut)]
        _lib.ref_last_error.restype = C.c_char_p
        _lib.ref_policy_trace.restype = C.c_int
        _lib.ref_policy_trace.argtypes = [C.POINTER(RefRunCfg), C.c_long] + [C.c_void_p] * 6 + [
            C.c_long] + [C.c_void_p] * 4 + [C.c_long] + [C.c_void_p] * 4 + [
            C.c_ulonglong, C.c_ulonglong, C.c_void_p, C.c_void_p]
        _lib.ref_exact_survival.restype = C.c_double
        _lib.ref_exact_survival.argtypes = [C.c_ulonglong, C.c_int, C.c_long, C.c_void_p,
                                            C.c_void_p, C.c_ulonglong]
        _lib.ref_learner_eval.restype = C.c_long
        _lib.ref_learner_eval.argtypes = [C.c_long, C.c_void_p, C.c_void_p, C.c_long, C.c_long, C.c_ulonglong,
                                          C.c_double, C.c_int, C.c_int] + [C.c_void_p] * 9
        _lib.ref_preset_trace_jsonl.restype = C.c_long
        _lib.ref_preset_trace_jsonl.argtypes = [C.c_char_p, C.c_int, C.c_longlong, C.c_char_p, C.c_long]
        _lib.ref_run_experiment_text.restype = C.c_int
        _lib.ref_run_experiment_text.argtypes = [C.c_char_p]
        _lib.ref_run_sim_jsonl.restype = C.c_int
        _lib.ref_run_sim_jsonl.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
        _lib.ref_evict_bench.restype = C.c_double
        _lib.ref_evict_bench.argtypes = [C.c_long, C.c_int, C.c_long, C.c_long, C.c_long, C.c_int,
                                         C.POINTER(C.c_double), C.POINTER(C.c_ulonglong)]
    return _lib


def _err():
    return lib().ref_last_error().decode()


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def chain_hash(parent, tokens):
    t = np.ascontiguousarray(tokens, dtype=np.uint32)
    return int(lib().ref_chain_hash(0 if parent is None else 1, 0 if parent is None else parent,
                                    _ptr(t), t.size))


def block_keys(tokens, block_size=16):
    t = np.ascontiguousarray(tokens, dtype=np.uint32)
    n = (t.size + block_size - 1) // block_size
    keys = np.zeros(max(n, 1), dtype=np.uint64)
    cnt = np.zeros(max(n, 1), dtype=np.int32)
    r = lib().ref_block_keys(_ptr(t), t.size, block_size, _ptr(keys), _ptr(cnt))
    if r < 0:
        raise ValueError(_err())
    return keys[:r], cnt[:r]


def identity(keys, skip=4, take=4):
    k = np.ascontiguousarray(keys, dtype=np.uint64)
    out = C.c_ulonglong(0)
    if lib().ref_identity(_ptr(k), k.size, skip, take, C.byref(out)) != 0:
        raise ValueError(_err())
    return int(out.value)


def _spec_struct(spec):
    anchors = np.ascontiguousarray(spec["anchor_tokens"], dtype=np.int32)
    trans = np.ascontiguousarray(spec["transition"], dtype=np.float64).reshape(-1)
    s = RefSpec()
    s.n_agents = anchors.size
    s.anchor_tokens = anchors.ctypes.data_as(C.POINTER(C.c_int))
    s.transition = trans.ctypes.data_as(C.POINTER(C.c_double))
    s.supervisor = -1 if spec.get("supervisor") is None else spec["supervisor"]
    for f in ("turns_min", "turns_max", "sessions", "task_tokens", "history_growth",
              "decode_tokens", "template_tokens", "concurrency", "budget_blocks"):
        setattr(s, f, int(spec[f]))
    s.seed = int(spec["seed"])
    s._keep = (anchors, trans)
    return s


def preset_spec(name):
    s = RefSpec()
    if lib().ref_preset_spec(name.encode(), C.byref(s)) != 0:
        raise ValueError(_err())
    n = s.n_agents
    return {
        "name": name,
        "anchor_tokens": [s.anchor_tokens[i] for i in range(n)],
        "transition": [[s.transition[i * n + j] for j in range(n)] for i in range(n)],
        "supervisor": None if s.supervisor < 0 else s.supervisor,
        "turns_min": s.turns_min, "turns_max": s.turns_max, "sessions": s.sessions,
        "task_tokens": s.task_tokens, "history_growth": s.history_growth,
        "decode_tokens": s.decode_tokens, "template_tokens": s.template_tokens,
        "concurrency": s.concurrency, "budget_blocks": s.budget_blocks, "seed": s.seed,
    }


def generate(spec):
    s = _spec_struct(spec)
    n = lib().ref_generate(C.byref(s), None, 0)
    if n < 0:
        raise ValueError(_err())
    out = np.zeros((max(n, 1), 7), dtype=np.int64)
    lib().ref_generate(C.byref(s), _ptr(out), n)
    return out[:n]


def turn_tokens(spec, idx, cap=1 << 20):
    s = _spec_struct(spec)
    out = np.zeros(cap, dtype=np.uint32)
    n = lib().ref_turn_tokens(C.byref(s), idx, _ptr(out), cap)
    if n < 0:
        raise ValueError(_err())
    return out[:n]


POLICY_IDS = {"lru": 0, "cachesage": 1, "ttl": 2, "belady": 3}


def run_cfg(policy="cachesage", budget=None, concurrency=None, block_size=16, prefetch=True,
            skip=4, take=4, tau=0.01, e_max=8, w_pred=1.0, window=1024, min_confidence=0.5,
            min_row_count=5, budget_per_step=1, cost=None):
    """cost = (prefill_base_us, prefill_per_token_us, decode_per_token_us) or None (defaults)."""
    c = RefRunCfg()
    c.policy = POLICY_IDS[policy]
    c.budget_blocks = budget or 0
    c.concurrency = concurrency or 0
    c.block_size = block_size
    c.prefetch = 1 if prefetch else 0
    c.skip, c.take, c.tau, c.e_max, c.w_pred = skip, take, tau, e_max, w_pred
    c.window, c.min_confidence, c.min_row_count = window, min_confidence, min_row_count
    c.budget_per_step = budget_per_step
    if cost is not None:
        c.prefill_base_us, c.prefill_per_token_us, c.decode_per_token_us = cost
    return c


def run(spec, **kw):
    s = _spec_struct(spec)
    c = run_cfg(**kw)
    o = RefRunOut()
    if lib().ref_run(C.byref(s), C.byref(c), C.byref(o)) != 0:
        raise RuntimeError(_err())
    try:
        nt, ne, nw = o.n_turns, o.n_evictions, o.n_warmups
        res = {
            "cached_tokens": np.ctypeslib.as_array(o.cached_tokens, (max(nt, 1),))[:nt].copy(),
            "prompt_tokens": np.ctypeslib.as_array(o.prompt_tokens, (max(nt, 1),))[:nt].copy(),
            "start_us": np.ctypeslib.as_array(o.start_us, (max(nt, 1),))[:nt].copy(),
            "end_us": np.ctypeslib.as_array(o.end_us, (max(nt, 1),))[:nt].copy(),
            "evictions": np.ctypeslib.as_array(o.evictions, (max(ne, 1),))[:ne].copy().astype(np.uint64),
            "warmup_step": np.ctypeslib.as_array(o.warmup_step, (max(nw, 1),))[:nw].copy(),
            "warmup_target": np.ctypeslib.as_array(o.warmup_target, (max(nw, 1),))[:nw].copy().astype(np.uint64),
            "warmup_tick": np.ctypeslib.as_array(o.warmup_tick, (max(nw, 1),))[:nw].copy().astype(np.uint64),
            "hit_rate": o.hit_rate, "truncated": o.truncated,
            "warmups_executed": o.warmups_executed, "warmups_dropped": o.warmups_dropped,
            "sim_us": o.sim_us, "n_steps": o.n_steps, "events": o.events,
        }
    finally:
        lib().ref_free_run(C.byref(o))
    return res


def last_state():
    """The final Policy::serialize_state().dump() of the last run() on this thread."""
    f = lib().ref_last_state
    f.restype = C.c_char_p
    return f().decode()


def fnv1a64(keys) -> int:
    """FNV-1a-64 over each key's 8 little-endian bytes in order (SURVEY.md §4.4 recipe)."""
    h = 1469598103934665603
    b = np.ascontiguousarray(keys, dtype="<u8").tobytes()
    for byte in b:
        h ^= byte
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def evict_bench(N, n_agents, n_agent_blocks, k, cachesage=True, k_warm=0):
    """Reference EngineSim at pool N: (seconds per evict_one over k timed evictions, fill s)."""
    fill = C.c_double(0)
    last = C.c_ulonglong(0)
    s = lib().ref_evict_bench(N, n_agents, n_agent_blocks, k_warm, k, 1 if cachesage else 0,
                              C.byref(fill), C.byref(last))
    if s < 0:
        raise RuntimeError(_err())
    return s, fill.value, int(last.value)


def learner_eval(pairs_a, pairs_b, window=1024, current=0, tau=0.01, e_max=8, k=-1, cap=64):
    """The reference TransitionLearner after recording the pairs (see ref_learner_eval)."""
    import numpy as np

    a = np.ascontiguousarray(pairs_a, dtype=np.uint64)
    b = np.ascontiguousarray(pairs_b, dtype=np.uint64)
    ag = np.zeros(cap, np.uint64)
    prob = np.zeros(cap * cap, np.float64)
    tot = np.zeros(cap, np.uint64)
    sb = np.zeros(1, np.uint64)
    ai = np.zeros(cap, np.uint64)
    ap = np.zeros(cap, np.float64)
    af = np.zeros(cap, np.int32)
    hops = np.zeros(cap, np.int32)
    surv = np.zeros(cap, np.float64)
    n = lib().ref_learner_eval(a.size, _ptr(a), _ptr(b), window, cap, current, tau, e_max, k, _ptr(ag), _ptr(prob),
                               _ptr(tot), _ptr(sb), _ptr(ai), _ptr(ap), _ptr(af), _ptr(hops), _ptr(surv))
    if n < 0:
        raise RuntimeError(_err())
    return {"agents": [int(x) for x in ag[:n]], "prob": prob[:n * n].reshape(n, n), "totals": tot[:n],
            "state_bytes": int(sb[0]), "argmax": [(int(i), float(p)) if f else None for i, p, f in zip(ai[:n], ap[:n], af[:n])],
            "hops": hops[:n], "surv": surv[:n]}


def preset_trace_jsonl(preset, sessions=None, seed=None):
    """The reference's generate_trace(preset, sessions, seed).to_jsonl()."""
    n = lib().ref_preset_trace_jsonl(preset.encode(), sessions or -1, -1 if seed is None else seed, None, 0)
    if n < 0:
        raise RuntimeError(_err())
    buf = C.create_string_buffer(n)
    lib().ref_preset_trace_jsonl(preset.encode(), sessions or -1, -1 if seed is None else seed, buf, n)
    return buf.raw[:n].decode()


METRIC_KEYS = ["hit_rate", "mean_ttft_ms", "mean_latency_ms", "throughput_turns_per_s", "sim_duration_ms", "turns",
               "total_prompt_tokens", "total_cached_tokens", "evictions", "truncated_admissions", "warmups_executed",
               "warmup_prompt_tokens"]


def run_sim_jsonl(jsonl, policy="cachesage", budget=None, concurrency=None, block_size=16, prefetch=True):
    """The reference's run_sim(read_trace_jsonl(jsonl), ...) metrics dict."""
    import numpy as np

    out = np.zeros(12, np.float64)
    if lib().ref_run_sim_jsonl(jsonl.encode(), policy.encode(), budget or 0, concurrency or 0, block_size,
                               1 if prefetch else 0, _ptr(out)) != 0:
        raise RuntimeError(_err())
    d = dict(zip(METRIC_KEYS, out.tolist()))
    for k in METRIC_KEYS[5:]:
        d[k] = int(d[k])
    return d


def run_experiment(config):
    """The reference's run_experiment over a config dict (the `cachesage run` config schema,
    experiment.cpp:238-330); files land under config["output"]["dir"]. Runs oracle/_ref/
    ref_experiment in a child process (its std::filesystem clashes with the interpreter's
    libstdc++ in-process)."""
    import json as _json
    import subprocess

    exe = os.path.join(os.path.dirname(LIB_PATH), "ref_experiment")
    r = subprocess.run([exe], input=_json.dumps(config).encode(), capture_output=True)
    if r.returncode != 0:
        raise RuntimeError(r.stderr.decode())


def policy_events(events, **kw):
    """ref_policy_events: the reference Runtime + policy over an event stream. events: list of
    dicts {kind (0..4), tick, agent, prev (None or id), request, drain (bool), ckpt (bool)}.
    Returns (checkpoints, None) or (None, (fail_index, message))."""
    import json

    c = run_cfg(**kw)
    n = len(events)
    kind = np.array([e["kind"] for e in events], np.int32)
    tick = np.array([e["tick"] for e in events], np.uint64)
    agent = np.array([e.get("agent", 0) for e in events], np.uint64)
    has_prev = np.array([e.get("prev") is not None for e in events], np.int32)
    prev = np.array([e.get("prev") or 0 for e in events], np.uint64)
    req = np.array([e.get("request", 0) for e in events], np.uint64)
    drain = np.array([1 if e.get("drain") else 0 for e in events], np.uint8)
    ckpt = np.array([1 if e.get("ckpt") else 0 for e in events], np.uint8)
    fail = C.c_long(-1)
    L = lib()
    f = L.ref_policy_events
    f.restype = C.c_long
    f.argtypes = [C.POINTER(RefRunCfg), C.c_long] + [C.c_void_p] * 8 + [C.c_char_p, C.c_long, C.POINTER(C.c_long)]
    args = [C.byref(c), n] + [_ptr(a) for a in (kind, tick, agent, has_prev, prev, req, drain, ckpt)]
    m = f(*args, None, 0, C.byref(fail))
    if m < 0:
        return None, (fail.value, _err())
    buf = C.create_string_buffer(m + 1)
    f(*args, buf, m + 1, C.byref(fail))
    return json.loads(buf.value.decode()), None
