"""ctypes binding of the plain-C oracle (oracle/cs_oracle.c -> oracle/_build/libcs_oracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() (as the checker) and
bench.py's cpu_baseline leg. The product package never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "libcs_oracle.so")
_lib = None


class Spec(C.Structure):
    _fields_ = [
        ("n_agents", C.c_int), ("anchor_tokens", C.POINTER(C.c_int)),
        ("transition", C.POINTER(C.c_double)), ("supervisor", C.c_int),
        ("turns_min", C.c_int), ("turns_max", C.c_int), ("sessions", C.c_int),
        ("task_tokens", C.c_int), ("history_growth", C.c_int), ("decode_tokens", C.c_int),
        ("template_tokens", C.c_int), ("concurrency", C.c_int), ("budget_blocks", C.c_int),
        ("seed", C.c_uint64), ("anchor_stride", C.c_uint32), ("hist_pos_bits", C.c_int),
        ("start_dist", C.POINTER(C.c_double)),
    ]


class Cfg(C.Structure):
    _fields_ = [
        ("policy", C.c_int), ("budget_blocks", C.c_int), ("concurrency", C.c_int),
        ("block_size", C.c_int), ("prefetch", C.c_int), ("skip", C.c_int), ("take", C.c_int),
        ("tau", C.c_double), ("e_max", C.c_int), ("w_pred", C.c_double), ("window", C.c_long),
        ("min_confidence", C.c_double), ("min_row_count", C.c_uint64),
        ("budget_per_step", C.c_int), ("fast_evict", C.c_int),
        ("prefill_base_us", C.c_double), ("prefill_per_token_us", C.c_double),
        ("decode_per_token_us", C.c_double),
    ]


class Snapshot(C.Structure):
    _fields_ = [
        ("n", C.c_long), ("keys", C.c_void_p), ("last_touch", C.c_void_p), ("has_agent", C.c_void_p),
        ("agents", C.c_void_p), ("refs", C.c_void_p),
    ]


class RunOut(C.Structure):
    _fields_ = [
        ("n_turns", C.c_long), ("cached_tokens", C.POINTER(C.c_long)),
        ("prompt_tokens", C.POINTER(C.c_long)), ("start_us", C.POINTER(C.c_double)),
        ("end_us", C.POINTER(C.c_double)), ("n_evictions", C.c_long),
        ("evictions", C.POINTER(C.c_uint64)), ("n_warmups", C.c_long),
        ("warmup_step", C.POINTER(C.c_long)), ("warmup_target", C.POINTER(C.c_uint64)),
        ("warmup_tick", C.POINTER(C.c_uint64)), ("hit_rate", C.c_double),
        ("truncated", C.c_long), ("warmups_executed", C.c_long), ("warmups_dropped", C.c_long),
        ("sim_us", C.c_double), ("n_steps", C.c_long), ("n_admissions", C.c_long),
        ("completed", C.POINTER(C.c_uint8)),
    ]


def build():
    subprocess.run(["make", "-s", "-C", _HERE, "oracle"], check=True)


def lib():
    global _lib
    if _lib is None:
        src = os.path.join(_HERE, "cs_oracle.c")
        if not os.path.exists(LIB_PATH) or (os.path.exists(src) and
                                            os.path.getmtime(src) > os.path.getmtime(LIB_PATH)):
            build()
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        L.cso_mix64.restype = C.c_uint64
        L.cso_mix64.argtypes = [C.c_uint64]
        L.cso_chain_hash.restype = C.c_uint64
        L.cso_chain_hash.argtypes = [C.c_int, C.c_uint64, vp, C.c_size_t, vp]
        L.cso_block_keys.restype = C.c_long
        L.cso_block_keys.argtypes = [vp, C.c_size_t, C.c_int, vp, vp]
        L.cso_identity.restype = C.c_int
        L.cso_identity.argtypes = [vp, C.c_size_t, C.c_int, C.c_int, vp]
        L.cso_generate.restype = C.c_long
        L.cso_generate.argtypes = [C.POINTER(Spec), vp, C.c_long]
        L.cso_turn_tokens.restype = C.c_long
        L.cso_turn_tokens.argtypes = [C.POINTER(Spec), vp, vp, C.c_long]
        L.cso_run.restype = C.c_int
        L.cso_run.argtypes = [C.POINTER(Spec), C.POINTER(Cfg), C.POINTER(RunOut)]
        L.cso_run_ex.restype = C.c_int
        L.cso_run_ex.argtypes = [C.POINTER(Spec), C.POINTER(Cfg), C.POINTER(Snapshot), C.c_long, C.POINTER(RunOut)]
        L.cso_free_run.argtypes = [C.POINTER(RunOut)]
        L.cso_engine_new.restype = vp
        L.cso_engine_new.argtypes = [C.POINTER(Cfg), C.c_long]
        L.cso_engine_free.argtypes = [vp]
        L.cso_engine_lookup.restype = C.c_long
        L.cso_engine_lookup.argtypes = [vp, vp, vp, C.c_long, vp]
        L.cso_engine_dispatch.restype = C.c_int
        L.cso_engine_dispatch.argtypes = [vp, C.c_uint64]
        L.cso_engine_admit_pinned.restype = C.c_int
        L.cso_engine_admit_pinned.argtypes = [vp, vp, vp, C.c_long, C.c_int, C.c_uint64, C.c_int]
        L.cso_engine_unpin.restype = C.c_int
        L.cso_engine_unpin.argtypes = [vp, vp, C.c_long]
        L.cso_engine_restore.restype = C.c_int
        L.cso_engine_restore.argtypes = [vp, vp, vp, vp, vp, vp, C.c_long, C.c_uint64]
        L.cso_engine_evictions.restype = C.c_long
        L.cso_engine_evictions.argtypes = [vp, vp, C.c_long]
        L.cso_engine_tick.restype = C.c_uint64
        L.cso_engine_tick.argtypes = [vp]
        L.cso_engine_resident.restype = C.c_long
        L.cso_engine_resident.argtypes = [vp]
        L.cso_engine_pinned.restype = C.c_long
        L.cso_engine_pinned.argtypes = [vp]
        L.cso_engine_poll.restype = C.c_long
        L.cso_engine_poll.argtypes = [vp, vp, vp, C.c_long]
        L.cso_engine_hops.restype = C.c_int
        L.cso_engine_hops.argtypes = [vp, vp, C.c_long, vp]
        L.cso_engine_scores.restype = C.c_long
        L.cso_engine_scores.argtypes = [vp, vp, vp, C.c_long]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def mix64(x):
    return int(lib().cso_mix64(x))


def chain_hash(parent, tokens):
    t = np.ascontiguousarray(tokens, dtype=np.uint32)
    err = C.c_int(0)
    h = lib().cso_chain_hash(0 if parent is None else 1, 0 if parent is None else parent, _p(t),
                             t.size, C.byref(err))
    if err.value:
        raise ValueError("chain_hash: token sequence must be nonempty")
    return int(h)


def block_keys(tokens, block_size=16):
    t = np.ascontiguousarray(tokens, dtype=np.uint32)
    n = max((t.size + block_size - 1) // block_size, 1)
    k = np.zeros(n, np.uint64)
    c = np.zeros(n, np.int32)
    m = lib().cso_block_keys(_p(t), t.size, block_size, _p(k), _p(c))
    if m < 0:
        raise ValueError("block_keys_for: block_size must be positive")
    return k[:m], c[:m]


def identity(keys, skip=4, take=4):
    k = np.ascontiguousarray(keys, dtype=np.uint64)
    out = C.c_uint64(0)
    if lib().cso_identity(_p(k), k.size, skip, take, C.byref(out)) != 0:
        raise ValueError("derive_agent_identity: invalid window or no block keys")
    return int(out.value)


def spec_struct(spec):
    anchors = np.ascontiguousarray(spec["anchor_tokens"], dtype=np.int32)
    trans = np.ascontiguousarray(spec["transition"], dtype=np.float64).reshape(-1)
    s = Spec()
    s.n_agents = anchors.size
    s.anchor_tokens = anchors.ctypes.data_as(C.POINTER(C.c_int))
    s.transition = trans.ctypes.data_as(C.POINTER(C.c_double))
    s.supervisor = -1 if spec.get("supervisor") is None else int(spec["supervisor"])
    for f in ("turns_min", "turns_max", "sessions", "task_tokens", "history_growth",
              "decode_tokens", "template_tokens", "concurrency", "budget_blocks"):
        setattr(s, f, int(spec[f]))
    s.seed = int(spec["seed"])
    s.anchor_stride = int(spec.get("anchor_stride", 0))
    s.hist_pos_bits = int(spec.get("hist_pos_bits", 0))
    sd = None
    if spec.get("start_dist") is not None:
        sd = np.ascontiguousarray(spec["start_dist"], dtype=np.float64)
        s.start_dist = sd.ctypes.data_as(C.POINTER(C.c_double))
        s.supervisor = -2
    s._keep = (anchors, trans, sd)
    return s


def generate(spec):
    s = spec_struct(spec)
    n = lib().cso_generate(C.byref(s), None, 0)
    out = np.zeros((max(n, 1), 7), np.int64)
    lib().cso_generate(C.byref(s), _p(out), n)
    return out[:n]


def turn_tokens(spec, turn7):
    s = spec_struct(spec)
    t = np.ascontiguousarray(turn7, dtype=np.int64)
    n = lib().cso_turn_tokens(C.byref(s), _p(t), None, 0)
    out = np.zeros(max(n, 1), np.uint32)
    lib().cso_turn_tokens(C.byref(s), _p(t), _p(out), n)
    return out[:n]


POLICY_IDS = {"lru": 0, "cachesage": 1, "ttl": 2, "belady": 3}


def cfg_struct(policy="cachesage", budget=None, concurrency=None, block_size=16, prefetch=True,
               skip=4, take=4, tau=0.01, e_max=8, w_pred=1.0, window=1024, min_confidence=0.5,
               min_row_count=5, budget_per_step=1, fast=False, cost=None):
    """fast: the indexed evict_one (exact by the class-head lemma; see cs_oracle.c). cost:
    (prefill_base_us, prefill_per_token_us, decode_per_token_us), None = the reference defaults."""
    c = Cfg()
    c.policy = POLICY_IDS[policy]
    c.budget_blocks = budget or 0
    c.concurrency = concurrency or 0
    c.block_size = block_size
    c.prefetch = 1 if prefetch else 0
    c.skip, c.take, c.tau, c.e_max, c.w_pred = skip, take, tau, e_max, w_pred
    c.window, c.min_confidence, c.min_row_count = window, min_confidence, min_row_count
    c.budget_per_step = budget_per_step
    c.fast_evict = 1 if fast else 0
    if cost is not None:
        c.prefill_base_us, c.prefill_per_token_us, c.decode_per_token_us = (float(x) for x in cost)
    return c


def run(spec, snapshot=None, max_steps=-1, **kw):
    """cso_run_ex: one simulation cell; snapshot = (keys, last_touch, agent ids or None per slot
    as a u64 array with has_agent mask, refs) installed before the first step; max_steps bounds
    the scheduler steps (-1: to the end)."""
    s = spec_struct(spec)
    c = cfg_struct(**kw)
    o = RunOut()
    snp = None
    if snapshot is not None:
        keys, lt, has, ids, refs = (np.ascontiguousarray(snapshot[0], np.uint64),
                                    np.ascontiguousarray(snapshot[1], np.uint64),
                                    np.ascontiguousarray(snapshot[2], np.int32),
                                    np.ascontiguousarray(snapshot[3], np.uint64),
                                    None if snapshot[4] is None else np.ascontiguousarray(snapshot[4], np.int32))
        snp = Snapshot(keys.size, keys.ctypes.data, lt.ctypes.data, has.ctypes.data, ids.ctypes.data,
                       None if refs is None else refs.ctypes.data)
        snp._keep = (keys, lt, has, ids, refs)
    rc = lib().cso_run_ex(C.byref(s), C.byref(c), None if snp is None else C.byref(snp), int(max_steps),
                          C.byref(o))
    try:
        if rc != 0:
            raise RuntimeError({-1: "evict_one: all resident blocks are pinned",
                                -2: "scheduler stalled with an idle engine",
                                -3: "EngineSim: cost model parameters must be positive",
                                -4: "snapshot: duplicate keys or larger than the budget"}.get(rc, str(rc)))
        nt, ne, nw = o.n_turns, o.n_evictions, o.n_warmups
        arr = lambda p, n, dt: (np.ctypeslib.as_array(p, (n,)).copy().astype(dt) if n > 0
                               else np.zeros(0, dt))
        return {
            "cached_tokens": arr(o.cached_tokens, nt, np.int64),
            "prompt_tokens": arr(o.prompt_tokens, nt, np.int64),
            "start_us": arr(o.start_us, nt, np.float64),
            "end_us": arr(o.end_us, nt, np.float64),
            "evictions": arr(o.evictions, ne, np.uint64),
            "warmup_step": arr(o.warmup_step, nw, np.int64),
            "warmup_target": arr(o.warmup_target, nw, np.uint64),
            "warmup_tick": arr(o.warmup_tick, nw, np.uint64),
            "hit_rate": o.hit_rate, "truncated": o.truncated,
            "warmups_executed": o.warmups_executed, "warmups_dropped": o.warmups_dropped,
            "sim_us": o.sim_us, "n_steps": o.n_steps, "n_admissions": o.n_admissions,
            "completed": arr(o.completed, nt, np.uint8).astype(bool),
        }
    finally:
        lib().cso_free_run(C.byref(o))


class Engine:
    """EngineSim surface of the oracle (pool + policy), for admission-level parity tests."""

    def __init__(self, budget, agent_cap=64, **kw):
        self._cfg = cfg_struct(budget=budget, **kw)
        self.h = lib().cso_engine_new(C.byref(self._cfg), agent_cap)

    def close(self):
        if self.h:
            lib().cso_engine_free(self.h)
            self.h = None

    __del__ = close

    def lookup(self, keys, counts):
        k = np.ascontiguousarray(keys, np.uint64)
        c = np.ascontiguousarray(counts, np.int32)
        fm = C.c_long(0)
        cached = lib().cso_engine_lookup(self.h, _p(k), _p(c), k.size, C.byref(fm))
        return int(cached), int(fm.value)

    def dispatch(self, agent):
        if lib().cso_engine_dispatch(self.h, agent) != 0:
            raise RuntimeError("agent capacity exceeded")

    def admit_pinned(self, keys, counts, agent=None, anchor=0):
        k = np.ascontiguousarray(keys, np.uint64)
        c = np.ascontiguousarray(counts, np.int32)
        if lib().cso_engine_admit_pinned(self.h, _p(k), _p(c), k.size, 0 if agent is None else 1,
                                         0 if agent is None else agent, anchor) != 0:
            raise RuntimeError("evict_one: all resident blocks are pinned")

    def unpin(self, keys):
        k = np.ascontiguousarray(keys, np.uint64)
        if lib().cso_engine_unpin(self.h, _p(k), k.size) != 0:
            raise RuntimeError("unpin: block vanished while referenced")

    def restore(self, keys, last_touch, agents=None, refs=None, tick=0):
        k = np.ascontiguousarray(keys, np.uint64)
        lt = np.ascontiguousarray(last_touch, np.uint64)
        if agents is None:
            has = np.zeros(k.size, np.int32)
            ag = np.zeros(k.size, np.uint64)
        else:
            ag = np.ascontiguousarray([0 if a is None else a for a in agents], np.uint64)
            has = np.ascontiguousarray([0 if a is None else 1 for a in agents], np.int32)
        r = None if refs is None else np.ascontiguousarray(refs, np.int32)
        if lib().cso_engine_restore(self.h, _p(k), _p(lt), _p(has), _p(ag),
                                    None if r is None else _p(r), k.size, tick) != 0:
            raise RuntimeError("restore failed")

    def evictions(self):
        n = lib().cso_engine_evictions(self.h, None, 0)
        out = np.zeros(max(n, 1), np.uint64)
        lib().cso_engine_evictions(self.h, _p(out), n)
        return out[:n]

    @property
    def tick(self):
        return int(lib().cso_engine_tick(self.h))

    @property
    def resident(self):
        return int(lib().cso_engine_resident(self.h))

    @property
    def pinned(self):
        return int(lib().cso_engine_pinned(self.h))

    def poll(self):
        n = lib().cso_engine_poll(self.h, None, None, 0)
        # poll drained the queue already when n>0 and cap 0; re-query is not possible, so the
        # API is: call with capacity first
        return n

    def poll_into(self, cap=64):
        t = np.zeros(cap, np.uint64)
        k = np.zeros(cap, np.uint64)
        n = lib().cso_engine_poll(self.h, _p(t), _p(k), cap)
        return t[:n], k[:n]

    def hops(self, agents):
        a = np.ascontiguousarray(agents, np.uint64)
        h = np.zeros(max(a.size, 1), np.int32)
        lib().cso_engine_hops(self.h, _p(a), a.size, _p(h))
        return h[:a.size]

    def scores(self):
        n = lib().cso_engine_scores(self.h, None, None, 0)
        k = np.zeros(max(n, 1), np.uint64)
        s = np.zeros(max(n, 1), np.float64)
        lib().cso_engine_scores(self.h, _p(k), _p(s), n)
        return k[:n], s[:n]


# ---------------------------------------------------------------------------------------------
# TransitionLearner / rebuild_reachability / exact_survival_prob, restated in Python for small
# alphabets (test-scale, like the reference's own oracle). Paths relative to /root/reference/proj.

class Learner:
    """TransitionLearner (transition_learner.cpp:10-96): alphabet in first-seen order, sparse
    counts and row totals over a sliding window of pairs."""

    def __init__(self, window=1024):
        if window <= 0:
            raise ValueError("TransitionLearner: window capacity must be positive")
        self.cap = window
        self.alphabet = []
        self._seen = set()
        self.window = []
        self.counts = {}  # a -> {b: n}
        self.totals = {}

    def note_agent(self, a):  # transition_learner.cpp:16-20
        if a not in self._seen:
            self._seen.add(a)
            self.alphabet.append(a)

    def record(self, a, b):  # transition_learner.cpp:22-51
        self.note_agent(a)
        self.note_agent(b)
        self.window.append((a, b))
        row = self.counts.setdefault(a, {})
        row[b] = row.get(b, 0) + 1
        self.totals[a] = self.totals.get(a, 0) + 1
        if len(self.window) > self.cap:
            oa, ob = self.window.pop(0)
            r = self.counts[oa]
            r[ob] -= 1
            if r[ob] == 0:
                del r[ob]
            if not r:
                del self.counts[oa]
            self.totals[oa] -= 1
            if self.totals[oa] == 0:
                del self.totals[oa]

    def prob(self, a, b):  # transition_learner.cpp:53-67
        t = self.totals.get(a, 0)
        c = self.counts.get(a, {}).get(b, 0)
        return 0.0 if t == 0 or c == 0 else float(c) / float(t)

    def row_total(self, a):
        return self.totals.get(a, 0)

    def argmax_row(self, a):  # transition_learner.cpp:79-96 (ties -> smaller id)
        r = self.counts.get(a)
        t = self.totals.get(a, 0)
        if not r or t == 0:
            return None
        best, bc = None, 0
        for b, c in r.items():
            if best is None or c > bc or (c == bc and b < best):
                best, bc = b, c
        return best, float(bc) / float(t)

    def state_bytes(self):  # transition_learner.cpp:98-106
        nz = sum(len(r) for r in self.counts.values())
        return len(self.window) * 4 + nz * 12 + len(self.totals) * 10 + len(self.alphabet) * 8 + 8


def rebuild_reachability(learner, current, tau, e_max):
    """reachability.cpp:39-81: hop per agent (e_max = unreachable)."""
    if e_max <= 0:
        raise ValueError("rebuild_reachability: e_max must be positive")
    hops = {a: e_max for a in learner.alphabet}
    hops[current] = 0
    frontier = [current]
    while frontier:
        a = frontier.pop(0)
        d = hops[a]
        if d + 1 >= e_max:
            continue
        row = learner.counts.get(a)
        if not row:
            continue
        total = float(learner.totals[a])
        for b, c in row.items():
            if float(c) / total < tau:
                continue
            if hops.get(b, e_max) > d + 1:
                hops[b] = d + 1
                frontier.append(b)
    return hops


def exact_survival_prob(target, k, learner, current):
    """survival_oracle.cpp:9-62, fp64 operations in the reference's order."""
    agents = learner.alphabet
    if len(agents) > 64:
        raise ValueError("exact_survival_prob: alphabet too large (test-scale <= 64)")
    if k > 32:
        raise ValueError("exact_survival_prob: horizon too deep (test-scale <= 32)")
    if k < 0:
        raise ValueError("exact_survival_prob: negative horizon")
    if target == current:
        return 1.0
    index = {a: i for i, a in enumerate(agents)}
    if target not in index or current not in index:
        return 0.0
    n = len(agents)
    ti = index[target]
    dist = [0.0] * n
    dist[index[current]] = 1.0
    absorbed = 0.0
    for _ in range(k):
        nxt = [0.0] * n
        for i in range(n):
            if dist[i] == 0.0:
                continue
            row = learner.counts.get(agents[i])
            if not row:
                continue
            total = float(learner.totals[agents[i]])
            for b, c in row.items():
                nxt[index[b]] += dist[i] * float(c) / total
        absorbed += nxt[ti]
        nxt[ti] = 0.0
        dist = nxt
    return absorbed
