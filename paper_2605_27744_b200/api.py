"""Python mirror of the reference's public surface, backed by the sm_100a library.

Names and argument meaning follow the reference's python module (py_module.cpp:79-186,
python/cachesage/__init__.py) and C++ classes (EngineSim engine.hpp:90-208, CacheSagePolicy
cachesage_policy.hpp:48-85). Everything computes on the GPU through include/cachesage_b200.h.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import workloads
from ._lib import (CS_NO_AGENT, EV_AGENT_DISPATCH, EV_BLOCK_TOUCH, EV_REQUEST_ARRIVAL, EV_TOOL_RETURN,
                   EV_TURN_COMPLETE, EngineCfg, EngineResult, Event, PoolCfg, PoolStats, WorkloadSpec, check,
                   lib)

EVENT_KINDS = {"block_touch": EV_BLOCK_TOUCH, "request_arrival": EV_REQUEST_ARRIVAL,
               "agent_dispatch": EV_AGENT_DISPATCH, "tool_return": EV_TOOL_RETURN,
               "turn_complete": EV_TURN_COMPLETE}

POLICIES = {"lru": 0, "cachesage": 1, "ttl": 2, "belady": 3}


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _u64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def pool_cfg(budget, policy="cachesage", e_max=8, tau=0.01, w_pred=1.0, window=1024, min_confidence=0.5,
             min_row_count=5, budget_per_step=1, agent_capacity=1024, device=0, grid_ctas=0):
    c = PoolCfg()
    lib().cs_pool_cfg_default(C.byref(c))
    c.budget_blocks = int(budget)
    c.policy = POLICIES[policy]
    c.e_max, c.tau, c.w_pred, c.window = e_max, tau, w_pred, window
    c.min_confidence, c.min_row_count, c.budget_per_step = min_confidence, min_row_count, budget_per_step
    c.agent_capacity, c.device, c.grid_ctas = agent_capacity, device, grid_ctas
    return c


class Pool:
    """A device block pool + transition learner (cs_pool_t).

    The per-call methods mirror EngineSim::lookup / admit_pinned / unpin (engine.cpp:127-180)
    and CacheSagePolicy::observe / poll_actions / score (cachesage_policy.cpp:50-130); the
    caller owns the tick clock exactly like EngineSim::tick_.
    """

    def __init__(self, budget, **kw):
        self._cfg = pool_cfg(budget, **kw)
        h = C.c_void_p()
        check(lib().cs_pool_create(C.byref(self._cfg), C.byref(h)))
        self.h = h
        self.budget = int(budget)

    def close(self):
        if getattr(self, "h", None):
            lib().cs_pool_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def register_agents(self, ids):
        ids = _u64(ids)
        first = C.c_int(0)
        check(lib().cs_register_agents(self.h, _p(ids), ids.size, C.byref(first)))
        return first.value

    def lookup(self, keys, counts, tick_base):
        keys, counts = _u64(keys), _i32(counts)
        cached, fm = C.c_int64(0), C.c_int(0)
        check(lib().cs_lookup(self.h, _p(keys), _p(counts), keys.size, tick_base, C.byref(cached), C.byref(fm)))
        return cached.value, fm.value

    def probe_needed(self, keys):
        keys = _u64(keys)
        n = C.c_int(0)
        check(lib().cs_probe_needed(self.h, _p(keys), keys.size, C.byref(n)))
        return n.value

    def observe_dispatch(self, prev, nxt, tick):
        w = C.c_int(-1)
        check(lib().cs_observe_dispatch(self.h, -1 if prev is None else prev, nxt, tick, C.byref(w)))
        return None if w.value < 0 else w.value

    def admit_pinned(self, keys, counts, agent=None, anchor=0, tick_base=0):
        keys, counts = _u64(keys), _i32(counts)
        n = keys.size
        ev = np.zeros(max(n, 1), np.uint64)
        pins = np.zeros(max(n, 1), np.uint32)
        ne = C.c_int64(0)
        check(lib().cs_admit_pinned(self.h, _p(keys), _p(counts), n, CS_NO_AGENT if agent is None else agent,
                                    anchor, tick_base, _p(ev), ev.size, C.byref(ne), _p(pins)))
        return ev[:ne.value].copy(), pins[:n].copy()

    def unpin(self, keys):
        """EngineSim::unpin (engine.cpp:170-180): one pin per BlockKey; a key that is not resident
        raises RuntimeError (logic_error "unpin: block vanished while referenced")."""
        k = _u64(keys)
        check(lib().cs_unpin(self.h, _p(k), k.size))

    def unpin_slots(self, slots):
        """The same by the pinned slots admit_pinned returned (no table probe)."""
        s = np.ascontiguousarray(slots, dtype=np.uint32)
        check(lib().cs_unpin_slots(self.h, _p(s), s.size))

    def dispatch_event(self, tick, kind, agent=-1, prev=None, request=0):
        """Runtime::dispatch_event (runtime.cpp:59-69) -> observe. kind: a key of EVENT_KINDS.
        A tick below the previous event's raises RuntimeError (tick regression). Returns the
        agent index of a warmup the dispatch issued, or None."""
        ev = Event(int(tick), EVENT_KINDS[kind], int(agent), -1 if prev is None else int(prev), int(request))
        w = C.c_int(-1)
        check(lib().cs_dispatch_event(self.h, C.byref(ev), C.byref(w)))
        return None if w.value < 0 else w.value

    def predict(self, horizon=1, current=None):
        """CacheSagePolicy::predict(horizon) / predict_next(current, horizon)
        (cachesage_policy.cpp:87-107): [(agent_id, probability, agent_index)] ranked by
        probability (ties: smaller AgentId first). The Forecast's distribution is
        {id: p for id, p, _ in result}."""
        cap = max(self.stats()["n_agents"], 1)
        ids, pr, ix = np.zeros(cap, np.uint64), np.zeros(cap, np.float64), np.zeros(cap, np.int32)
        n = C.c_int(0)
        check(lib().cs_predict(self.h, int(horizon), -1 if current is None else int(current), _p(ids), _p(pr),
                               _p(ix), cap, C.byref(n)))
        return [(int(ids[i]), float(pr[i]), int(ix[i])) for i in range(n.value)]

    def serialize_state(self):
        """Policy::serialize_state().dump() (cachesage_policy.cpp:139-153), as a str."""
        return serialize_state(self.h)

    def state_bytes(self):
        """CacheSagePolicy::state_bytes (cachesage_policy.cpp:133-138)."""
        b = C.c_uint64(0)
        check(lib().cs_policy_state_bytes(self.h, C.byref(b)))
        return b.value

    def restore(self, keys, last_touch, agents=None, refs=None):
        keys, lt = _u64(keys), _u64(last_touch)
        ag = None if agents is None else np.ascontiguousarray(agents, dtype=np.uint32)
        rf = None if refs is None else np.ascontiguousarray(refs, dtype=np.uint32)
        check(lib().cs_restore(self.h, _p(keys), _p(lt), None if ag is None else _p(ag),
                               None if rf is None else _p(rf), keys.size))

    def score_snapshot(self, now_tick):
        st = self.stats()
        cap = max(st["resident"], 1)
        k = np.zeros(cap, np.uint64)
        s = np.zeros(cap, np.float64)
        n = C.c_int64(0)
        check(lib().cs_score_snapshot(self.h, now_tick, _p(k), _p(s), cap, C.byref(n)))
        return k[:n.value], s[:n.value]

    def set_hops(self, hops):
        """Install externally computed reachability hops (cs_set_hops), per agent index."""
        h = np.ascontiguousarray(hops, dtype=np.uint8)
        check(lib().cs_set_hops(self.h, _p(h), h.size))

    def hops(self, n):
        h = np.zeros(max(n, 1), np.int32)
        check(lib().cs_hops(self.h, _p(h), n))
        return h[:n]

    def poll_actions(self, cap=64):
        t = np.zeros(cap, np.int32)
        k = np.zeros(cap, np.uint64)
        n = C.c_int(0)
        check(lib().cs_poll_actions(self.h, _p(t), _p(k), cap, C.byref(n)))
        return t[:n.value].copy(), k[:n.value].copy()

    def stats(self):
        s = PoolStats()
        check(lib().cs_pool_get_stats(self.h, C.byref(s)))
        d = {f: getattr(s, f) for f, _ in PoolStats._fields_}
        d["phase_ns"] = list(s.phase_ns)
        return d


def serialize_state(pool_handle):
    n = C.c_size_t(0)
    check(lib().cs_serialize_state(pool_handle, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(lib().cs_serialize_state(pool_handle, buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


def hash_prompts(prompts, block_size=16, skip=4, take=4, pool=None):
    """K1 over a list of token sequences: (keys per prompt, counts per prompt, agent ids)."""
    own = pool is None
    if own:
        pool = Pool(1024)
    try:
        lens = np.array([len(p) for p in prompts], dtype=np.int64)
        tok_off = np.zeros(len(prompts) + 1, np.int64)
        tok_off[1:] = np.cumsum(lens)
        tokens = np.concatenate([np.asarray(p, dtype=np.uint32) for p in prompts]) if prompts else np.zeros(0, np.uint32)
        tokens = np.ascontiguousarray(tokens, dtype=np.uint32)
        blk_off = np.zeros(len(prompts) + 1, np.int64)
        nblk = lib().cs_blocks_for(_p(tok_off), len(prompts), block_size, _p(blk_off))
        if nblk < 0:
            raise ValueError("block_keys_for: block_size must be positive")
        keys = np.zeros(max(nblk, 1), np.uint64)
        counts = np.zeros(max(nblk, 1), np.int32)
        agents = np.zeros(max(len(prompts), 1), np.uint64)
        check(lib().cs_hash_prompts(pool.h, _p(tokens), _p(tok_off), len(prompts), block_size, skip, take,
                                    _p(blk_off), _p(keys), _p(counts), _p(agents)))
        ks = [keys[blk_off[i]:blk_off[i + 1]].copy() for i in range(len(prompts))]
        cs = [counts[blk_off[i]:blk_off[i + 1]].copy() for i in range(len(prompts))]
        return ks, cs, agents[:len(prompts)].copy()
    finally:
        if own:
            pool.close()


def chain_hash(parent, tokens):
    """chain_hash (hashing.cpp:26-35; Python binding py_module.cpp:82-88) on the GPU: parent None
    chains from the root. Empty token sequences are invalid_argument (ValueError)."""
    toks = np.ascontiguousarray(tokens, dtype=np.uint32)
    off = np.array([0, toks.size], np.int64)
    par = np.array([0 if parent is None else int(parent)], np.uint64)
    hp = np.array([0 if parent is None else 1], np.uint8)
    out = np.zeros(1, np.uint64)
    check(lib().cs_chain_hash(_p(par), _p(hp), _p(toks), _p(off), 1, _p(out)))
    return int(out[0])


def derive_agent_identity(block_keys, skip=4, take=4):
    """derive_agent_identity (cachesage_policy.cpp:9-31; py_module.cpp:90-101) on the GPU."""
    k = _u64(block_keys)
    off = np.array([0, k.size], np.int64)
    out = np.zeros(1, np.uint64)
    check(lib().cs_derive_agent_identity(_p(k) if k.size else None, _p(off), 1, skip, take, _p(out)))
    return int(out[0])


class TransitionLearner:
    """TransitionLearner (transition_learner.hpp:19-60; Python binding py_module.cpp:103-123)
    on the device: record (K3), prob, row_total, agents, state_bytes, argmax_row (K6) and the
    reachability rebuild (K3b). Agent ids are the 64-bit AgentId values."""

    def __init__(self, window=1024, agent_capacity=1024, device=0):
        h = C.c_void_p()
        check(lib().cs_learner_create(int(window), int(agent_capacity), int(device), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().cs_learner_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def record(self, prev, nxt):
        self.record_many([prev], [nxt])

    def record_many(self, prev, nxt):
        """record() of each (prev[i], next[i]) in order, as one device batch."""
        a, b = _u64(prev), _u64(nxt)
        if a.size != b.size:
            raise ValueError("record_many: prev and next differ in length")
        check(lib().cs_learner_record(self.h, _p(a), _p(b), a.size))

    def prob(self, a, b):
        p = C.c_double(0.0)
        check(lib().cs_learner_prob(self.h, int(a), int(b), C.byref(p)))
        return p.value

    def row_total(self, a):
        t = C.c_uint64(0)
        check(lib().cs_learner_row_total(self.h, int(a), C.byref(t)))
        return t.value

    def agents(self):
        n = check(lib().cs_learner_agents(self.h, None, 0))
        out = np.zeros(max(n, 1), np.uint64)
        lib().cs_learner_agents(self.h, _p(out), n)
        return [int(x) for x in out[:n]]

    def state_bytes(self):
        b = C.c_uint64(0)
        check(lib().cs_learner_state_bytes(self.h, C.byref(b)))
        return b.value

    def argmax_row(self, a):
        """(best successor id, probability), or None for an unseen row (ties -> smaller id)."""
        best, p, found = C.c_uint64(0), C.c_double(0.0), C.c_int(0)
        check(lib().cs_learner_argmax(self.h, int(a), C.byref(best), C.byref(p), C.byref(found)))
        return (best.value, p.value) if found.value else None

    def rebuild_reachability(self, current, tau=0.01, e_max=8):
        """rebuild_reachability (reachability.cpp:39-81): {agent id: hop} over the known agents
        (plus `current` at hop 0, as the reference inserts it)."""
        ids = self.agents()
        hops = np.zeros(max(len(ids), 1), np.int32)
        check(lib().cs_learner_rebuild(self.h, int(current), float(tau), int(e_max), _p(hops), len(ids)))
        out = {a: int(h) for a, h in zip(ids, hops[:len(ids)])}
        out[int(current)] = 0
        return out


def exact_survival_prob(target, k, matrix, current):
    """oracle::exact_survival_prob (survival_oracle.cpp:9-62; py_module.cpp:125-131) on the GPU:
    P(a walk from `current` visits `target` within k steps) on the learner's MLE matrix. Same
    fp64 operation order as the reference; alphabet <= 64 and k <= 32 (else ValueError)."""
    out = C.c_double(0.0)
    check(lib().cs_exact_survival_prob(matrix.h, int(target), int(k), int(current), C.byref(out)))
    return out.value


def block_keys_for(tokens, block_size=16):
    ks, cs, _ = hash_prompts([tokens], block_size=block_size)
    return ks[0], cs[0]


def derive_agent_identity_of_prompt(tokens, block_size=16, skip=4, take=4):
    _, _, ag = hash_prompts([tokens], block_size=block_size, skip=skip, take=take)
    return int(ag[0])


def spec_struct(spec):
    anchors = np.ascontiguousarray(spec["anchor_tokens"], dtype=np.int32)
    trans = np.ascontiguousarray(spec["transition"], dtype=np.float64).reshape(-1)
    s = WorkloadSpec()
    s.n_agents = anchors.size
    s.anchor_tokens = anchors.ctypes.data_as(C.POINTER(C.c_int))
    s.transition = trans.ctypes.data_as(C.POINTER(C.c_double))
    s.supervisor = -1 if spec.get("supervisor") is None else int(spec["supervisor"])
    for f in ("turns_min", "turns_max", "sessions", "task_tokens", "history_growth", "decode_tokens",
              "template_tokens", "concurrency", "budget_blocks"):
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


def generate_trace_rows(spec):
    """generate_trace (workload.cpp:156-182): rows (session, turn, agent, anchor, history,
    prompt, decode). Host code (no GPU needed). The reference's Trace API: trace.generate_trace."""
    s = spec_struct(spec)
    n = check(lib().cs_generate_trace(C.byref(s), None, 0))
    out = np.zeros((max(n, 1), 7), np.int64)
    lib().cs_generate_trace(C.byref(s), _p(out), n)
    return out[:n]


class Engine:
    """EngineSim (engine.hpp:90-208) with the block pool, learner and eviction on the GPU."""

    def __init__(self, spec, policy="cachesage", budget=None, concurrency=None, block_size=16, prefetch=True,
                 skip=4, take=4, timing=False, host_inputs=False, comm=None, shard_slots=0,
                 device_scheduler=False, cost_model=None, **pool_kw):
        """comm (shard.Comm): this engine drives ONE shard of a hash-sharded pool of global
        budget `budget`; every shard runs the same trace and reaches the same
        decisions. shard_slots: the shard's physical slots (0 = 1.25 budget / world + 4096).
        cost_model: dict with any of prefill_per_token_us / prefill_base_us / decode_per_token_us
        (CostModel, engine.hpp:22-26; the experiment config's "cost_model", experiment.cpp:270-280)."""
        cfg = EngineCfg()
        lib().cs_engine_cfg_default(C.byref(cfg))
        cfg.pool = pool_cfg(budget or 0, policy=policy, **pool_kw)
        cfg.concurrency = concurrency or 0
        cfg.block_size = block_size
        cfg.prefetch = 1 if prefetch else 0
        cfg.skip, cfg.take = skip, take
        cfg.timing = 1 if timing else 0
        cfg.host_inputs = 1 if host_inputs else 0
        cfg.device_scheduler = 1 if device_scheduler else 0
        for k, v in (cost_model or {}).items():
            if k not in ("prefill_per_token_us", "prefill_base_us", "decode_per_token_us"):
                raise ValueError(f"unknown cost_model key {k!r}")
            setattr(cfg, k, float(v))
        self._spec = spec_struct(spec)
        self._spec_dict = spec
        self._policy = policy
        h = C.c_void_p()
        self.comm = comm
        if comm is None:
            check(lib().cs_engine_create(C.byref(cfg), C.byref(self._spec), C.byref(h)))
        else:
            check(lib().cs_engine_create_sharded(C.byref(cfg), C.byref(self._spec), int(shard_slots), comm.h,
                                                 C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().cs_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self):
        d = C.c_int(0)
        check(lib().cs_engine_step(self.h, C.byref(d)))
        return bool(d.value)

    def run(self):
        check(lib().cs_engine_run(self.h))
        return self.result()

    def run_for(self, admissions):
        d = C.c_int(0)
        check(lib().cs_engine_run_for(self.h, admissions, C.byref(d)))
        return bool(d.value)

    def run_timed(self, admissions):
        """(device milliseconds from CUDA events on the engine stream, done)."""
        ms, d = C.c_double(0), C.c_int(0)
        check(lib().cs_engine_run_timed(self.h, admissions, C.byref(ms), C.byref(d)))
        return ms.value, bool(d.value)

    def agents(self):
        n = check(lib().cs_engine_agents(self.h, None, 0))
        out = np.zeros(max(n, 1), np.uint64)
        lib().cs_engine_agents(self.h, _p(out), n)
        return out[:n]

    def restore(self, keys, last_touch, agents=None, refs=None):
        keys, lt = _u64(keys), _u64(last_touch)
        ag = None if agents is None else np.ascontiguousarray(agents, dtype=np.uint32)
        rf = None if refs is None else np.ascontiguousarray(refs, dtype=np.uint32)
        check(lib().cs_engine_restore(self.h, _p(keys), _p(lt), None if ag is None else _p(ag),
                                      None if rf is None else _p(rf), keys.size))

    def pool_stats(self):
        """Pool counters of the engine's device pool (cs_pool_get_stats), incl. the per-phase
        device time of the admission kernel (phase_ns, CTA-0 globaltimer)."""
        s = PoolStats()
        check(lib().cs_pool_get_stats(lib().cs_engine_pool(self.h), C.byref(s)))
        d = {f: getattr(s, f) for f, _ in PoolStats._fields_}
        d["phase_ns"] = list(s.phase_ns)
        return d

    def result(self):
        r = EngineResult()
        check(lib().cs_engine_result_get(self.h, C.byref(r)))
        return {f: getattr(r, f) for f, _ in EngineResult._fields_}

    def turns(self):
        n = self.result()["turns"]
        cached = np.zeros(max(n, 1), np.int64)
        prompt = np.zeros(max(n, 1), np.int64)
        st = np.zeros(max(n, 1), np.float64)
        en = np.zeros(max(n, 1), np.float64)
        check(lib().cs_engine_turns(self.h, _p(cached), _p(prompt), _p(st), _p(en), n))
        return {"cached_tokens": cached[:n], "prompt_tokens": prompt[:n], "start_us": st[:n], "end_us": en[:n]}

    def serialize_state(self):
        """The engine policy's Policy::serialize_state().dump() (cachesage_policy.cpp:139-153)."""
        return serialize_state(lib().cs_engine_pool(self.h))

    def evictions(self):
        n = check(lib().cs_engine_evictions(self.h, None, 0))
        out = np.zeros(max(n, 1), np.uint64)
        lib().cs_engine_evictions(self.h, _p(out), n)
        return out[:n]

    def check(self):
        """Pool invariants (cs_pool_check): all zero on a consistent pool."""
        out = np.zeros(4, np.int64)
        check(lib().cs_pool_check(lib().cs_engine_pool(self.h), _p(out)))
        return {"pk_mismatch": int(out[0]), "resident_delta": int(out[1]), "pinned_delta": int(out[2]),
                "table_mismatch": int(out[3])}

    def record_events(self, on=True):
        """Record EngineSim's event stream (engine.cpp:72-88) for write_outputs' events.jsonl;
        call before the first step (host scheduler only)."""
        check(lib().cs_engine_record_events(self.h, 1 if on else 0))

    def write_outputs(self, out_dir, workload=None, policy=None, seed=None, labels=None, events=True):
        """run_experiment's per-cell files (experiment.cpp:94-183, 424-440) for this finished run:
        <out_dir>/metrics.json, turns.csv and (events) events.jsonl, byte-identical to the
        reference's. Defaults come from the spec this engine was built from."""
        import os

        spec = self._spec_dict
        workload = workload if workload is not None else spec.get("name", "custom")
        policy = policy if policy is not None else self._policy
        seed = int(seed if seed is not None else spec.get("seed", 0))
        labels = list(labels if labels is not None else spec.get("labels", []))
        os.makedirs(out_dir, exist_ok=True)
        arr = (C.c_char_p * max(1, len(labels)))(*[x.encode() for x in labels])
        check(lib().cs_engine_write_outputs(self.h, str(out_dir).encode(), workload.encode(), policy.encode(), seed,
                                            C.cast(arr, C.c_void_p), len(labels), 1 if events else 0))

    def warmups(self):
        n = check(lib().cs_engine_warmups(self.h, None, None, None, 0))
        st = np.zeros(max(n, 1), np.int64)
        tg = np.zeros(max(n, 1), np.uint64)
        tk = np.zeros(max(n, 1), np.uint64)
        lib().cs_engine_warmups(self.h, _p(st), _p(tg), _p(tk), n)
        return st[:n], tg[:n], tk[:n]


def run_sim_spec(spec, policy="cachesage", budget=None, concurrency=None, block_size=16, prefetch=True, **kw):
    """One (spec, policy) simulation; the engine's own result dict (see trace.run_sim for the
    reference's metrics dict)."""
    if isinstance(spec, str):
        spec = workloads.preset_by_name(spec)
    eng = Engine(spec, policy=policy, budget=budget, concurrency=concurrency, block_size=block_size,
                 prefetch=prefetch, **kw)
    try:
        return eng.run()
    finally:
        eng.close()
