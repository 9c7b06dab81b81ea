"""Loader of the in-tree libcachesage_b200.so (the C ABI of include/cachesage_b200.h).

There is no CPU fallback: when the library is missing or no CUDA device is present every
compute entry point raises. The shared object is built in-tree by build.py (nvcc, sm_100a).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcachesage_b200.so")

CS_OK = 0
CS_ERR_INVALID_ARGUMENT = -1
CS_ERR_RUNTIME = -2
CS_ERR_LOGIC = -3
CS_ERR_CUDA = -4
CS_ERR_CAPACITY = -5
CS_NO_AGENT = 0xFFFFFFFF

vp = C.c_void_p


class Event(C.Structure):
    """cs_event: one observe-stream Event (types.hpp:51-82)."""
    _fields_ = [("tick", C.c_uint64), ("kind", C.c_int), ("agent", C.c_int), ("prev", C.c_int),
                ("request", C.c_uint64)]


EV_BLOCK_TOUCH, EV_REQUEST_ARRIVAL, EV_AGENT_DISPATCH, EV_TOOL_RETURN, EV_TURN_COMPLETE = range(5)


class PoolCfg(C.Structure):
    _fields_ = [
        ("budget_blocks", C.c_int64), ("policy", C.c_int), ("e_max", C.c_int), ("tau", C.c_double),
        ("w_pred", C.c_double), ("window", C.c_int64), ("min_confidence", C.c_double),
        ("min_row_count", C.c_uint64), ("budget_per_step", C.c_int), ("agent_capacity", C.c_int),
        ("device", C.c_int), ("grid_ctas", C.c_int),
    ]


class PoolStats(C.Structure):
    _fields_ = [
        ("resident", C.c_int64), ("pinned", C.c_int64), ("evictions", C.c_int64),
        ("tombstones", C.c_int64), ("scans", C.c_int64), ("scanned_slots", C.c_int64),
        ("rebuilds", C.c_uint64), ("n_agents", C.c_int), ("phase_ns", C.c_uint64 * 16),
        ("prescan_used", C.c_int64), ("prescan_fallbacks", C.c_int64), ("prescan_unusable", C.c_int64),
        ("server_launches", C.c_int64), ("host_turnarounds", C.c_int64), ("host_turnaround_ns", C.c_uint64),
    ]


class WorkloadSpec(C.Structure):
    _fields_ = [
        ("n_agents", C.c_int), ("anchor_tokens", C.POINTER(C.c_int)),
        ("transition", C.POINTER(C.c_double)), ("supervisor", C.c_int),
        ("turns_min", C.c_int), ("turns_max", C.c_int), ("sessions", C.c_int),
        ("task_tokens", C.c_int), ("history_growth", C.c_int), ("decode_tokens", C.c_int),
        ("template_tokens", C.c_int), ("concurrency", C.c_int), ("budget_blocks", C.c_int),
        ("seed", C.c_uint64), ("anchor_stride", C.c_uint32), ("hist_pos_bits", C.c_int),
        ("start_dist", C.POINTER(C.c_double)),
    ]


class EngineCfg(C.Structure):
    _fields_ = [
        ("pool", PoolCfg), ("concurrency", C.c_int), ("block_size", C.c_int), ("prefetch", C.c_int),
        ("skip", C.c_int), ("take", C.c_int), ("timing", C.c_int), ("host_inputs", C.c_int),
        ("device_scheduler", C.c_int), ("prefill_per_token_us", C.c_double),
        ("prefill_base_us", C.c_double), ("decode_per_token_us", C.c_double),
    ]


class EngineResult(C.Structure):
    _fields_ = [
        ("turns", C.c_int64), ("completed", C.c_int64), ("hit_rate", C.c_double),
        ("total_prompt_tokens", C.c_int64), ("total_cached_tokens", C.c_int64),
        ("evictions", C.c_int64), ("truncated", C.c_int64), ("warmups_executed", C.c_int64),
        ("warmups_dropped", C.c_int64), ("warmups_issued", C.c_int64), ("sim_us", C.c_double),
        ("steps", C.c_int64), ("admissions", C.c_int64), ("scans", C.c_int64),
        ("scanned_slots", C.c_int64), ("tick", C.c_uint64), ("scan_ms", C.c_double),
        ("admit_ms", C.c_double), ("scan_launches", C.c_int64), ("h2d_bytes", C.c_int64),
        ("d2h_bytes", C.c_int64), ("gpu_launches", C.c_int64), ("warmup_prompt_tokens", C.c_int64),
    ]


# name -> (restype, argtypes); mirrors include/cachesage_b200.h one to one
SIGNATURES = {
    "cs_pool_cfg_default": (None, [C.POINTER(PoolCfg)]),
    "cs_pool_create": (C.c_int, [C.POINTER(PoolCfg), C.POINTER(vp)]),
    "cs_pool_destroy": (C.c_int, [vp]),
    "cs_register_agents": (C.c_int, [vp, vp, C.c_int, C.POINTER(C.c_int)]),
    "cs_hash_prompts": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp]),
    "cs_blocks_for": (C.c_int64, [vp, C.c_int, C.c_int, vp]),
    "cs_lookup": (C.c_int, [vp, vp, vp, C.c_int, C.c_uint64, C.POINTER(C.c_int64), C.POINTER(C.c_int)]),
    "cs_probe_needed": (C.c_int, [vp, vp, C.c_int, C.POINTER(C.c_int)]),
    "cs_observe_dispatch": (C.c_int, [vp, C.c_int, C.c_int, C.c_uint64, C.POINTER(C.c_int)]),
    "cs_admit_pinned": (C.c_int, [vp, vp, vp, C.c_int, C.c_uint32, C.c_int, C.c_uint64, vp, C.c_int64,
                                  C.POINTER(C.c_int64), vp]),
    "cs_unpin_slots": (C.c_int, [vp, vp, C.c_int]),
    "cs_unpin": (C.c_int, [vp, vp, C.c_int]),
    "cs_dispatch_event": (C.c_int, [vp, C.POINTER(Event), C.POINTER(C.c_int)]),
    "cs_predict": (C.c_int, [vp, C.c_int, C.c_int, vp, vp, vp, C.c_int, C.POINTER(C.c_int)]),
    "cs_serialize_state": (C.c_int, [vp, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "cs_policy_state_bytes": (C.c_int, [vp, C.POINTER(C.c_uint64)]),
    "cs_restore": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64]),
    "cs_score_snapshot": (C.c_int, [vp, C.c_uint64, vp, vp, C.c_int64, C.POINTER(C.c_int64)]),
    "cs_hops": (C.c_int, [vp, vp, C.c_int]),
    "cs_poll_actions": (C.c_int, [vp, vp, vp, C.c_int, C.POINTER(C.c_int)]),
    "cs_pool_get_stats": (C.c_int, [vp, C.POINTER(PoolStats)]),
    "cs_pool_debug": (C.c_int, [vp, vp, C.c_int, C.POINTER(C.c_int)]),
    "cs_pool_check": (C.c_int, [vp, vp]),
    "cs_set_hops": (C.c_int, [vp, vp, C.c_int]),
    "cs_generate_trace": (C.c_int64, [C.POINTER(WorkloadSpec), vp, C.c_int64]),
    "cs_engine_cfg_default": (None, [C.POINTER(EngineCfg)]),
    "cs_engine_create": (C.c_int, [C.POINTER(EngineCfg), C.POINTER(WorkloadSpec), C.POINTER(vp)]),
    "cs_engine_destroy": (C.c_int, [vp]),
    "cs_engine_step": (C.c_int, [vp, C.POINTER(C.c_int)]),
    "cs_engine_run": (C.c_int, [vp]),
    "cs_engine_run_for": (C.c_int, [vp, C.c_int64, C.POINTER(C.c_int)]),
    "cs_engine_run_timed": (C.c_int, [vp, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_int)]),
    "cs_engine_restore": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64]),
    "cs_engine_agents": (C.c_int, [vp, vp, C.c_int]),
    "cs_engine_result_get": (C.c_int, [vp, C.POINTER(EngineResult)]),
    "cs_engine_turns": (C.c_int, [vp, vp, vp, vp, vp, C.c_int64]),
    "cs_engine_evictions": (C.c_int64, [vp, vp, C.c_int64]),
    "cs_engine_warmups": (C.c_int64, [vp, vp, vp, vp, C.c_int64]),
    "cs_engine_pool": (vp, [vp]),
    "cs_comm_local_group": (C.c_int, [C.c_int, vp]),
    "cs_comm_callback": (C.c_int, [C.c_int, C.c_int, vp, vp, C.POINTER(vp)]),
    "cs_nccl_unique_id": (C.c_int, [vp]),
    "cs_comm_nccl": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]),
    "cs_comm_destroy": (C.c_int, [vp]),
    "cs_comm_peer_group": (C.c_int, [C.c_int, vp, C.c_size_t, vp]),
    "cs_comm_peer_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_size_t, vp, C.POINTER(vp)]),
    "cs_comm_peer_connect": (C.c_int, [vp, vp]),
    "cs_comm_allgather_host": (C.c_int, [vp, vp, vp, C.c_size_t]),
    "cs_shard_owner": (C.c_int, [C.c_uint64, C.c_int]),
    "cs_pool_create_sharded": (C.c_int, [C.POINTER(PoolCfg), C.c_int64, vp, C.POINTER(vp)]),
    "cs_engine_create_sharded": (C.c_int, [C.POINTER(EngineCfg), C.POINTER(WorkloadSpec), C.c_int64, vp,
                                           C.POINTER(vp)]),
    "cs_learner_create": (C.c_int, [C.c_int64, C.c_int, C.c_int, C.POINTER(vp)]),
    "cs_learner_destroy": (C.c_int, [vp]),
    "cs_learner_record": (C.c_int, [vp, vp, vp, C.c_int64]),
    "cs_learner_prob": (C.c_int, [vp, C.c_uint64, C.c_uint64, C.POINTER(C.c_double)]),
    "cs_learner_row_total": (C.c_int, [vp, C.c_uint64, C.POINTER(C.c_uint64)]),
    "cs_learner_agents": (C.c_int, [vp, vp, C.c_int]),
    "cs_learner_state_bytes": (C.c_int, [vp, C.POINTER(C.c_uint64)]),
    "cs_learner_rebuild": (C.c_int, [vp, C.c_uint64, C.c_double, C.c_int, vp, C.c_int]),
    "cs_learner_argmax": (C.c_int, [vp, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_double),
                                    C.POINTER(C.c_int)]),
    "cs_exact_survival_prob": (C.c_int, [vp, C.c_uint64, C.c_int, C.c_uint64, C.POINTER(C.c_double)]),
    "cs_chain_hash": (C.c_int, [vp, vp, vp, vp, C.c_int, vp]),
    "cs_engine_create_from_turns": (C.c_int, [C.POINTER(EngineCfg), C.POINTER(WorkloadSpec), vp, C.c_int64,
                                              C.POINTER(vp)]),
    "cs_engine_turn_arrivals": (C.c_int, [vp, vp, C.c_int64]),
    "cs_engine_record_events": (C.c_int, [vp, C.c_int]),
    "cs_engine_write_outputs": (C.c_int, [vp, C.c_char_p, C.c_char_p, C.c_char_p, C.c_uint64, vp, C.c_int, C.c_int]),
    "cs_derive_agent_identity": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_int, vp]),
    "cs_last_error": (C.c_char_p, []),
    "cs_debug_trap_word": (C.c_uint64, []),
    "cs_version": (C.c_char_p, []),
}

_lib = None


class CacheSageError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def lib():
    """The loaded library; raises (no fallback) when it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a). "
                              "There is no CPU fallback.")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc):
    if rc < 0:
        msg = lib().cs_last_error().decode()
        if rc == CS_ERR_INVALID_ARGUMENT:
            raise ValueError(msg)
        if rc == CS_ERR_LOGIC:
            raise AssertionError(msg)
        raise CacheSageError(rc, msg)
    return rc
