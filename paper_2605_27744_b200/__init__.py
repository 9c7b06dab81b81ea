"""cachesage_b200: the CacheSage per-step cache-policy hot path (arXiv 2605.27744), B200-native.

The block pool, block table, transition learner, reachability classes, survival scoring and the
k-victim select run as sm_100a kernels behind the C ABI in include/cachesage_b200.h; this
package is the Python mirror of the reference's API over that ABI. No CPU fallback.
"""
from . import workloads
from ._lib import CacheSageError, lib
from .api import (Engine, Pool, TransitionLearner, block_keys_for, chain_hash, derive_agent_identity,
                  derive_agent_identity_of_prompt, exact_survival_prob, generate_trace_rows, hash_prompts, run_sim_spec)
from .trace import Trace, generate_trace, read_trace_jsonl, run_sim
from .workloads import preset_by_name, preset_names, preset_workloads

__all__ = [
    "CacheSageError", "Engine", "Pool", "TransitionLearner", "block_keys_for", "chain_hash", "derive_agent_identity",
    "derive_agent_identity_of_prompt", "exact_survival_prob", "Trace", "read_trace_jsonl", "generate_trace_rows",
    "run_sim_spec",
    "generate_trace", "hash_prompts", "lib", "preset_by_name", "preset_names", "preset_workloads", "run_sim",
    "workloads",
]
