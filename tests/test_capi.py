"""The drop-in boundary without a GPU: the C-ABI library loads, exports every entry point
include/cachesage_b200.h declares, its structs have the layout the Python binding assumes,
host-only entry points (generator, block-offset planning, defaults) give the reference's
answers, and every device entry point fails loudly (CS_ERR_CUDA) instead of falling back to
the CPU.
"""
import ctypes as C
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest

from paper_2605_27744_b200 import _lib
from paper_2605_27744_b200 import api
from conftest import HAS_GPU

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cachesage_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    src = re.sub(r"//[^\n]*", "", src)
    names = set(re.findall(r"\b(cs_[a-z0-9_]+)\s*\(", src))
    return sorted(names)


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("cs_pool_create", "cs_hash_prompts", "cs_lookup", "cs_observe_dispatch", "cs_admit_pinned",
                 "cs_unpin_slots", "cs_score_snapshot", "cs_hops", "cs_poll_actions", "cs_engine_run"):
        assert must in names
    assert len(names) >= 30


def test_library_exports_every_declared_symbol():
    L = C.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(L, n)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    # every declared entry point has a ctypes signature (so none is called with default int args)
    assert set(declared_functions()) <= set(_lib.SIGNATURES)


def test_library_is_sm100a_and_not_the_oracle():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
    syms = subprocess.run(["nm", "-D", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "cso_" not in syms and "ref_" not in syms.replace("pref_", "")  # no oracle/reference linked in
    deps = subprocess.run(["ldd", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "cs_oracle" not in deps and "cachesage_ref" not in deps


STRUCT_PROBE = r"""
#include <stdio.h>
#include <stddef.h>
#include "cachesage_b200.h"
#define P(T, f) printf(#T "." #f " %zu\n", offsetof(T, f));
int main(void) {
  printf("cs_pool_cfg %zu\ncs_pool_stats %zu\ncs_workload_spec %zu\ncs_engine_cfg %zu\ncs_engine_result %zu\n",
         sizeof(cs_pool_cfg), sizeof(cs_pool_stats), sizeof(cs_workload_spec), sizeof(cs_engine_cfg),
         sizeof(cs_engine_result));
  P(cs_pool_cfg, grid_ctas) P(cs_pool_cfg, min_row_count) P(cs_pool_stats, phase_ns)
  P(cs_workload_spec, seed) P(cs_workload_spec, start_dist) P(cs_engine_cfg, host_inputs)
  return 0;
}
"""


def test_struct_layout_matches_binding():
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "probe.c")
        open(c, "w").write(STRUCT_PROBE)
        exe = os.path.join(d, "probe")
        subprocess.run(["gcc", "-std=c99", "-I", os.path.dirname(HEADER), c, "-o", exe], check=True)
        lines = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split("\n")
    got = dict(l.rsplit(" ", 1) for l in lines if l)
    assert int(got["cs_pool_cfg"]) == C.sizeof(_lib.PoolCfg)
    assert int(got["cs_pool_stats"]) == C.sizeof(_lib.PoolStats)
    assert int(got["cs_workload_spec"]) == C.sizeof(_lib.WorkloadSpec)
    assert int(got["cs_engine_cfg"]) == C.sizeof(_lib.EngineCfg)
    assert int(got["cs_engine_result"]) == C.sizeof(_lib.EngineResult)
    assert int(got["cs_pool_cfg.grid_ctas"]) == _lib.PoolCfg.grid_ctas.offset
    assert int(got["cs_pool_cfg.min_row_count"]) == _lib.PoolCfg.min_row_count.offset
    assert int(got["cs_pool_stats.phase_ns"]) == _lib.PoolStats.phase_ns.offset
    assert int(got["cs_workload_spec.seed"]) == _lib.WorkloadSpec.seed.offset
    assert int(got["cs_workload_spec.start_dist"]) == _lib.WorkloadSpec.start_dist.offset
    assert int(got["cs_engine_cfg.host_inputs"]) == _lib.EngineCfg.host_inputs.offset


def test_defaults_are_the_reference_defaults():
    # CacheSageConfig (cachesage_policy.hpp:16-26), EngineConfig (engine.hpp:28-36)
    c = _lib.PoolCfg()
    _lib.lib().cs_pool_cfg_default(C.byref(c))
    assert (c.e_max, c.tau, c.w_pred, c.window, c.min_confidence, c.min_row_count, c.budget_per_step) == \
        (8, 0.01, 1.0, 1024, 0.5, 5, 1)
    assert c.policy == 1
    e = _lib.EngineCfg()
    _lib.lib().cs_engine_cfg_default(C.byref(e))
    assert (e.block_size, e.prefetch, e.skip, e.take) == (16, 1, 4, 4)


def test_version_string():
    v = _lib.lib().cs_version().decode()
    assert "sm_100a" in v or v


def test_blocks_for_plans_ceil_splits():
    off = np.array([0, 1, 16, 17, 17, 50], np.int64)  # prompts of 1, 15, 1, 0, 33 tokens
    blk = np.zeros(off.size, np.int64)
    n = _lib.lib().cs_blocks_for(off.ctypes.data_as(C.c_void_p), off.size - 1, 16, blk.ctypes.data_as(C.c_void_p))
    assert n == 1 + 1 + 1 + 0 + 3
    assert blk.tolist() == [0, 1, 2, 3, 3, 6]


def test_generator_matches_reference_golden():
    import json
    gens = json.load(open(os.path.join(ROOT, "tests", "golden", "generator.json")))
    import refshim
    for g in gens:
        t = api.generate_trace_rows(g["spec"])
        assert t.shape[0] == g["n"], g["name"]
        assert hex(refshim.fnv1a64(t.astype(np.uint64).reshape(-1))) == g["fnv"], g["name"]


def test_generator_rejects_bad_specs():
    from paper_2605_27744_b200.workloads import preset_by_name
    s = dict(preset_by_name("supervisor-a"))
    s["turns_min"], s["turns_max"] = 5, 2
    with pytest.raises(ValueError):
        api.generate_trace_rows(s)
    s = dict(preset_by_name("supervisor-a"))
    s["transition"] = [[0.0] * len(s["anchor_tokens"])] * len(s["anchor_tokens"])
    with pytest.raises(ValueError):
        api.generate_trace_rows(s)


def test_null_arguments_are_rejected():
    L = _lib.lib()
    assert L.cs_pool_create(None, None) == _lib.CS_ERR_INVALID_ARGUMENT
    assert L.cs_pool_destroy(None) in (_lib.CS_OK, _lib.CS_ERR_INVALID_ARGUMENT)
    assert L.cs_engine_create(None, None, None) == _lib.CS_ERR_INVALID_ARGUMENT
    assert L.cs_last_error()


@pytest.mark.skipif(HAS_GPU, reason="checks the no-device behaviour")
def test_no_device_fails_loudly():
    with pytest.raises(_lib.CacheSageError) as ei:
        api.Pool(1024)
    assert ei.value.code == _lib.CS_ERR_CUDA
    with pytest.raises(_lib.CacheSageError):
        api.hash_prompts([[1, 2, 3]])
    from paper_2605_27744_b200.workloads import preset_by_name
    with pytest.raises(_lib.CacheSageError):
        api.run_sim_spec(preset_by_name("supervisor-a"))
