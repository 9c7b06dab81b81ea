"""The reference-side drop-in (include/cachesage_b200_policy.hpp), compiled against the reference's
own headers (oracle/adapter_check.cpp, `make -C oracle adapter`) and driven by the UNMODIFIED
reference engine:

- B200Policy registered in the reference Runtime runs whole reference cells: the reference
  EngineSim's evict_one consults B200Policy::score per block, and observe / poll_actions /
  predict / serialize_state go to the GPU pool. Hit rate, victims, cached tokens, completion
  times and warmups must equal the reference fixtures (tests/golden/runs.json).
- B200Policy and the reference CacheSagePolicy observe the same event streams: scores, drains,
  forecasts, serialize_state().dump() and state_bytes agree.
- B200BatchEvictor (one device launch per admission) next to the reference EngineSim: the
  same victims admission by admission.
"""
import ctypes as C
import json
import os

import numpy as np
import pytest

import refshim

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(os.path.dirname(HERE), "oracle", "_ref", "libb200_adapter_check.so")
RUNS = json.load(open(os.path.join(HERE, "golden", "runs.json")))["runs"]
STATE = json.load(open(os.path.join(HERE, "golden", "policy_state.json")))
# the CacheSage cells whose reference run finishes in seconds (the per-block score loop is the
# reference's own: O(N) per eviction)
CELLS = [g for g in RUNS if g["kw"]["policy"] == "cachesage" and g["kw"].get("budget", 0) <= 256]

needs_lib = pytest.mark.skipif(not (os.path.exists(LIB) and refshim.available()),
                               reason="oracle/_ref adapter check not built (needs /root/reference at build time)")


def _lib():
    L = C.CDLL(LIB)
    L.adapter_run.argtypes = [C.c_void_p, C.POINTER(refshim.RefRunCfg), C.POINTER(refshim.RefRunOut), C.c_int]
    L.adapter_lockstep.argtypes = [C.c_void_p, C.POINTER(refshim.RefRunCfg), C.c_long, C.c_int, C.c_void_p,
                                   C.c_void_p, C.c_long, C.c_void_p]
    L.adapter_lockstep.restype = C.c_long
    L.adapter_state_after.argtypes = ([C.POINTER(refshim.RefRunCfg), C.c_long] + [C.c_void_p] * 6
                                      + [C.c_int, C.POINTER(C.c_int)])
    L.adapter_last_error.restype = C.c_char_p
    return L


def _fnv(a):
    return hex(refshim.fnv1a64(np.ascontiguousarray(a, dtype="<u8")))


@needs_lib
@pytest.mark.parametrize("g", CELLS, ids=[g["name"] for g in CELLS])
def test_reference_engine_over_b200_policy(g):
    L = _lib()
    s = refshim._spec_struct(g["spec"])
    kw = dict(g["kw"])
    c = refshim.run_cfg(**kw)
    o = refshim.RefRunOut()
    rc = L.adapter_run(C.byref(s), C.byref(c), C.byref(o), 0)
    assert rc == 0, refshim._err()
    try:
        nt, ne, nw = o.n_turns, o.n_evictions, o.n_warmups
        ev = np.ctypeslib.as_array(o.evictions, (max(ne, 1),))[:ne].astype(np.uint64)
        cached = np.ctypeslib.as_array(o.cached_tokens, (max(nt, 1),))[:nt].astype(np.int64)
        end = np.ctypeslib.as_array(o.end_us, (max(nt, 1),))[:nt].copy()
        wt = np.ctypeslib.as_array(o.warmup_target, (max(nw, 1),))[:nw].astype(np.uint64)
        assert repr(o.hit_rate) == g["hit_rate"]
        assert ne == g["evictions"] and _fnv(ev) == g["evictions_fnv"]
        assert _fnv(cached) == g["cached_fnv"]
        assert _fnv(end.view(np.uint64)) == g["end_us_fnv"]
        assert nw == g["n_warmups"] and _fnv(wt) == g["warmups_fnv"]
        assert o.n_steps == g["steps"]
    finally:
        refshim.lib().ref_free_run(C.byref(o))


@needs_lib
@pytest.mark.parametrize("case", [c for c in STATE["cases"] if c["kw"]["policy"] == "cachesage" and "checkpoints" in c],
                         ids=lambda c: c["name"])
def test_b200_policy_tracks_cachesage_policy(case):
    L = _lib()
    ev = case["events"]
    kind = np.array([e["kind"] for e in ev], np.int32)
    tick = np.array([e["tick"] for e in ev], np.uint64)
    agent = np.array([e.get("agent", 0) for e in ev], np.uint64)
    has_prev = np.array([e.get("prev") is not None for e in ev], np.int32)
    prev = np.array([e.get("prev") or 0 for e in ev], np.uint64)
    req = np.array([e.get("request", 0) for e in ev], np.uint64)
    c = refshim.run_cfg(**case["kw"])
    same = C.c_int(0)
    p = refshim._ptr
    rc = L.adapter_state_after(C.byref(c), len(ev), p(kind), p(tick), p(agent), p(has_prev), p(prev), p(req), 0,
                               C.byref(same))
    assert rc == 0, L.adapter_last_error().decode()
    assert same.value == 1


@needs_lib
@pytest.mark.parametrize("name,budget,n_req", [("supervisor-a", 60, 400), ("cfg1", 128, 1500),
                                               ("synthetic-chain", 120, 400)])
def test_batch_evictor_lockstep_with_reference_engine(name, budget, n_req):
    from paper_2605_27744_b200 import workloads as W

    L = _lib()
    spec = W.cfg1(budget) if name == "cfg1" else W.preset_by_name(name)
    s = refshim._spec_struct(spec)
    c = refshim.run_cfg(policy="cachesage", budget=budget)
    nv = np.zeros(n_req, np.int64)
    cached = np.zeros(n_req, np.int64)
    vic = np.zeros(n_req * 64, np.uint64)
    p = refshim._ptr
    done = L.adapter_lockstep(C.byref(s), C.byref(c), n_req, 0, p(nv), p(vic), vic.size, p(cached))
    assert done != -1, L.adapter_last_error().decode()
    assert done >= 0, f"admission {-2 - done}: the B200 victims differ from the reference evict_one loop"
    assert done == n_req and nv.sum() > 0
