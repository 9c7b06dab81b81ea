"""The admission server (csrc/cs_admit.cu server_kernel): one persistent cooperative launch serves
every admission of an engine loop through a host-mapped mailbox. It must make exactly the
decisions of one admit_kernel launch per admission (CS_SERVER=0), whatever the segmentation of
the engine loop (the server stops at the end of every engine call and whenever the host needs
the stream), on the device-input and the end-to-end path. Bit-exact: every victim in order,
cached tokens per turn, fp64 completion times, warmups.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

POOL = 1 << 20


def _run(server, host_inputs=False, chunks=(400,), mode="realistic", sessions=4000, by_steps=False):
    import paper_2605_27744_b200 as cb
    from paper_2605_27744_b200 import workloads as W

    old = os.environ.get("CS_SERVER")
    os.environ["CS_SERVER"] = "1" if server else "0"
    try:
        spec = W.cfg4_mixed(sessions=sessions, budget=POOL, seed=2608)
        eng = cb.Engine(spec, policy="cachesage", budget=POOL, host_inputs=host_inputs, agent_capacity=1024,
                        prefetch=True)
    finally:
        if old is None:
            del os.environ["CS_SERVER"]
        else:
            os.environ["CS_SERVER"] = old
    try:
        keys, lt, agents, refs = W.pool_snapshot(POOL, len(eng.agents()), seed=11, mode=mode)
        eng.restore(keys, lt, agents=agents, refs=refs)
        if by_steps:  # one engine call (one server launch and stop) per scheduler step, to the end
            while not eng.step():
                pass
        else:
            for c in chunks:
                eng.run_for(c)
        t = eng.turns()
        ws, wt, wk = eng.warmups()
        out = {"ev": eng.evictions(), "cached": t["cached_tokens"], "end": t["end_us"].view(np.uint64),
               "w": (ws, wt, wk), "res": eng.result(), "ps": eng.pool_stats(), "check": eng.check()}
    finally:
        eng.close()
    return out


def _same(a, b):
    assert a["ev"].size == b["ev"].size and np.array_equal(a["ev"], b["ev"])
    assert np.array_equal(a["cached"], b["cached"])
    assert np.array_equal(a["end"], b["end"])
    for x, y in zip(a["w"], b["w"]):
        assert np.array_equal(x, y)
    assert a["res"]["admissions"] == b["res"]["admissions"]


@pytest.mark.parametrize("mode", ["realistic", "adversarial"])
def test_server_equals_per_admission_launches(mode):
    s = _run(True, mode=mode)
    k = _run(False, mode=mode)
    _same(s, k)
    assert s["ps"]["server_launches"] >= 1 and k["ps"]["server_launches"] == 0
    assert s["res"]["gpu_launches"] < k["res"]["gpu_launches"]
    assert s["check"] == {"pk_mismatch": 0, "resident_delta": 0, "pinned_delta": 0, "table_mismatch": 0}
    assert s["ev"].size > 1000


def test_server_segmentation_does_not_matter():
    """One engine call per scheduler step (a server launch and a stop each) against one call,
    over a whole trace."""
    a = _run(True, sessions=200, by_steps=True)
    b = _run(True, sessions=200, chunks=(10**9,))
    _same(a, b)
    assert a["ps"]["server_launches"] > b["ps"]["server_launches"]
    assert a["ev"].size > 100


def test_server_end_to_end_path():
    """Host inputs: CTA 0 copies each admission's prompt blocks from pinned memory, the victims come
    back through the early status; the same decisions as per-admission launches."""
    s = _run(True, host_inputs=True)
    k = _run(False, host_inputs=True)
    _same(s, k)
    assert s["res"]["h2d_bytes"] == k["res"]["h2d_bytes"] > 0
