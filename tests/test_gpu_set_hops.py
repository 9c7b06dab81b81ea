"""cs_set_hops: reachability hops computed outside the pool (cs_learner_rebuild, or
an external learner) drive the survival classes the pool scores with: score = w_pred * (1 -
min(hop, e_max) / e_max) + rho (cachesage_policy.cpp:79-85, reachability.cpp:12-20)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_set_hops_drives_scores():
    from paper_2605_27744_b200 import api

    p = api.Pool(64, policy="cachesage", e_max=8, w_pred=1.0)
    try:
        p.register_agents([11, 22, 33])
        keys = np.arange(1, 6, dtype=np.uint64)
        lt = np.array([10, 20, 30, 40, 50], np.uint64)
        agents = np.array([0, 1, 2, 0xFFFFFFFF, 0], np.uint32)
        p.restore(keys, lt, agents=agents)
        p.set_hops([0, 3, 200])
        assert p.hops(3).tolist() == [0, 3, 200]
        k, s = p.score_snapshot(100)
        got = dict(zip(k.tolist(), s.tolist()))
        old, now = 10.0, 100.0
        surv = {0: 1.0, 1: 1.0 - 3.0 / 8.0, 2: 0.0, 0xFFFFFFFF: 0.0}
        for key, t, a in zip(keys.tolist(), lt.tolist(), agents.tolist()):
            rho = (float(t) - old) / (now - old)
            assert got[key] == 1.0 * surv[a] + rho, (key, got[key])
    finally:
        p.close()


def test_set_hops_from_the_standalone_learner():
    """The learner's rebuild (cs_learner_rebuild) feeds the pool: same classes as the pool's own
    observe would build from the same dispatch stream."""
    from paper_2605_27744_b200 import api

    ids = [101, 202, 303, 404]
    L = api.TransitionLearner(window=1024)
    pool_a = api.Pool(64, policy="cachesage", e_max=4)
    pool_b = api.Pool(64, policy="cachesage", e_max=4)
    try:
        pool_a.register_agents(ids)
        pool_b.register_agents(ids)
        seq = [0, 1, 2, 1, 3, 0, 2, 3, 1]
        for i in range(1, len(seq)):
            L.record(ids[seq[i - 1]], ids[seq[i]])
        for i, a in enumerate(seq):  # the pool's own observe(AgentDispatch) chain
            pool_b.observe_dispatch(seq[i - 1] if i else None, a, i + 1)
        hops = L.rebuild_reachability(ids[seq[-1]], tau=0.01, e_max=4)
        pool_a.set_hops([hops[ids[j]] for j in range(4)])
        assert pool_a.hops(4).tolist() == pool_b.hops(4).tolist()
    finally:
        pool_a.close()
        pool_b.close()
        L.close()
