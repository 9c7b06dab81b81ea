"""The device TransitionLearner / rebuild_reachability / argmax_row / exact_survival_prob
(cs_learner_*, cs_exact_survival_prob) and the Python-API hashing entry points against the
UNMODIFIED reference (oracle/_ref via tests/refshim.py). The bar is bit-exact: integer counts,
fp64 probabilities and the horizon-k survival probabilities (the north star's tolerance for
survival scores is 1e-6 relative; the device reproduces the reference's operation order, so
the test demands equality and reports the relative error if that ever fails)."""
import numpy as np
import pytest

import refshim
from test_learner_oracle import stream

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not refshim.available(), reason="oracle/_ref not built")]


def _device(a, b, window, batches):
    import paper_2605_27744_b200 as cb

    L = cb.TransitionLearner(window=window)
    i = 0
    for bs in batches:  # single records and device batches (incl. batches larger than the window)
        if i >= len(a):
            break
        if bs == 1:
            L.record(a[i], b[i])
        else:
            L.record_many(a[i:i + bs], b[i:i + bs])
        i += bs
    if i < len(a):
        L.record_many(a[i:], b[i:])
    return L


@pytest.mark.parametrize("A,n,window,batches", [
    (3, 50, 1024, [1] * 50),
    (8, 400, 16, [1, 5, 40, 3, 100]),
    (20, 3000, 1024, [1000, 1, 1, 1500]),
    (64, 5000, 256, [700, 1, 2000, 37]),
])
def test_device_learner_matches_reference(A, n, window, batches):
    import paper_2605_27744_b200 as cb

    a, b, ids = stream(A * 7 + n, A, n)
    cur = a[-1]
    ref = refshim.learner_eval(a, b, window=window, current=cur, tau=0.05, e_max=8, k=12)
    L = _device(a, b, window, batches)
    try:
        assert L.agents() == ref["agents"]
        for i, x in enumerate(ref["agents"]):
            assert L.row_total(x) == int(ref["totals"][i])
            assert L.argmax_row(x) == ref["argmax"][i]
            for j, y in enumerate(ref["agents"]):
                assert L.prob(x, y) == ref["prob"][i, j]
        assert L.state_bytes() == ref["state_bytes"]
        hops = L.rebuild_reachability(cur, tau=0.05, e_max=8)
        assert [hops[x] for x in ref["agents"]] == list(ref["hops"])
        for i, x in enumerate(ref["agents"]):
            got = cb.exact_survival_prob(x, 12, L, cur)
            want = float(ref["surv"][i])
            rel = abs(got - want) / max(abs(want), 1e-300)
            assert got == want, f"survival {got!r} vs {want!r} (rel {rel:.3g}, tolerance 1e-6)"
    finally:
        L.close()


@pytest.mark.parametrize("k", [0, 1, 5, 32])
def test_device_survival_horizons(k):
    import paper_2605_27744_b200 as cb

    a, b, ids = stream(99 + k, 10, 800)
    ref = refshim.learner_eval(a, b, window=1024, current=a[0], k=k)
    L = _device(a, b, 1024, [800])
    try:
        assert [cb.exact_survival_prob(x, k, L, a[0]) for x in ref["agents"]] == list(ref["surv"])
    finally:
        L.close()


def test_device_survival_errors_and_edges():
    import paper_2605_27744_b200 as cb

    L = cb.TransitionLearner(window=8)
    try:
        L.record(1, 2)
        assert cb.exact_survival_prob(7, 3, L, 7) == 1.0
        assert cb.exact_survival_prob(9, 3, L, 1) == 0.0
        for k in (33, -1):
            with pytest.raises(ValueError):
                cb.exact_survival_prob(2, k, L, 1)
        assert L.argmax_row(2) is None and L.row_total(2) == 0
        big = cb.TransitionLearner(window=4096)
        big.record_many(list(range(1, 70)), list(range(2, 71)))
        with pytest.raises(ValueError):  # alphabet > 64 (survival_oracle.cpp:12-14)
            cb.exact_survival_prob(3, 2, big, 1)
        big.close()
    finally:
        L.close()


def test_python_api_hashing_matches_reference():
    import paper_2605_27744_b200 as cb

    rng = np.random.default_rng(5)
    for _ in range(20):
        toks = rng.integers(0, 2**32, size=int(rng.integers(1, 40)), dtype=np.uint64).astype(np.uint32).tolist()
        parent = None if rng.random() < 0.3 else int(rng.integers(0, 2**63))
        assert cb.chain_hash(parent, toks) == refshim.chain_hash(parent, toks)
        keys = rng.integers(0, 2**63, size=int(rng.integers(0, 12)), dtype=np.uint64).tolist()
        for skip, take in ((4, 4), (0, 1), (2, 6)):
            assert cb.derive_agent_identity(keys, skip, take) == refshim.identity(keys, skip, take)
    assert cb.chain_hash(0x1234, [5]) == 0xCAFB0C62E76313A8
    with pytest.raises(ValueError):
        cb.chain_hash(None, [])
