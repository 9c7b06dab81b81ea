"""The Python restatement of the reference TransitionLearner, rebuild_reachability and
exact_survival_prob (oracle/pyoracle.py) pinned against the UNMODIFIED reference compiled in
place (oracle/_ref via tests/refshim.py): bit-exact probabilities, totals, hops, argmax and
survival probabilities on seeded random transition streams (CPU)."""
import numpy as np
import pytest

import refshim
from oracle import pyoracle as O

pytestmark = pytest.mark.skipif(not refshim.available(), reason="oracle/_ref not built")


def stream(seed, A, n):
    rng = np.random.default_rng(seed)
    ids = rng.integers(1, 2**63, size=A, dtype=np.uint64)
    # a sparse random chain: each agent has a few likely successors
    succ = {i: rng.choice(A, size=min(A, 3), replace=False) for i in range(A)}
    a, b = [], []
    cur = int(rng.integers(A))
    for _ in range(n):
        nxt = int(rng.choice(succ[cur])) if rng.random() < 0.9 else int(rng.integers(A))
        a.append(int(ids[cur]))
        b.append(int(ids[nxt]))
        cur = nxt
    return a, b, [int(x) for x in ids]


@pytest.mark.parametrize("A,n,window", [(3, 50, 1024), (8, 400, 16), (20, 3000, 1024), (64, 5000, 256)])
def test_learner_matches_reference(A, n, window):
    a, b, ids = stream(A * 7 + n, A, n)
    cur = a[-1]
    ref = refshim.learner_eval(a, b, window=window, current=cur, tau=0.05, e_max=8, k=12)
    L = O.Learner(window)
    for x, y in zip(a, b):
        L.record(x, y)
    assert L.alphabet == ref["agents"]
    for i, x in enumerate(L.alphabet):
        assert L.row_total(x) == int(ref["totals"][i])
        assert L.argmax_row(x) == ref["argmax"][i]
        for j, y in enumerate(L.alphabet):
            assert L.prob(x, y) == ref["prob"][i, j]
    assert L.state_bytes() == ref["state_bytes"]
    hops = O.rebuild_reachability(L, cur, 0.05, 8)
    assert [hops[x] for x in L.alphabet] == list(ref["hops"])
    surv = [O.exact_survival_prob(x, 12, L, cur) for x in L.alphabet]
    assert surv == list(ref["surv"])  # bit-exact: same operation order


def test_survival_edge_cases():
    L = O.Learner(8)
    L.record(1, 2)
    assert O.exact_survival_prob(5, 3, L, 5) == 1.0  # target == current
    assert O.exact_survival_prob(9, 3, L, 1) == 0.0  # unknown agent
    with pytest.raises(ValueError):
        O.exact_survival_prob(2, 33, L, 1)
    with pytest.raises(ValueError):
        O.exact_survival_prob(2, -1, L, 1)
