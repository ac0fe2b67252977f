"""Pins of the NEXT-4 oracle (oracle/bbref.c): the exact Eq. 3 optimum by plain
enumeration, against an independent exhaustive search over all D^B dispatches
(tests/bruteforce.py), the Eq. 2 value of the returned assignment, and the heuristics it bounds."""
import numpy as np

import oracle
import workload as w
from tests import bruteforce as bf


def test_equals_exhaustive_and_assignment_achieves_it():
    rng = np.random.default_rng(11)
    for _ in range(60):
        B, D = int(rng.integers(1, 8)), int(rng.integers(1, 4))
        W = w.random_small_instance(rng, B, D)
        s, _, cst, _ = oracle.cost_table(W.lengths[0], W.schemes, W.k_pad)
        row = [int(k) for k in W.cand[0, : W.cand_np[0]]]
        ok, v, pipe, nodes = oracle.eq3_exact(s, cst, W.schemes, row)
        assert ok and v == bf.eq3_opt([int(x) for x in s], W.schemes, row)
        groups = [[int(s[i]) for i in range(B) if pipe[i] == j] for j in range(D)]
        assert all(l <= int(W.schemes[row[j]]["max_len"]) for j, g in enumerate(groups) for l in g)
        assert v == max(bf.lower_bound(g, W.schemes[row[j]]) for j, g in enumerate(groups))


def test_bounds_the_heuristics_and_node_limit():
    W = w.make_workload(4, n_cand=24, n_iter=2)
    for t in range(2):
        L = W.lengths[t][:11]
        s, _, cst, _ = oracle.cost_table(L, W.schemes, W.k_pad)
        for c in range(8):
            row = [int(k) for k in W.cand[c, : W.cand_np[c]]][:4]
            row_ok = int(W.schemes[row[0]]["max_len"]) >= int(s[0])
            ok, v, pipe, nodes = oracle.eq3_exact(s, cst, W.schemes, row)
            if not row_ok:
                assert not ok and v == 2**64 - 1
                continue
            assert ok
            feas, _, lb = oracle.dispatch(s, cst, W.schemes, row)  # HYD-H1's Eq. 3 value
            assert feas and v <= lb
            okA, _, lbA, _ = oracle.alg1_dispatch(s, cst, W.schemes, row, 3, t, 16)  # Alg. 1
            assert okA and v <= lbA
            ok2, v2, _, n2 = oracle.eq3_exact(s, cst, W.schemes, row, node_limit=3)
            assert not ok2 and n2 > 3 and v2 >= v  # budget exhausted: not proved


def first_feasible_above(lengths, scheme, lo, hi):
    for v in range(hi + 1, len(lengths) + 1):
        r = bf.pack_opt(lengths, scheme, [v])
        if r is not None:
            return r
    return None


def test_eq1_equals_exhaustive_partitions_and_bounds_lpt():
    """Eq. 1 exact (oracle/bbref.c) against the set-partition enumeration of tests/bruteforce.py
    over App. D's range (first feasible V above it when none is, reading 5); LPT never beats it."""
    rng = np.random.default_rng(21)
    n = 0
    for _ in range(150):
        W = w.random_small_instance(rng, int(rng.integers(1, 9)), 1)
        k = int(W.cand[0, 0])
        sch = W.schemes[k:k + 1]
        s, _, cst, _ = oracle.cost_table(W.lengths[0], W.schemes, W.k_pad)
        L = [int(x) for x in s]
        ok, V, obj, nodes = oracle.eq1_exact(s, cst[:, k], sch)
        lo, hi = bf.v_range(L, sch)
        ref = bf.pack_opt(L, sch, range(lo, hi + 1))
        if ref is None:
            ref = first_feasible_above(L, sch, lo, hi)
        assert ok and obj == ref
        hv, hp, _, _ = oracle.pack_pipeline(s, cst[:, k], sch)
        assert hp >= obj  # the LPT heuristic (HYD-H1) never beats the optimum
        n += 1
    assert n == 150
