"""CPU pins of the oracle's packing of a GIVEN stage-1 result (``oracle.pack_pair``,
``oracle.eq2_lb``, ``oracle.is_assignment``), the reference for hyd_pipe_index + hyd_pack.

* Hand-worked cases on SURVEY §8(c)'s example (T(l) = l + 100, PP = 2, MaxLen 8192, two
  identical pipelines; Eq. 1, App. D range P:1097, Eq. 2), derivations below.
* Consistency: packing HYD-H1's own rows reproduces the whole-method oracle.
* The assignment definition (J_i; infeasible pairs S:371) on hand-made rows."""
import json
import os

import numpy as np
import pytest

import workload as w

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def O():
    import oracle

    oracle.build()
    return oracle


def _example(O):
    g = json.load(open(os.path.join(GOLDEN, "worked_example.json")))
    sch = w.make_scheme(**g["scheme"])
    s, _, cst, st = O.cost_table(np.array(g["lengths"], np.uint32), sch, 4)
    assert st == 0
    return g, sch, s, cst


def test_hand_worked_mirror(O):
    """pipe = [1,0,0,1,0,1]: the worked example's dispatch with the pipelines swapped (identical
    schemes), so each pipeline's packing is the other's from the golden derivation."""
    g, sch, s, cst = _example(O)
    ms, mb, v, pt, lb, ok = O.pack_pair(s, cst, sch, [0, 0], np.array([1, 0, 0, 1, 0, 1], np.uint8))
    assert ok and ms == 12000
    assert list(v[:2]) == [2, 1] and list(pt[:2]) == [10500, 12000] and not v[2:].any()
    assert list(mb) == [0, 0, 1, 0, 1, 0]
    assert lb == 10100  # Eq. 2 is symmetric in the swap


def test_hand_worked_single_pipeline(O):
    """Everything on pipeline 0: items (4000,3000,2500,1200,800,500), costs
    (4100,3100,2600,1300,900,600), S = 12000 -> V in [ceil(12000/8192) = 2, U = 6].
      V=2: bins 4100 | 3100, 2500->b1 5700, 1200->b0 5400, 800->b0 6300, 500->b1 6300: 6300*3 = 18900
      V=3: 4100 | 3100 | 2600, 1200->b2 3900, 800->b1 4000, 500->b2 4500: 4500*4 = 18000
      V=4: max 4100 -> 20500; V=5: 24600; V=6: 28700  =>  V* = 3, ptime 18000, mb [0,1,2,2,1,2]
    Pipeline 1 is empty (V = 0, ptime 0, reading 12).  Eq. 2: 12600 + 4100 (PP-1) = 16700."""
    g, sch, s, cst = _example(O)
    ms, mb, v, pt, lb, ok = O.pack_pair(s, cst, sch, [0, 0], np.zeros(6, np.uint8))
    assert ok and ms == 18000
    assert list(v[:2]) == [3, 0] and list(pt[:2]) == [18000, 0]
    assert list(mb) == [0, 1, 2, 2, 1, 2]
    assert lb == 16700


def test_is_assignment_definition(O):
    sch = np.concatenate([w.make_scheme(max_len=100, b_q32=1 << 32), w.make_scheme(max_len=50, b_q32=1 << 32)])
    s = np.array([80, 40, 10], np.uint32)
    assert O.is_assignment(s, sch, [0, 1], [0, 1, 1]) == (True, True)
    assert O.is_assignment(s, sch, [0, 1], [1, 1, 1]) == (False, True)  # 80 > MaxLen_1
    assert O.is_assignment(s, sch, [0, 1], [0, 2, 1]) == (False, True)  # no pipeline 2
    assert O.is_assignment(s, sch, [0, 1], [0, 0, 0xFF]) == (False, True)  # partial row
    s2 = np.array([120, 40, 10], np.uint32)  # l_0 > MaxLen_0: infeasible pair
    assert O.is_assignment(s2, sch, [0, 1], [0xFF] * 3) == (True, False)
    assert O.is_assignment(s2, sch, [0, 1], [0xFF, 1, 1]) == (False, False)


def test_pack_pair_reproduces_hyd_h1(O):
    W = w.make_workload(3, n_cand=25, n_iter=2)
    r = O.assign_batch(W)
    s, _, cst, _ = O.cost_tables(W)
    for c in range(W.n_cand):
        row = [int(k) for k in W.cand[c, : W.cand_np[c]]]
        for t in range(W.n_iter):
            ms, mb, v, pt, lb, ok = O.pack_pair(s[t], cst[t], W.schemes, row, r["pipe"][c, t])
            assert ok
            assert ms == int(r["makespan"][t, c]) and lb == int(r["lb"][c, t])
            assert np.array_equal(mb, r["mb"][c, t])
            assert np.array_equal(v, r["v"][c, t]) and np.array_equal(pt, r["ptime"][c, t])
