"""GPU parity of NEXT-4 (include/hyd.h hyd_eq3_exact): the exact Eq. 3 optimum per (c, t)
equals the oracle's (unique); the GPU's assignment is valid and achieves it (optimal
assignments may differ on ties); it never exceeds the HYD-H1 or Alg. 1 values."""
import numpy as np
import pytest

import workload as w

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import oracle
    from paper_2412_07894_b200 import assign, hyd

    oracle.build()
    hyd.lib()
    return dict(torch=torch, oracle=oracle, assign=assign, hyd=hyd)


def small_workload(B, D, n_cand, n_iter, seed):
    """Config 4's schemes; candidates cut to their first D pipelines; B-sequence iterations."""
    base = w.make_workload(4, n_cand=n_cand, n_iter=1)
    rng = np.random.default_rng(seed)
    L = w.lengths_lognormal(rng, n_iter * B, hi=32768).reshape(n_iter, B)
    cand = base.cand.copy()
    cnp = np.minimum(base.cand_np, D).astype(np.uint8)
    for c in range(n_cand):
        cand[c, cnp[c]:] = 0xFF
    return w.Workload(0, "bb", L, base.schemes, cand, cnp, base.k_pad)


@pytest.mark.parametrize("B,D", [(6, 3), (10, 4), (12, 3)])
def test_eq3_exact_parity(env, B, D):
    O, assign = env["oracle"], env["assign"]
    W = small_workload(B, D, 40, 3, B * 10 + D)
    A = assign.Assigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad)
    pc = np.repeat(np.arange(W.n_cand), W.n_iter)
    pt = np.tile(np.arange(W.n_iter), W.n_cand)
    val, pipe, nodes, proved = A.eq3_exact(assign.lengths_to_device(W.lengths), pc, pt)
    from tests import bruteforce as bf

    for q, (c, t) in enumerate(zip(pc, pt)):
        s, _, cst, _ = O.cost_table(W.lengths[t], W.schemes, W.k_pad)
        row = [int(k) for k in W.cand[c, : W.cand_np[c]]]
        ok, v, _, _ = O.eq3_exact(s, cst, W.schemes, row)
        assert proved[q] == ok and int(val[q]) == v, (c, t)
        if not ok:
            continue
        groups = [[int(s[i]) for i in range(B) if pipe[q, i] == j] for j in range(len(row))]
        assert all(l <= int(W.schemes[row[j]]["max_len"]) for j, g in enumerate(groups) for l in g)
        assert v == max(bf.lower_bound(g, W.schemes[row[j]]) for j, g in enumerate(groups))
        feas, _, lb = O.dispatch(s, cst, W.schemes, row)
        assert v <= lb


def test_eq3_exact_at_scale_runs(env):
    """Config-4 candidates (8 pipelines) on 20-sequence iterations: 4096 instances."""
    assign = env["assign"]
    W = small_workload(20, 8, 512, 8, 7)
    A = assign.Assigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad)
    pc = np.repeat(np.arange(W.n_cand), W.n_iter)
    pt = np.tile(np.arange(W.n_iter), W.n_cand)
    val, pipe, nodes, proved = A.eq3_exact(assign.lengths_to_device(W.lengths), pc, pt, node_limit=1 << 22)
    A.run(assign.lengths_to_device(W.lengths))
    lb = A.numpy()["lb"]
    feas = val != np.uint64(2**64 - 1)
    assert proved[feas].mean() > 0.9
    assert (val[feas] <= lb[pc[feas], pt[feas]]).all()


@pytest.mark.parametrize("B,D", [(10, 2), (16, 4)])
def test_eq1_exact_parity(env, B, D):
    """Exact Eq. 1 per pipeline of the GPU's own dispatch equals the oracle's (unique optimum);
    never above the heuristic's ptime."""
    O, assign = env["oracle"], env["assign"]
    W = small_workload(B, D, 30, 2, 100 + B)
    A = assign.Assigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad, fused=False)  # reads members
    A.run(assign.lengths_to_device(W.lengths))
    g = A.numpy()
    pc, pt, pj = [], [], []
    for c in range(W.n_cand):
        for t in range(W.n_iter):
            if g["makespan"][t, c] == np.uint64(2**64 - 1):
                continue
            for j in range(int(W.cand_np[c])):
                pc.append(c), pt.append(t), pj.append(j)
    v, obj, nodes, proved = A.eq1_exact(pc, pt, pj)
    for q, (c, t, j) in enumerate(zip(pc, pt, pj)):
        s, _, cst, _ = O.cost_table(W.lengths[t], W.schemes, W.k_pad)
        k = int(W.cand[c, j])
        idx = np.nonzero(g["pipe"][c, t] == j)[0]
        ok, V, o, _ = O.eq1_exact(s[idx], cst[idx, k], W.schemes[k:k + 1])
        if idx.size == 0:
            assert proved[q] and v[q] == 0
            continue
        assert proved[q] == ok and int(obj[q]) == o and int(v[q]) == V, (c, t, j)
        assert o <= int(g["ptime"][c, t, j])
