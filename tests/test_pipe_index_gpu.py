"""GPU parity of the stage-1 -> stage-2 interface for an ARBITRARY stage-1 result (include/hyd.h
hyd_pipe_index, then hyd_pack): any assignment pipe -- random feasible rows, the oracle's
paper-faithful Alg. 1 rows, HYD-H1's own rows -- is indexed and packed on the GPU and
compared element by element with the oracle's packing of the same rows (``oracle.pack_pair``:
Eq. 1 per pipeline).  Rows that are not assignments (an entry naming no pipeline of
the candidate, a pipeline that cannot hold the sequence, a partial 0xFF row) must raise
HYD_F_BAD_PIPE and come out as infeasible pairs."""
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


def random_assignment(rng, sorted_len, schemes, cand_row):
    """Each sequence on a uniformly drawn pipeline of J_i (test input generator)."""
    ml = np.array([int(schemes["max_len"][k]) for k in cand_row])
    if int(sorted_len[0]) > ml[0]:
        return np.full(sorted_len.size, 0xFF, np.uint8)
    out = np.empty(sorted_len.size, np.uint8)
    for i, l in enumerate(sorted_len):
        js = np.nonzero(ml >= int(l))[0]
        out[i] = js[rng.integers(0, js.size)]
    return out


def index_and_pack(env, A, pipe_np):
    """hyd_pipe_index + hyd_pack on the assigner's buffers with pipe = pipe_np [C][It][B]."""
    torch, hyd = env["torch"], env["hyd"]
    It, B, K, kp, Cn = A.n_iter, A.batch, A.n_schemes, A.k_pad, A.n_cand
    A.pipe.copy_(torch.from_numpy(np.ascontiguousarray(pipe_np)).to(A.dev))
    A.status.zero_()
    hyd.pipe_index(A.sorted_len, A.cost, It, B, kp, A.schemes, K, A.cand, A.cand_np, Cn, A.max_np, A.pipe, A.lb,
                   A.stats, A.members, A.status)
    hyd.pack(A.sorted_len, A.cost, It, B, kp, A.schemes, K, A.cand, A.cand_np, Cn, A.max_np, A.pipe, A.stats,
             A.members, A.mb, A.v, A.ptime, A.makespan, A.status, A.ws)
    return A.numpy()


def oracle_rows(env, W, pipe_np, s, cst):
    O = env["oracle"]
    out = []
    for c in range(W.n_cand):
        row = [int(k) for k in W.cand[c, : W.cand_np[c]]]
        for t in range(W.n_iter):
            out.append(((c, t), O.pack_pair(s[t], cst[t], W.schemes, row, pipe_np[c, t])))
    return out


def check(g, ref, tag):
    bad_any = False
    for (c, t), (ms, mb, v, pt, lb, ok) in ref:
        assert int(g["makespan"][t, c]) == ms, (tag, c, t)
        assert np.array_equal(g["mb"][c, t], mb), (tag, c, t)
        assert np.array_equal(g["v"][c, t], v), (tag, c, t)
        assert np.array_equal(g["ptime"][c, t], pt), (tag, c, t)
        assert int(g["lb"][c, t]) == lb, (tag, c, t)
        bad_any |= not ok
    assert bool(g["status"] & 32) == bad_any, (tag, g["status"])


@pytest.mark.parametrize("cfg,n_cand,n_iter", [(2, 40, 4), (3, 24, 3), (4, 70, 3)])
def test_pack_random_assignments(env, cfg, n_cand, n_iter):
    W = w.make_workload(cfg, n_cand=n_cand, n_iter=n_iter)
    s, _, cst, _ = env["oracle"].cost_tables(W)
    rng = np.random.default_rng(100 + cfg)
    pipe = np.empty((W.n_cand, W.n_iter, W.batch), np.uint8)
    for c in range(W.n_cand):
        row = [int(k) for k in W.cand[c, : W.cand_np[c]]]
        for t in range(W.n_iter):
            pipe[c, t] = random_assignment(rng, s[t], W.schemes, row)
    A = env["assign"].Assigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad)
    A.run(env["assign"].lengths_to_device(W.lengths))  # sort + cost table (+ a dispatch we overwrite)
    g = index_and_pack(env, A, pipe)
    check(g, oracle_rows(env, W, pipe, s, cst), f"random cfg{cfg}")


def test_pack_oracle_alg1_rows(env):
    """The paper's dispatcher run on the HOST (oracle Alg. 1, T = 8), packed on the GPU."""
    O = env["oracle"]
    W = w.make_workload(4, n_cand=36, n_iter=3)
    s, _, cst, _ = O.cost_tables(W)
    pipe = np.empty((W.n_cand, W.n_iter, W.batch), np.uint8)
    for c in range(W.n_cand):
        row = [int(k) for k in W.cand[c, : W.cand_np[c]]]
        for t in range(W.n_iter):
            ok, p, _lb, _trial = O.alg1_dispatch(s[t], cst[t], W.schemes, row, 77, t, 8)
            pipe[c, t] = p if ok else 0xFF
    A = env["assign"].Assigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad)
    A.run(env["assign"].lengths_to_device(W.lengths))
    g = index_and_pack(env, A, pipe)
    check(g, oracle_rows(env, W, pipe, s, cst), "alg1")


def test_index_of_dispatch_rows_equals_dispatch_index(env):
    """HYD-H1's own rows: hyd_pipe_index rebuilds exactly the stats / members hyd_dispatch emits."""
    torch, hyd = env["torch"], env["hyd"]
    W = w.make_workload(4, n_cand=50, n_iter=4)
    A = env["assign"].Assigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad)
    A.run(env["assign"].lengths_to_device(W.lengths))
    torch.cuda.synchronize()
    st0, mem0, lb0, g0 = A.stats.clone(), A.members.clone(), A.lb.clone(), A.numpy()
    A.status.zero_()
    hyd.pipe_index(A.sorted_len, A.cost, A.n_iter, A.batch, A.k_pad, A.schemes, A.n_schemes, A.cand, A.cand_np,
                   A.n_cand, A.max_np, A.pipe, A.lb, A.stats, A.members, A.status)
    torch.cuda.synchronize()
    assert A.status_bits() == 0
    assert torch.equal(A.lb, lb0)
    feas = g0["makespan"].T != np.uint64(2**64 - 1)  # [C][It]
    st0n, st1n = st0.cpu().numpy(), A.stats.cpu().numpy()  # [C', It', mnp, 24] bytes, iteration-major rows
    m0n, m1n = mem0.cpu().numpy(), A.members.cpu().numpy()
    flat_s0 = st0n.reshape(W.n_iter, W.n_cand, A.max_np, 24)
    flat_s1 = st1n.reshape(W.n_iter, W.n_cand, A.max_np, 24)
    for c in range(W.n_cand):
        npc = int(W.cand_np[c])
        for t in range(W.n_iter):
            if not feas[c, t]:
                continue
            assert np.array_equal(flat_s0[t, c, :npc], flat_s1[t, c, :npc]), (c, t)
            assert np.array_equal(m0n[t, c, :, :npc], m1n[t, c, :, :npc]), (c, t)


def test_bad_rows_are_flagged_infeasible(env):
    O = env["oracle"]
    W = w.make_workload(4, n_cand=12, n_iter=2)
    s, _, cst, _ = O.cost_tables(W)
    rng = np.random.default_rng(5)
    pipe = np.empty((W.n_cand, W.n_iter, W.batch), np.uint8)
    for c in range(W.n_cand):
        row = [int(k) for k in W.cand[c, : W.cand_np[c]]]
        for t in range(W.n_iter):
            pipe[c, t] = random_assignment(rng, s[t], W.schemes, row)
    feas = [(c, t) for c in range(W.n_cand) for t in range(W.n_iter) if pipe[c, t, 0] != 0xFF]
    (c1, t1), (c2, t2), (c3, t3), (c4, t4) = feas[:4]
    pipe[c1, t1, 7] = W.cand_np[c1]  # no such pipeline
    ml = W.schemes["max_len"][W.cand[c2, : W.cand_np[c2]]]
    pipe[c2, t2, 0] = int(np.argmin(ml)) if ml.min() < s[t2][0] else W.cand_np[c2]  # cannot hold l_0
    pipe[c3, t3, W.batch - 1] = 0xFF  # partial row
    pipe[c4, t4, :] = 0xFF  # a feasible pair left unassigned
    A = env["assign"].Assigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad)
    A.run(env["assign"].lengths_to_device(W.lengths))
    g = index_and_pack(env, A, pipe)
    ref = oracle_rows(env, W, pipe, s, cst)
    assert sum(not r[1][5] for r in ref) == 4
    check(g, ref, "bad rows")
    for c, t in ((c1, t1), (c2, t2), (c3, t3), (c4, t4)):
        assert int(g["makespan"][t, c]) == 2**64 - 1


def test_pipe_index_ragged(env):
    """Token-budget batches: random assignments through hyd_pipe_index_ragged + hyd_pack_ragged."""
    torch, hyd, O = env["torch"], env["hyd"], env["oracle"]
    W = w.make_workload(6, n_cand=30, n_iter=4)
    A = env["assign"].Assigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad, offsets=W.offsets)
    A.run(env["assign"].lengths_to_device(W.lengths))
    rng = np.random.default_rng(6)
    off = W.offsets.astype(np.int64)
    pipe = np.empty((W.n_cand, W.n_total), np.uint8)
    tabs = []
    for t in range(W.n_iter):
        s, _, cst, _ = O.cost_table(W.iteration(t), W.schemes, W.k_pad)
        tabs.append((s, cst))
        for c in range(W.n_cand):
            row = [int(k) for k in W.cand[c, : W.cand_np[c]]]
            pipe[c, off[t]:off[t + 1]] = random_assignment(rng, s, W.schemes, row)
    A.pipe.copy_(torch.from_numpy(pipe).to(A.dev))
    A.status.zero_()
    It, B, K, kp, Cn, N = A.n_iter, A.batch, A.n_schemes, A.k_pad, A.n_cand, A.n_total
    hyd.pipe_index_ragged(A.sorted_len, A.cost, It, A.off, N, B, kp, A.schemes, K, A.cand, A.cand_np, Cn, A.max_np,
                          A.pipe, A.lb, A.stats, A.members, A.status)
    hyd.pack_ragged(A.sorted_len, A.cost, It, A.off, N, B, kp, A.schemes, K, A.cand, A.cand_np, Cn, A.max_np, A.pipe,
                    A.stats, A.members, A.mb, A.v, A.ptime, A.makespan, A.status, A.ws)
    g = A.numpy()
    assert g["status"] == 0
    for t in range(W.n_iter):
        s, cst = tabs[t]
        for c in range(W.n_cand):
            row = [int(k) for k in W.cand[c, : W.cand_np[c]]]
            ms, mb, v, pt, lb, ok = O.pack_pair(s, cst, W.schemes, row, pipe[c, off[t]:off[t + 1]])
            assert ok
            assert int(g["makespan"][t, c]) == ms and int(g["lb"][c, t]) == lb, (c, t)
            assert np.array_equal(g["mb"][c, off[t]:off[t + 1]], mb), (c, t)
            assert np.array_equal(g["v"][c, t], v) and np.array_equal(g["ptime"][c, t], pt), (c, t)
