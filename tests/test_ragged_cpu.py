"""NEXT-2 host side: the token-budget sampler and the ragged
oracle, which is by definition the uniform method applied to each iteration separately."""
import numpy as np

import oracle
import workload as w


def test_sampler_spec_example():
    # sample [50000], budget 100000, context 32768 -> four truncated draws
    L, off = w.sample_minibatches(np.random.default_rng(1), [50000], 3, 100000, 32768)
    assert off.tolist() == [0, 4, 8, 12] and (L == 32768).all()


def test_sampler_budget_one_is_one_sequence():
    L, off = w.sample_minibatches(np.random.default_rng(2), [5, 9, 100], 7, 1, 32768)
    assert np.diff(off).tolist() == [1] * 7


def test_sampler_invariants():
    rng = np.random.default_rng(3)
    corpus = np.maximum(np.floor(rng.lognormal(6.9, 1.2, 20000)), 1)
    budget, ctx = 100000, 32768
    L, off = w.sample_minibatches(np.random.default_rng(4), corpus, 300, budget, ctx)
    assert off[0] == 0 and off[-1] == L.size and (np.diff(off.astype(np.int64)) >= 1).all()
    assert L.max() <= ctx and L.min() >= 1
    for t in range(300):
        s = int(L[off[t]:off[t + 1]].astype(np.int64).sum())
        assert budget <= s < budget + ctx  # budget bracketing
        assert int(L[off[t]:off[t + 1] - 1].astype(np.int64).sum()) < budget  # stops at the first draw reaching it
    L2, off2 = w.sample_minibatches(np.random.default_rng(4), corpus, 300, budget, ctx)
    assert np.array_equal(L, L2) and np.array_equal(off, off2)  # determinism


def test_cfg6_shape():
    W = w.make_workload(6, n_cand=8, n_iter=64)
    assert W.ragged and W.n_iter == 64 and W.n_total == int(W.offsets[-1]) == W.lengths.size
    b = np.diff(W.offsets.astype(np.int64))
    assert 20 < b.mean() < 120 and W.batch == b.max()
    Wp = w.make_workload(6, n_cand=8, n_iter=16)  # iteration prefix
    assert np.array_equal(Wp.offsets, W.offsets[:17]) and np.array_equal(Wp.lengths, W.lengths[: Wp.n_total])


def test_ragged_oracle_equals_uniform_on_uniform_offsets():
    W = w.make_workload(2, n_cand=12, n_iter=3)
    u = oracle.assign_batch(W)
    R = w.Workload(W.cfg, W.name, W.lengths.reshape(-1).copy(), W.schemes, W.cand, W.cand_np, W.k_pad,
                   offsets=np.arange(W.n_iter + 1, dtype=np.uint32) * W.batch)
    r = oracle.assign_batch_ragged(R)
    for k in ("sorted_len", "perm", "cost", "pipe", "mb"):
        assert np.array_equal(r[k].reshape(-1), u[k].reshape(-1)), k
    for k in ("lb", "v", "ptime", "makespan", "key"):
        assert np.array_equal(r[k], u[k]), k
