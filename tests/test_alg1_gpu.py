"""GPU parity of NEXT-1 (Alg. 1 as stage 1, include/hyd.h hyd_dispatch_alg1) against the CPU
oracle (oracle/alg1ref.c), element by element: trial permutations, the winning trial per
(c,t), pipe, lb (= O_best), and every downstream output (mb, v, ptime, makespan, key)."""
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


def run_gpu(env, W, trials, seed):
    A = env["assign"].Assigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad, trials=trials, seed=seed)
    A.run(env["assign"].lengths_to_device(W.lengths))
    return A, A.numpy()


def compare(g, o, tag):
    for k in ("sorted_len", "perm", "cost", "best_trial", "pipe", "lb", "mb", "v", "ptime", "makespan", "key"):
        a, b = g[k], o[k]
        assert a.shape == b.shape, (tag, k, a.shape, b.shape)
        if not np.array_equal(a, b):
            bad = np.argwhere(a != b)
            raise AssertionError(f"{tag} {k}: {len(bad)} mismatches, first at {bad[:5].tolist()}: "
                                 f"gpu={a[tuple(bad[0])]} oracle={b[tuple(bad[0])]}")
    feas = g["best_trial"] >= 0
    assert np.array_equal(g["best_obj"][feas], g["lb"][feas])
    assert g["status"] == o["status"], (tag, g["status"], o["status"])


@pytest.mark.parametrize("B,trials", [(1, 3), (8, 1), (37, 5), (512, 13), (1000, 9)])
def test_permutations_match_oracle(env, B, trials):
    torch, hyd, O = env["torch"], env["hyd"], env["oracle"]
    It, seed = 3, 0x1234_5678_9ABC
    order = torch.empty((It, trials, B), dtype=torch.int16, device="cuda")
    hyd.alg1_permutations(seed, It, B, trials, order)
    g = order.cpu().numpy().view(np.uint16)
    for t in range(It):
        for tr in range(trials):
            assert np.array_equal(g[t, tr].astype(np.uint32), O.alg1_permutation(seed, t, tr, B)), (t, tr)


# (cfg, n_cand, n_iter, trials): CTA tiles over candidates (32) and trials (8) with ragged tails
CASES = [
    (2, 64, 3, 8),
    (2, 37, 2, 13),
    (3, 70, 2, 10),
    (4, 45, 2, 17),
    (4, 96, 1, 100),
    (1, 1, 40, 4),
]


@pytest.mark.parametrize("cfg,n_cand,n_iter,trials", CASES)
def test_alg1_parity_reduced(env, cfg, n_cand, n_iter, trials):
    W = w.make_workload(cfg, n_cand=n_cand, n_iter=n_iter)
    seed = 1000 + cfg
    _, g = run_gpu(env, W, trials, seed)
    o = env["oracle"].assign_batch(W, n_threads=0, trials=trials, seed=seed)
    compare(g, o, f"alg1-cfg{cfg}")


def test_alg1_parity_cfg5_prefix(env):
    """16 pipelines, lengths to 256K, a 1000-sequence prefix (B % 8 != 0: unstaged path)."""
    W = w.make_workload(5, n_cand=10, n_iter=1)
    W.lengths = np.ascontiguousarray(W.lengths[:, :1000])
    _, g = run_gpu(env, W, 3, 5)
    o = env["oracle"].assign_batch(W, n_threads=0, trials=3, seed=5)
    compare(g, o, "alg1-cfg5")


def test_alg1_parity_edges(env):
    rng = np.random.default_rng(21)
    sch = w.make_workload(4, n_cand=40, n_iter=1)
    L = w.lengths_lognormal(rng, 4 * 96, hi=32768).reshape(4, 96)
    L[1, 5] = 120000  # infeasible candidates
    L[2, 7] = 2**24  # all-infeasible iteration
    W = w.Workload(0, "edge", L, sch.schemes, sch.cand, sch.cand_np, sch.k_pad)
    _, g = run_gpu(env, W, 6, 77)
    o = env["oracle"].assign_batch(W, n_threads=0, trials=6, seed=77)
    compare(g, o, "alg1-infeasible")
    for s in range(3):
        W = w.random_small_instance(np.random.default_rng(s), 7, 3)
        _, g = run_gpu(env, W, 20, s)
        o = env["oracle"].assign_batch(W, n_threads=0, trials=20, seed=s)
        compare(g, o, f"alg1-tiny{s}")


def test_alg1_parity_u64_path(env):
    """Loads above the packed-key bound: the 64-bit trial kernel."""
    rng = np.random.default_rng(9)
    sch = np.concatenate([
        w.make_scheme(pp=4, max_len=2**20, util_len=0, a_q32=0, b_q32=(3 << 40), c_q32=0),
        w.make_scheme(pp=1, max_len=2**19, util_len=0, a_q32=0, b_q32=(1 << 41), c_q32=1 << 32),
    ])
    L = rng.integers(1000, 2**18, (2, 600)).astype(np.uint32)
    W = w.custom_workload(L, sch, [[0, 1], [0, 0, 1], [0, 0, 0, 1, 1]])
    _, g = run_gpu(env, W, 11, 3)
    assert int(g["lb"].max()) > 2**32
    o = env["oracle"].assign_batch(W, n_threads=0, trials=11, seed=3)
    compare(g, o, "alg1-u64")


def test_alg1_full_size_sampled(env):
    """cfg4 full size (4096 candidates x 1024 iterations) with T = 4 trials; sampled pairs."""
    torch = env["torch"]
    W = w.make_workload(4)
    A, _ = run_gpu(env, W, 4, 2024)
    O = env["oracle"]
    tables = O.cost_tables(W)
    rng = np.random.default_rng(4)
    pc = rng.integers(0, W.n_cand, 60)
    pt = rng.integers(0, W.n_iter, 60)
    o = O.assign_pairs(W, pc, pt, tables=tables, trials=4, seed=2024)
    u = lambda x, dt: x.cpu().numpy().view(dt)
    ic, it = torch.from_numpy(pc).cuda(), torch.from_numpy(pt).cuda()
    assert np.array_equal(u(A.pipe[ic, it], np.uint8), o["pipe"])
    assert np.array_equal(u(A.lb[ic, it], np.uint64), o["lb"])
    assert np.array_equal(u(A.mb[ic, it], np.uint16), o["mb"])
    assert np.array_equal(u(A.ptime[ic, it], np.uint64), o["ptime"])
    assert np.array_equal(u(A.makespan[it, ic], np.uint64), o["makespan"])
    bt = u(A.best[ic, it], np.uint64)
    assert np.array_equal(np.where(bt == np.uint64(2**64 - 1), -1, (bt & np.uint64(0xFF)).astype(np.int64)),
                          o["best_trial"])
    assert A.status_bits() == tables[3]
