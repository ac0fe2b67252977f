"""GPU parity of the fused small-batch kernel (include/hyd.h hyd_dispatch_pack: a3 + a4 in one
kernel for batches of at most 128 sequences) against the CPU oracle, element by element, and
against the two-kernel path (hyd_dispatch + hyd_pack) on the same inputs.  Cases cover the
register-key fast path (4 / 8 / 16 bins), the generic 64-bit path (V > 16, large costs), the
64-bit dispatch sums, infeasible pairs and iterations, 2 / 4 / 8 / 16 pipelines, B = 1 and 128,
and unaligned rows."""
import numpy as np
import pytest

import workload as w

pytestmark = pytest.mark.gpu
KEYS = ("sorted_len", "perm", "cost", "pipe", "lb", "mb", "v", "ptime", "makespan", "key")


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


def run(env, W, fused):
    A = env["assign"].Assigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad,
                               offsets=W.offsets if W.ragged else None, fused=fused)
    assert A.fused == fused
    A.run(env["assign"].lengths_to_device(W.lengths))
    return A.numpy()


def compare(g, o, tag):
    for k in KEYS:
        a, b = g[k], o[k]
        assert a.shape == b.shape, (tag, k)
        if not np.array_equal(a, b):
            bad = np.argwhere(a != b)
            raise AssertionError(f"{tag} {k}: {len(bad)} mismatches, first at {bad[:5].tolist()}: "
                                 f"gpu={a[tuple(bad[0])]} oracle={b[tuple(bad[0])]}")
    assert g["status"] == o["status"], (tag, g["status"], o["status"])


def check(env, W, tag):
    o = env["oracle"].assign_batch_ragged(W) if W.ragged else env["oracle"].assign_batch(W)
    g = run(env, W, True)
    compare(g, o, tag + " fused")
    g2 = run(env, W, False)
    compare(g2, o, tag + " two-kernel")


@pytest.mark.parametrize("cfg,n_cand,n_iter", [(1, 1, 700), (6, 260, 5)])
def test_small_configs(env, cfg, n_cand, n_iter):
    check(env, w.make_workload(cfg, n_cand=n_cand, n_iter=n_iter), f"cfg{cfg}")


@pytest.mark.parametrize("B", [1, 2, 31, 32, 33, 64, 100, 128])
def test_small_batch_sizes(env, B):
    rng = np.random.default_rng(B)
    base = w.make_workload(4, n_cand=150, n_iter=1)
    L = w.lengths_lognormal(rng, 3 * B, hi=32768).reshape(3, B)
    check(env, w.Workload(0, "small", L, base.schemes, base.cand, base.cand_np, base.k_pad), f"B{B}")


def test_small_wide_v_and_u64(env):
    """Small MaxLen forces V > 16 (generic path); large coefficients force 64-bit bin times and
    64-bit dispatch sums."""
    rng = np.random.default_rng(3)
    sch = np.concatenate([
        w.make_scheme(pp=2, max_len=3000, util_len=0, a_q32=1 << 20, b_q32=3 << 32, c_q32=50 << 32),
        w.make_scheme(pp=1, max_len=1500, util_len=0, a_q32=1 << 22, b_q32=2 << 32, c_q32=10 << 32),
        w.make_scheme(pp=4, max_len=2**20, util_len=0, a_q32=0, b_q32=(3 << 40), c_q32=0),
    ])
    L = rng.integers(50, 1500, (3, 120)).astype(np.uint32)
    W = w.custom_workload(L, sch, [[0, 1], [0, 0, 1], [2, 0, 1], [2, 2], [1], [2, 0, 0, 1, 1, 1]])
    check(env, W, "wideV-u64")


def test_small_pipelines_and_infeasible(env):
    """2 / 4 / 8 / 16 pipelines; lengths above some or all MaxLen (infeasible pairs, an
    all-infeasible iteration); equal lengths (ties)."""
    rng = np.random.default_rng(11)
    W5 = w.make_workload(5, n_cand=4, n_iter=1)
    rows = []
    for D in (2, 4, 8, 16, 16, 8):
        rows.append(w.canonical(W5.schemes, [int(x) for x in rng.integers(0, len(W5.schemes), D)]))
    L = w.lengths_mix(rng, 4 * 90).reshape(4, 90).astype(np.uint32)
    L[1, 3] = 200000
    L[2, 5] = 2**24
    L[3, :] = 777
    check(env, w.custom_workload(L, W5.schemes, rows), "pipes-infeasible")


def test_small_ragged_unaligned(env):
    rng = np.random.default_rng(4)
    base = w.make_workload(4, n_cand=90, n_iter=1)
    sizes = [1, 3, 17, 128, 5, 2, 127, 33]
    L = np.concatenate([w.lengths_lognormal(rng, b, hi=32768) for b in sizes]).astype(np.uint32)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.uint32)
    check(env, w.Workload(0, "ragged-small", L, base.schemes, base.cand, base.cand_np, base.k_pad, offsets=off),
          "ragged-unaligned")
