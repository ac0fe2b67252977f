"""GPU parity of NEXT-2 (token-budget ragged batches, include/hyd.h *_ragged) against the CPU
oracle, element by element, through the C ABI."""
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


def run_gpu(env, W, fused=None):
    A = env["assign"].Assigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad, offsets=W.offsets,
                               fused=fused)
    A.run(env["assign"].lengths_to_device(W.lengths))
    return A, A.numpy()


def compare(g, o, tag):
    for k in ("sorted_len", "perm", "cost", "pipe", "lb", "mb", "v", "ptime", "makespan", "key"):
        a, b = g[k], o[k]
        assert a.shape == b.shape, (tag, k, a.shape, b.shape)
        if not np.array_equal(a, b):
            bad = np.argwhere(a != b)
            raise AssertionError(f"{tag} {k}: {len(bad)} mismatches, first at {bad[:5].tolist()}: "
                                 f"gpu={a[tuple(bad[0])]} oracle={b[tuple(bad[0])]}")
    assert g["status"] == o["status"], (tag, g["status"], o["status"])


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("n_cand,n_iter", [(133, 6), (300, 3), (1, 9)])
def test_ragged_parity_cfg6(env, n_cand, n_iter, fused):
    """Both code paths: hyd_dispatch_pack (one kernel) and hyd_dispatch + hyd_pack."""
    W = w.make_workload(6, n_cand=n_cand, n_iter=n_iter)
    A, g = run_gpu(env, W, fused=fused)
    assert A.fused == fused
    compare(g, env["oracle"].assign_batch_ragged(W), f"cfg6-{n_cand}x{n_iter}")


def test_ragged_edges(env):
    """B_t = 1, odd and misaligned rows, the largest batch in the middle, infeasible iterations."""
    rng = np.random.default_rng(8)
    base = w.make_workload(4, n_cand=70, n_iter=1)
    sizes = [1, 3, 17, 1, 250, 33, 2, 96, 5]
    L = np.concatenate([w.lengths_lognormal(rng, b, hi=32768) for b in sizes]).astype(np.uint32)
    L[sizes[0] + sizes[1] + 4] = 120000  # an infeasible-for-most iteration
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.uint32)
    W = w.Workload(0, "ragged-edge", L, base.schemes, base.cand, base.cand_np, base.k_pad, offsets=off)
    _, g = run_gpu(env, W)
    compare(g, env["oracle"].assign_batch_ragged(W), "ragged-edges")
    W2 = w.Workload(0, "ragged-edge-small", np.ascontiguousarray(L[: off[4]]), base.schemes, base.cand, base.cand_np,
                    base.k_pad, offsets=off[:5].copy())  # batches <= 17: the fused kernel
    A2, g2 = run_gpu(env, W2)
    assert A2.fused
    compare(g2, env["oracle"].assign_batch_ragged(W2), "ragged-edges-fused")


def test_uniform_as_ragged_matches_uniform_path(env):
    W = w.make_workload(4, n_cand=90, n_iter=3)
    A = env["assign"].Assigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad)
    A.run(env["assign"].lengths_to_device(W.lengths))
    u = A.numpy()
    R = w.Workload(W.cfg, W.name, W.lengths.reshape(-1).copy(), W.schemes, W.cand, W.cand_np, W.k_pad,
                   offsets=np.arange(W.n_iter + 1, dtype=np.uint32) * W.batch)
    _, r = run_gpu(env, R)
    for k in ("pipe", "mb", "lb", "v", "ptime", "makespan", "key"):
        assert np.array_equal(r[k].reshape(-1), u[k].reshape(-1)), k


def test_ragged_e2e_host_path(env):
    torch, assign = env["torch"], env["assign"]
    W = w.make_workload(6, n_cand=200, n_iter=8)
    _, g = run_gpu(env, W)
    H = assign.HostAssigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad, offsets=W.offsets)
    lh = torch.from_numpy(W.lengths.view(np.int32).copy()).pin_memory()
    key = H(lh).numpy()
    assert np.array_equal(key, g["key"])
    ms, cw = assign.decode_key(key)
    off = W.offsets.astype(np.int64)
    wp = H.win_pipe.numpy()
    for t in range(W.n_iter):
        # winner's plan in original order: position perm[i] holds sorted position i's pipeline
        perm = g["perm"][off[t]:off[t + 1]]
        row = g["pipe"][cw[t], off[t]:off[t + 1]]
        exp = np.empty_like(row)
        exp[perm] = row
        assert np.array_equal(wp[off[t]:off[t + 1]], exp), t


def test_ragged_full_size_sampled(env):
    """cfg6 at full size (4096 candidates x 1024 token-budget iterations); oracle on sampled pairs."""
    torch = env["torch"]
    W = w.make_workload(6)
    A, _ = run_gpu(env, W)
    torch.cuda.synchronize()
    rng = np.random.default_rng(6)
    pc = rng.integers(0, W.n_cand, 300)
    pt = rng.integers(0, W.n_iter, 300)
    o = env["oracle"].assign_pairs_ragged(W, pc, pt)
    off = W.offsets.astype(np.int64)
    u = lambda x, dt: x.cpu().numpy().view(dt)
    pipe, mb = u(A.pipe, np.uint8), u(A.mb, np.uint16)
    lb, v, pti, ms = u(A.lb, np.uint64), u(A.v, np.uint16), u(A.ptime, np.uint64), u(A.makespan, np.uint64)
    for q, (c, t) in enumerate(zip(pc, pt)):
        a, b = off[t], off[t + 1]
        assert np.array_equal(pipe[c, a:b], o[q]["pipe"]), (c, t)
        assert np.array_equal(mb[c, a:b], o[q]["mb"]), (c, t)
        assert lb[c, t] == o[q]["lb"] and ms[t, c] == o[q]["makespan"], (c, t)
        assert np.array_equal(v[c, t], o[q]["v"]) and np.array_equal(pti[c, t], o[q]["ptime"]), (c, t)
    assert A.status_bits() == 0
