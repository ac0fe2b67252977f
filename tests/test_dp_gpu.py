"""GPU parity of NEXT-3 (include/hyd.h hyd_dp_propose) against the CPU oracle (oracle/dpref.c):
the exact DP tables (t as num/den, recorded choices), the strategies, the roundings and the
proposed subset, element by element."""
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


def check(env, lens, schemes, step, J, N, scale):
    O, assign = env["oracle"], env["assign"]
    P = assign.Proposer(schemes, step, J, N, scale)
    P.run(assign.lengths_to_device(lens))
    sel, cand, cnp = P.candidates()
    rows, (pre, tn, td, ch), st = O.dp_propose(lens, schemes, step, J, N, scale)
    u = lambda x, dt: x.cpu().numpy().view(dt)
    assert np.array_equal(u(P.t_num, np.uint64), tn)
    assert np.array_equal(u(P.t_den, np.uint64), td)
    assert np.array_equal(u(P.choice, np.int32), ch)
    counts = u(P.counts, np.uint16)
    for j in range(1, J + 1):
        ok, c, top = O.dp_strategy(ch, td, schemes, J, N, scale, j)
        assert np.array_equal(counts[j], c.astype(np.uint16)) if ok else (counts[j] == 0).all()
    assert [tuple(int(x) for x in r) for r in sel] == rows
    assert int(P.status.item()) == st
    # hyd_dp_candidates: each proposed row as a canonical candidate (MaxLen desc, index asc)
    ml = schemes["max_len"].astype(np.int64)
    order = sorted(range(len(schemes)), key=lambda k: (-ml[k], k))
    assert cand.shape[0] == len(rows)
    for m, r in enumerate(rows):
        ks = [k for k in order for _ in range(r[k])]
        assert int(cnp[m]) == len(ks) and cand[m, : len(ks)].tolist() == ks and (cand[m, len(ks):] == 0xFF).all()
    return sel, cand, cnp


@pytest.mark.parametrize("scale", [1, 10])
def test_dp_parity_cfg4_sample(env, scale):
    W = w.make_workload(4, n_cand=2, n_iter=40)
    lens = np.ascontiguousarray(W.lengths.reshape(-1))
    sel, cand, cnp = check(env, lens, W.schemes, 1024, 32, 16 if scale == 10 else 64, scale)
    assert len(sel) >= 1 and (cnp >= 1).all()


def test_dp_parity_tiny_and_ragged_grid(env):
    rng = np.random.default_rng(4)
    for _ in range(4):
        K = int(rng.integers(1, 5))
        sch = np.concatenate([w.make_scheme(tp=int(rng.integers(1, 3)), pp=int(rng.integers(1, 3)),
                                            max_len=int(rng.choice([512, 2048, 4096])),
                                            a_q32=int(rng.integers(0, 9)) << 20, b_q32=int(rng.integers(1, 5)) << 32,
                                            c_q32=int(rng.integers(0, 40)) << 32) for _ in range(K)])
        sch[0]["max_len"] = 4096
        lens = rng.integers(1, 6000, int(rng.integers(1, 3000))).astype(np.uint32)
        check(env, lens, sch, 128, 32, int(rng.integers(1, 9)), int(rng.choice([1, 10])))


def test_dp_full_grid_runs(env):
    """The paper's grid (l step 128 to 32K, n/d step 0.1, 64 GPUs): runs, is internally
    consistent (t non-increasing in n, non-decreasing in l) and proposes candidates within budget."""
    W = w.make_workload(6, n_cand=2, n_iter=64)
    assign = env["assign"]
    P = assign.Proposer(W.schemes, 128, 256, 64, 10)
    P.run(assign.lengths_to_device(np.ascontiguousarray(W.lengths)))
    sel, cand, cnp = P.candidates()
    g = np.array([int(s["tp"]) * int(s["pp"]) * int(s["cp"]) for s in W.schemes])
    assert len(sel) >= 1 and ((sel.astype(np.int64) * g).sum(1) <= 64).all()
    tn = P.t_num.cpu().numpy().view(np.uint64).astype(object)
    td = P.t_den.cpu().numpy().view(np.uint64).astype(object)
    for j in range(2, 257):  # t[N][l] non-decreasing in l (exact cross-multiplication)
        assert tn[640, j - 1] * td[640, j] <= tn[640, j] * td[640, j - 1]
    for nu in range(2, 641, 37):
        assert tn[nu, 256] * td[nu - 1, 256] <= tn[nu - 1, 256] * td[nu, 256] or td[nu - 1, 256] == 0
    assert int(P.status.item()) == 0


def test_dp_parity_paper_grid(env):
    """The paper's own grid (P:713 footnote: n and d in steps of 0.1, l in steps of 128 tokens to
    the 32K context; 64 GPUs) on config 6's 1024-iteration length sample -- the bench --dp
    workload -- bit-exact against the enumerating oracle (~4.7e9 transitions on the CPU)."""
    W = w.make_workload(6, n_cand=2, n_iter=1024)
    check(env, np.ascontiguousarray(W.lengths), W.schemes, 128, 256, 64, 10)
