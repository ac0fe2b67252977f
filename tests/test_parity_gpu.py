"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Integer path => bit-exact on every output: sorted_len, perm, cost, pipe, lb, mb, v, ptime,
makespan, key and the status word.  Reduced sizes span several CTA tiles and a ragged tail;
full BASELINE sizes are checked on sampled (c,t) pairs computed one by one by the oracle,
plus whole-iteration keys for sampled iterations.
"""
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


def run_gpu(env, W, cand_offset=0):
    A = env["assign"].Assigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad, cand_offset=cand_offset)
    A.run(env["assign"].lengths_to_device(W.lengths))
    return A.numpy()


def compare_all(g, o, tag=""):
    for k in ("sorted_len", "perm", "cost", "pipe", "lb", "mb", "v", "ptime", "makespan", "key"):
        a, b = g[k], o[k]
        assert a.shape == b.shape, (tag, k, a.shape, b.shape)
        if not np.array_equal(a, b):
            bad = np.argwhere(a != b)
            raise AssertionError(f"{tag} {k}: {len(bad)} mismatches, first at {bad[:5].tolist()}: "
                                 f"gpu={a[tuple(bad[0])]} oracle={b[tuple(bad[0])]}")
    assert g["status"] == o["status"], (tag, g["status"], o["status"])


# (cfg, n_cand, n_iter): several tiles + ragged tails per kernel geometry
CASES = [
    (1, 1, 300),
    (2, 64, 9),
    (2, 37, 5),
    (3, 150, 3),
    (4, 133, 3),
    (4, 300, 2),
]


@pytest.mark.parametrize("cfg,n_cand,n_iter", CASES)
def test_parity_reduced(env, cfg, n_cand, n_iter):
    W = w.make_workload(cfg, n_cand=n_cand, n_iter=n_iter)
    g = run_gpu(env, W)
    o = env["oracle"].assign_batch(W, n_threads=0)
    compare_all(g, o, f"cfg{cfg}")


def test_parity_cfg5_prefix(env):
    """Stress shape (16 pipelines, lengths to 256K) on a 2048-sequence prefix."""
    W = w.make_workload(5, n_cand=24, n_iter=2)
    W.lengths = np.ascontiguousarray(W.lengths[:, :2048])
    g = run_gpu(env, W)
    o = env["oracle"].assign_batch(W, n_threads=0)
    compare_all(g, o, "cfg5-prefix")


def test_parity_worked_example(env):
    import json
    import os

    gd = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_example.json")))
    W = w.custom_workload(gd["lengths"], w.make_scheme(**gd["scheme"]), [gd["candidate"]])
    g = run_gpu(env, W)
    e = gd["expect"]
    assert list(g["pipe"][0, 0]) == e["pipe"] and list(g["mb"][0, 0]) == e["mb"]
    assert int(g["makespan"][0, 0]) == e["makespan"] and int(g["key"][0]) == e["key"]


def _edge_workloads():
    rng = np.random.default_rng(77)
    out = []
    sch = w.make_workload(4, n_cand=40, n_iter=1)
    # ragged batch (B % 16 != 0, B % 4 != 0), B = 1, all lengths equal, infeasible iterations
    for B in (1, 3, 17, 250, 1001):
        L = w.lengths_lognormal(rng, 3 * B, hi=32768).reshape(3, B)
        out.append((f"B{B}", w.Workload(0, "edge", L, sch.schemes, sch.cand, sch.cand_np, sch.k_pad)))
    L = np.full((2, 64), 700, np.uint32)
    out.append(("equal", w.Workload(0, "edge", L, sch.schemes, sch.cand, sch.cand_np, sch.k_pad)))
    L = w.lengths_lognormal(rng, 4 * 96, hi=32768).reshape(4, 96)
    L[1, 5] = 120000  # longer than every MaxLen except the longest schemes -> infeasible candidates
    L[2, 7] = 2**24  # longer than every scheme: all-infeasible iteration -> key INT64_MAX
    out.append(("infeasible", w.Workload(0, "edge", L, sch.schemes, sch.cand, sch.cand_np, sch.k_pad)))
    # tiny random heterogeneous instances (brute-force regime), many candidates
    for s in range(3):
        W = w.random_small_instance(np.random.default_rng(s), 7, 3)
        out.append((f"tiny{s}", W))
    # many pipelines (D = 32): a wide candidate
    W5 = w.make_workload(5, n_cand=4, n_iter=1)
    cand = np.full((3, 32), 0xFF, np.uint8)
    for c in range(3):
        ks = w.canonical(W5.schemes, [int(x) for x in rng.integers(0, len(W5.schemes), 32)])
        cand[c, :32] = ks
    L = w.lengths_lognormal(rng, 2 * 300, hi=32768).reshape(2, 300)
    out.append(("D32", w.Workload(0, "edge", L, W5.schemes, cand, np.full(3, 32, np.uint8), W5.k_pad)))
    return out


@pytest.mark.parametrize("name,W", _edge_workloads(), ids=lambda x: x if isinstance(x, str) else "")
def test_parity_edges(env, name, W):
    g = run_gpu(env, W)
    o = env["oracle"].assign_batch(W, n_threads=0)
    compare_all(g, o, name)


def test_parity_big_v_path(env):
    """Force the warp-per-pipeline path (V > 32) and its scratch path (V > 256):
    UtilLen = 0 and a small MaxLen make V_lo large."""
    rng = np.random.default_rng(5)
    sch = np.concatenate([
        w.make_scheme(pp=2, max_len=3000, util_len=2400, a_q32=1 << 20, b_q32=3 << 32, c_q32=50 << 32),
        w.make_scheme(pp=1, max_len=1500, util_len=1200, a_q32=1 << 22, b_q32=2 << 32, c_q32=10 << 32),
        w.make_scheme(pp=3, max_len=900, util_len=700, a_q32=0, b_q32=5 << 32, c_q32=7 << 32),
    ])
    L = rng.integers(50, 900, (2, 2000)).astype(np.uint32)
    W = w.custom_workload(L, sch, [[0, 1, 2], [0, 0, 1, 2], [0], [1, 2, 2]])
    g = run_gpu(env, W)
    assert g["v"].max() > 256
    o = env["oracle"].assign_batch(W, n_threads=0)
    compare_all(g, o, "bigV")


def test_parity_wide_u64_path(env):
    """Bin times above 2^32 force the 64-bit paths of dispatch and pack."""
    rng = np.random.default_rng(9)
    sch = np.concatenate([
        w.make_scheme(pp=4, max_len=2**20, util_len=0, a_q32=0, b_q32=(3 << 40), c_q32=0),
        w.make_scheme(pp=1, max_len=2**19, util_len=0, a_q32=0, b_q32=(1 << 41), c_q32=1 << 32),
    ])
    L = rng.integers(1000, 2**18, (2, 600)).astype(np.uint32)
    W = w.custom_workload(L, sch, [[0, 1], [0, 0, 1], [0, 0, 0, 1, 1]])
    g = run_gpu(env, W)
    assert int(g["ptime"].max()) > 2**32
    o = env["oracle"].assign_batch(W, n_threads=0)
    compare_all(g, o, "u64")


def test_parity_capacity_free_boundary(env):
    """Linear costs (tau = b l exactly) make alpha = b and cap = b MaxLen tight: a bin's time is
    b times its tokens, so the capacity-free certificate (thr <= cap) holds up to equality while
    MaxLen binds often (lengths up to MaxLen / 2, V near ceil(S / MaxLen))."""
    rng = np.random.default_rng(21)
    sch = np.concatenate([
        w.make_scheme(pp=2, max_len=4096, util_len=0, a_q32=0, b_q32=3 << 32, c_q32=0),
        w.make_scheme(pp=1, max_len=2048, util_len=0, a_q32=0, b_q32=5 << 32, c_q32=0),
        w.make_scheme(pp=3, max_len=6000, util_len=0, a_q32=0, b_q32=2 << 32, c_q32=1 << 32),
        w.make_scheme(pp=4, max_len=3000, util_len=0, a_q32=0, b_q32=7 << 32, c_q32=0),
    ])
    L = rng.integers(100, 2049, (5, 256)).astype(np.uint32)
    rows = [w.canonical(sch, [int(x) for x in rng.integers(0, 4, int(rng.integers(1, 9)))]) for _ in range(60)]
    W = w.custom_workload(L, sch, rows)
    g = run_gpu(env, W)
    o = env["oracle"].assign_batch(W, n_threads=0)
    compare_all(g, o, "capfree")


@pytest.mark.parametrize("cfg", [2, 3, 4, 5])
def test_parity_full_size_sampled(env, cfg):
    """BASELINE full sizes in the bench launch configuration; oracle on sampled pairs."""
    torch = env["torch"]
    W = w.make_workload(cfg)
    A = env["assign"].Assigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad)
    A.run(env["assign"].lengths_to_device(W.lengths))
    torch.cuda.synchronize()
    O = env["oracle"]
    tables = O.cost_tables(W)
    s, p, cst, st = tables
    u = lambda x, dt: x.cpu().numpy().view(dt)
    assert np.array_equal(u(A.sorted_len, np.uint32), s) and np.array_equal(u(A.perm, np.uint32), p)
    assert np.array_equal(u(A.cost, np.uint32), cst)
    rng = np.random.default_rng(cfg)
    n = {2: 400, 3: 300, 4: 400, 5: 8}[cfg]
    pc = rng.integers(0, W.n_cand, n)
    pt = rng.integers(0, W.n_iter, n)
    o = O.assign_pairs(W, pc, pt, tables=tables)
    ic, it = torch.from_numpy(pc).cuda(), torch.from_numpy(pt).cuda()
    assert np.array_equal(u(A.pipe[ic, it], np.uint8), o["pipe"])
    assert np.array_equal(u(A.mb[ic, it], np.uint16), o["mb"])
    assert np.array_equal(u(A.v[ic, it], np.uint16), o["v"])
    assert np.array_equal(u(A.ptime[ic, it], np.uint64), o["ptime"])
    assert np.array_equal(u(A.lb[ic, it], np.uint64), o["lb"])
    assert np.array_equal(u(A.makespan[it, ic], np.uint64), o["makespan"])
    # whole-iteration keys on sampled iterations (needs every candidate of t)
    if cfg in (2, 3, 4):
        for t in rng.integers(0, W.n_iter, 2 if cfg == 4 else 3):
            t = int(t)
            o2 = O.assign_pairs(W, np.arange(W.n_cand), np.full(W.n_cand, t), tables=tables)
            assert np.array_equal(u(A.makespan[t], np.uint64), o2["makespan"]), t
            assert int(A.key[t].item()) == O.select(o2["makespan"])[0]
    assert A.status_bits() == st


def test_e2e_host_path_matches_device_path(env):
    torch = env["torch"]
    assign = env["assign"]
    W = w.make_workload(3, n_cand=200, n_iter=6)
    g = run_gpu(env, W)
    H = assign.HostAssigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad)
    lh = torch.from_numpy(W.lengths.view(np.int32)).pin_memory()
    key = H(lh).numpy()
    assert np.array_equal(key, g["key"])
    ms, cw = assign.decode_key(key)
    for t in range(W.n_iter):
        c = int(cw[t])
        if c < 0:
            continue
        perm = g["perm"][t]
        want_pipe = np.empty(W.batch, np.uint8)
        want_pipe[perm] = g["pipe"][c, t]
        want_mb = np.empty(W.batch, np.uint16)
        want_mb[perm] = g["mb"][c, t]
        assert np.array_equal(H.win_pipe[t].numpy(), want_pipe)
        assert np.array_equal(H.win_mb[t].numpy().view(np.uint16), want_mb)
        assert np.array_equal(H.win_ptime[t].numpy().view(np.uint64), g["ptime"][c, t])


def test_cand_offset_keys(env):
    W = w.make_workload(2, n_cand=20, n_iter=4)
    g = run_gpu(env, W, cand_offset=1000)
    o = env["oracle"].assign_batch(W, cand_offset=1000)
    assert np.array_equal(g["key"], o["key"])


def test_deterministic_repeat(env):
    W = w.make_workload(4, n_cand=64, n_iter=4)
    a = run_gpu(env, W)
    b = run_gpu(env, W)
    for k in ("pipe", "mb", "v", "ptime", "makespan", "key"):
        assert np.array_equal(a[k], b[k])
