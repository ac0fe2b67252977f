#!/usr/bin/env python
"""Small cases of every libhyd.so kernel family, run through the C ABI and checked against the
CPU oracle -- the program compute-sanitizer runs:

    compute-sanitizer --tool {memcheck,racecheck,initcheck,synccheck} python tools/sanitize_cases.py

Covers: sort + cost table (radix and warp sorts), HYD-H1 dispatch (packed and general kernels),
the pack lanes (VMAX 16 / 32 passes, warp queue incl. V > 32), select, gather / the host-buffer
call, the fused small-batch kernel (uniform and ragged), hyd_pipe_index, Alg. 1 (NEXT-1), the
proposal DP (NEXT-3), exact Eq. 3 / Eq. 1 (NEXT-4).  Prints SANITIZE_CASES_OK on success."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import workload as w  # noqa: E402
from paper_2412_07894_b200 import assign, hyd  # noqa: E402

KEYS = ("sorted_len", "perm", "cost", "pipe", "lb", "mb", "v", "ptime", "makespan", "key")


def same(g, o, tag, keys=KEYS):
    for k in keys:
        assert np.array_equal(g[k], o[k]), f"{tag}: {k} differs"
    assert g["status"] == o["status"], (tag, g["status"], o["status"])
    print("ok", tag, flush=True)


def run(W, **kw):
    A = assign.Assigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad,
                        offsets=W.offsets if W.ragged else None, **kw)
    A.run(assign.lengths_to_device(W.lengths))
    return A, A.numpy()


def main():
    torch.cuda.set_device(0)
    oracle.build()
    # uniform configs: warp sort (B <= 32, fused), radix sort + two-kernel path, lanes 16/32 + queue
    for cfg, nc, ni in ((1, 1, 40), (2, 9, 2), (4, 20, 2), (3, 6, 1)):
        W = w.make_workload(cfg, n_cand=nc, n_iter=ni)
        _, g = run(W)
        same(g, oracle.assign_batch(W), f"cfg{cfg}")
    # V > 32 (warp queue, scratch bins) and 64-bit paths
    rng = np.random.default_rng(5)
    sch = np.concatenate([
        w.make_scheme(pp=2, max_len=3000, util_len=2400, a_q32=1 << 20, b_q32=3 << 32, c_q32=50 << 32),
        w.make_scheme(pp=1, max_len=1500, util_len=1200, a_q32=1 << 22, b_q32=2 << 32, c_q32=10 << 32),
        w.make_scheme(pp=4, max_len=2**20, util_len=0, a_q32=0, b_q32=(3 << 40), c_q32=0),
    ])
    L = rng.integers(50, 900, (1, 700)).astype(np.uint32)
    W = w.custom_workload(L, sch, [[0, 1], [0, 0, 1], [2, 0, 1]])
    _, g = run(W)
    same(g, oracle.assign_batch(W), "bigV-u64")
    # fused small batches, uniform and ragged, and the two-kernel ragged path
    W6 = w.make_workload(6, n_cand=20, n_iter=2)
    for fused in (True, False):
        _, g = run(W6, fused=fused)
        same(g, oracle.assign_batch_ragged(W6), f"cfg6 fused={fused}")
    Wb = w.custom_workload(rng.integers(50, 1500, (2, 40)).astype(np.uint32), sch, [[0, 1], [2, 2, 0], [1]])
    _, g = run(Wb, fused=True)
    same(g, oracle.assign_batch(Wb), "small wideV-u64")
    # hyd_pipe_index + hyd_pack on the oracle's Alg. 1 rows; Alg. 1 on the GPU
    W4 = w.make_workload(4, n_cand=10, n_iter=2)
    A, _ = run(W4)
    s, _, cst, _ = oracle.cost_tables(W4)
    pipe = np.empty((W4.n_cand, W4.n_iter, W4.batch), np.uint8)
    for c in range(W4.n_cand):
        row = [int(k) for k in W4.cand[c, : W4.cand_np[c]]]
        for t in range(W4.n_iter):
            ok, p, _, _ = oracle.alg1_dispatch(s[t], cst[t], W4.schemes, row, 5, t, 3)
            pipe[c, t] = p if ok else 0xFF
    A.pipe.copy_(torch.from_numpy(pipe).cuda())
    hyd.pipe_index(A.sorted_len, A.cost, A.n_iter, A.batch, A.k_pad, A.schemes, A.n_schemes, A.cand, A.cand_np,
                   A.n_cand, A.max_np, A.pipe, A.lb, A.stats, A.members, A.status)
    hyd.pack(A.sorted_len, A.cost, A.n_iter, A.batch, A.k_pad, A.schemes, A.n_schemes, A.cand, A.cand_np, A.n_cand,
             A.max_np, A.pipe, A.stats, A.members, A.mb, A.v, A.ptime, A.makespan, A.status, A.ws)
    g = A.numpy()
    for c in range(W4.n_cand):
        row = [int(k) for k in W4.cand[c, : W4.cand_np[c]]]
        for t in range(W4.n_iter):
            ms, mb, _, pt, lb, _ = oracle.pack_pair(s[t], cst[t], W4.schemes, row, pipe[c, t])
            assert int(g["makespan"][t, c]) == ms and np.array_equal(g["mb"][c, t], mb), "pipe_index"
    print("ok pipe_index", flush=True)
    Wa = w.make_workload(4, n_cand=8, n_iter=2)
    _, g = run(Wa, trials=4, seed=9)
    o = oracle.assign_batch(Wa, trials=4, seed=9)
    same(g, o, "alg1", keys=("pipe", "lb", "mb", "makespan", "key"))
    # host-buffer call (gather winners)
    H = assign.HostAssigner(W4.schemes, W4.cand, W4.cand_np, W4.n_iter, W4.batch, W4.k_pad)
    key = H(torch.from_numpy(W4.lengths.view(np.int32)).pin_memory()).numpy()
    assert np.array_equal(key, oracle.assign_batch(W4)["key"]), "e2e"
    print("ok e2e", flush=True)
    # proposal DP (small grid) and the exact solvers
    lens = np.ascontiguousarray(w.make_workload(6, n_cand=2, n_iter=8).lengths)
    P = assign.Proposer(W4.schemes, 2048, 16, 16, 10)
    P.run(assign.lengths_to_device(lens))
    sel, _, _ = P.candidates()
    rows, _, _ = oracle.dp_propose(lens, W4.schemes, 2048, 16, 16, 10)
    assert [tuple(int(x) for x in r) for r in sel] == rows, "dp"
    print("ok dp", flush=True)
    Wq = w.Workload(0, "bb", W4.lengths[:, :9].copy(), W4.schemes, W4.cand[:4].copy(), np.minimum(W4.cand_np[:4], 3),
                    W4.k_pad)
    for cr in range(4):
        Wq.cand[cr, Wq.cand_np[cr]:] = 0xFF
    Aq = assign.Assigner(Wq.schemes, Wq.cand, Wq.cand_np, Wq.n_iter, Wq.batch, Wq.k_pad, fused=False)
    pc, pt = np.repeat(np.arange(4), 2), np.tile(np.arange(2), 4)
    val, _, _, proved = Aq.eq3_exact(assign.lengths_to_device(Wq.lengths), pc, pt)
    for q in range(pc.size):
        s_, _, c_, _ = oracle.cost_table(Wq.lengths[pt[q]], Wq.schemes, Wq.k_pad)
        ok, v, _, _ = oracle.eq3_exact(s_, c_, Wq.schemes, [int(k) for k in Wq.cand[pc[q], : Wq.cand_np[pc[q]]]])
        assert ok == bool(proved[q]) and v == int(val[q]), "eq3"
    Aq.run(assign.lengths_to_device(Wq.lengths))
    Aq.eq1_exact(pc, pt, np.zeros_like(pc))
    print("ok exact", flush=True)
    torch.cuda.synchronize()
    print("SANITIZE_CASES_OK", flush=True)


if __name__ == "__main__":
    main()
