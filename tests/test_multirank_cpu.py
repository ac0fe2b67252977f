"""N > 1 host logic on CPU: candidate/iteration sharding, key packing, the allreduce-MIN
argmin (a6) and the winner-row exchange, over torch.distributed gloo with world sizes 2 and 3.

Each rank computes its shard's keys with the CPU oracle (standing in for the GPU path,
which is parity-checked separately) and reduces them with the product's own
``assign.reduce_keys``; the result must equal the single-process selection.  Then each rank
fills the zero-initialised winner-row block (pipe | mb | v | ptime per iteration, original
sequence order) for the iterations its candidates won and ``assign.share_rows`` sums it: every
rank must end with the single-process winners' plans (include/hyd.h hyd_assign_host)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workload as w


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, n_cand, n_iter, out):
    import oracle
    from paper_2412_07894_b200 import assign

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        W = w.make_workload(cfg, n_cand=n_cand, n_iter=n_iter)
        sh = assign.plan_shard(W.n_cand, W.n_iter, world, rank)
        sub = w.Workload(W.cfg, W.name, W.lengths[sh.iter_lo:sh.iter_hi], W.schemes,
                         W.cand[sh.cand_lo:sh.cand_hi], W.cand_np[sh.cand_lo:sh.cand_hi], W.k_pad)
        r = oracle.assign_batch(sub, n_threads=1, cand_offset=sh.cand_lo)
        key = torch.from_numpy(r["key"].copy())
        if sh.needs_reduce:
            assign.reduce_keys(key)
            full = key
            block = _win_block(r, key.numpy(), sh.cand_lo, sub.n_cand)
            out[("rows", rank)] = assign.share_rows(torch.from_numpy(block)).numpy().tobytes()
        else:  # iteration shards: gather the disjoint slices (off the metric path)
            full = torch.full((W.n_iter,), -1, dtype=torch.int64)
            full[sh.iter_lo:sh.iter_hi] = key
            dist.all_reduce(full, op=dist.ReduceOp.MAX)
        out[rank] = full.numpy().tolist()
    finally:
        dist.destroy_process_group()


def _win_block(r, key, cand_lo, n_cand):
    """Winner rows of the iterations whose winner lies in [cand_lo, cand_lo + n_cand), zeros
    elsewhere, as one int32 block: pipe u8 [It][B] | mb u16 [It][B] | v u16 [It][32] | ptime u64."""
    It, B = r["perm"].shape
    pipe = np.zeros((It, B), np.uint8)
    mb = np.zeros((It, B), np.uint16)
    v = np.zeros((It, 32), np.uint16)
    pt = np.zeros((It, 32), np.uint64)
    for t in range(It):
        if key[t] == 2**63 - 1:
            continue
        c = int(key[t] & ((1 << 20) - 1)) - cand_lo
        if 0 <= c < n_cand:
            pipe[t, r["perm"][t]] = r["pipe"][c, t]
            mb[t, r["perm"][t]] = r["mb"][c, t]
            v[t], pt[t] = r["v"][c, t], r["ptime"][c, t]
    raw = b"".join(x.tobytes() for x in (pipe, mb, v, pt))
    raw += b"\0" * (-len(raw) % 4)
    return np.frombuffer(raw, np.int32).copy()


@pytest.mark.parametrize("world,cfg,n_cand,n_iter", [(2, 4, 37, 3), (3, 2, 20, 4), (2, 1, 1, 6), (3, 3, 5, 2)])
def test_sharded_argmin_matches_single(world, cfg, n_cand, n_iter, oracle_lib):
    from paper_2412_07894_b200 import assign

    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), cfg, n_cand, n_iter, out), nprocs=world, join=True)
    W = w.make_workload(cfg, n_cand=n_cand, n_iter=n_iter)
    ref = oracle_lib.assign_batch(W)["key"]
    for r in range(world):
        assert np.array_equal(np.array(out[r], dtype=np.int64), ref), (r, out[r], ref)
    full = oracle_lib.assign_batch(W)
    want = _win_block(full, ref, 0, W.n_cand).tobytes()
    for r in range(world):
        if ("rows", r) in out:
            assert out[("rows", r)] == want, r
    ms, c = assign.decode_key(ref)
    feas = ref != 2**63 - 1
    assert (c[feas] < W.n_cand).all() and (ms[feas] > 0).all()


def test_plan_shard_partition():
    from paper_2412_07894_b200 import assign

    for C, It, G in [(4096, 1024, 8), (16384, 16, 8), (1, 4096, 8), (5, 7, 3), (7, 3, 8)]:
        shards = [assign.plan_shard(C, It, G, r) for r in range(G)]
        if C >= G:
            assert all(s.by == "cand" for s in shards)
            assert shards[0].cand_lo == 0 and shards[-1].cand_hi == C
            assert all(a.cand_hi == b.cand_lo for a, b in zip(shards, shards[1:]))
        else:
            assert all(s.by == "iter" and s.cand_lo == 0 and s.cand_hi == C for s in shards)
            assert shards[-1].iter_hi == It
            assert all(a.iter_hi == b.iter_lo for a, b in zip(shards, shards[1:]))


def test_key_decode_roundtrip():
    from paper_2412_07894_b200 import assign

    # the largest legal key: makespan 2^43-1, candidate 2^20-2 (2^20-1 would collide with INT64_MAX)
    keys = np.array([(123 << 20) | 77, 2**63 - 1, ((2**43 - 1) << 20) | (2**20 - 2)], dtype=np.int64)
    ms, c = assign.decode_key(keys)
    assert ms.tolist() == [123, -1, 2**43 - 1] and c.tolist() == [77, -1, 2**20 - 2]
