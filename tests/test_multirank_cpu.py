"""N > 1 host logic on CPU: candidate/iteration sharding, key packing and the
allreduce-MIN argmin (a6), over torch.distributed gloo with world sizes 2 and 3.

Each rank computes its shard's keys with the CPU oracle (standing in for the GPU path,
which is parity-checked separately) and reduces them with the product's own
``assign.reduce_keys``; the result must equal the single-process selection."""
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
        else:  # iteration shards: gather the disjoint slices (off the metric path)
            full = torch.full((W.n_iter,), -1, dtype=torch.int64)
            full[sh.iter_lo:sh.iter_hi] = key
            dist.all_reduce(full, op=dist.ReduceOp.MAX)
        out[rank] = full.numpy().tolist()
    finally:
        dist.destroy_process_group()


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
