"""torchrun worker of tests/test_multigpu_gpu.py: N ranks over NCCL, one GPU each.

Checks (include/hyd.h hyd_assign_host):
  * a6 on hardware: the NCCL allreduce-MIN of the per-rank keys equals a one-rank run over all
    candidates (rank 0 computes it) -- device path (Assigner + assign.reduce_keys) and the
    host-buffer call (HostAssigner with its collective callback);
  * every rank receives every iteration's winning plan (win_pipe / win_mb / win_v / win_ptime)
    equal to the one-rank run's;
  * the collectives are ordered on the stream passed to the call (a side stream here)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import workload as w  # noqa: E402
from paper_2412_07894_b200 import assign  # noqa: E402


def host_rows(H):
    return [H.key.numpy().copy(), H.win_pipe.numpy().copy(), H.win_mb.numpy().copy(),
            H.win_v.numpy().copy(), H.win_ptime.numpy().copy()]


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    bad = []
    for cfg, n_cand, n_iter in ((4, 203, 5), (3, 64, 3), (6, 90, 4)):
        W = w.make_workload(cfg, n_cand=n_cand, n_iter=n_iter)
        sh = assign.plan_shard(W.n_cand, W.n_iter, world, rank)
        assert sh.by == "cand"
        cand, cnp = W.cand[sh.cand_lo:sh.cand_hi], W.cand_np[sh.cand_lo:sh.cand_hi]
        offs = W.offsets if W.ragged else None
        # device path: shard keys + NCCL allreduce-MIN
        A = assign.Assigner(W.schemes, cand, cnp, W.n_iter, W.batch, W.k_pad, cand_offset=sh.cand_lo, offsets=offs)
        A.run(assign.lengths_to_device(W.lengths))
        assign.reduce_keys(A.key)
        key_dev = A.key.cpu().numpy()
        # host-buffer call on a side stream with the collective callback
        side = torch.cuda.Stream()
        H = assign.HostAssigner(W.schemes, cand, cnp, W.n_iter, W.batch, W.k_pad, cand_offset=sh.cand_lo,
                                reduce=True, offsets=offs)
        lh = torch.from_numpy(np.ascontiguousarray(W.lengths).view(np.int32)).pin_memory()
        H(lh, stream=side)
        mine = host_rows(H)
        # reference: rank 0, one rank over every candidate
        if rank == 0:
            F = assign.Assigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad, offsets=offs)
            F.run(assign.lengths_to_device(W.lengths))
            ref_key = F.key.cpu().numpy()
            HF = assign.HostAssigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad, offsets=offs)
            HF(lh)
            ref = host_rows(HF)
            assert np.array_equal(ref[0], ref_key)
        else:
            ref = None
        obj = [ref]
        dist.broadcast_object_list(obj, src=0)
        ref = obj[0]
        tag = f"cfg{cfg} rank{rank}"
        if not np.array_equal(key_dev, ref[0]):
            bad.append(f"{tag}: device-path reduced keys differ from the one-rank run")
        for name, a, b in zip(("key", "win_pipe", "win_mb", "win_v", "win_ptime"), mine, ref):
            if not np.array_equal(a, b):
                bad.append(f"{tag}: host call {name} differs from the one-rank run")
        won = np.unique(assign.decode_key(ref[0])[1])
        if rank == 0:
            print(f"{tag}: {W.n_iter} iterations, winners {won.tolist()}", flush=True)
    ok = torch.tensor([0 if not bad else 1], device="cuda")
    dist.all_reduce(ok)
    for b in bad:
        print("FAIL", b, flush=True)
    if rank == 0 and int(ok.item()) == 0:
        print(f"MGPU_OK world={world}", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0 if int(ok.item()) == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
