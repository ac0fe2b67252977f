"""Race smoke test (compute-sanitizer's racecheck is closed on this GPU pool): the same workload
run repeatedly -- alone, and while another stream keeps the GPU's memory system and SMs busy,
which shifts how the CTAs' warps interleave -- must give bit-identical outputs.  Shared-memory
races in the lane scheduling (task records, unit lists, atomics, epoch protocol) or the fused
small-batch kernel would show up as run-to-run differences.  Config 4 / 6 / 5 shapes, reduced."""
import numpy as np
import pytest

import workload as w

pytestmark = pytest.mark.gpu
KEYS = ("pipe", "lb", "mb", "v", "ptime", "makespan", "key")


@pytest.fixture(scope="module")
def env():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_07894_b200 import assign

    return dict(torch=torch, assign=assign)


@pytest.mark.parametrize("cfg,n_cand,n_iter", [(4, 700, 12), (6, 900, 16), (5, 300, 1)])
def test_repeat_under_interference(env, cfg, n_cand, n_iter):
    torch, assign = env["torch"], env["assign"]
    W = w.make_workload(cfg, n_cand=n_cand, n_iter=n_iter)
    A = assign.Assigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad,
                        offsets=W.offsets if W.ragged else None)
    L = assign.lengths_to_device(W.lengths)
    A.run(L)
    ref = A.numpy()
    noise = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    side = torch.cuda.Stream()
    for rep in range(4):
        if rep % 2:
            with torch.cuda.stream(side):
                for _ in range(8):
                    noise.mul_(1.0001).add_(0.5)  # concurrent HBM + SM load on another stream
        A.run(L)
        g = A.numpy()
        for k in KEYS:
            assert np.array_equal(g[k], ref[k]), (cfg, rep, k)
    torch.cuda.synchronize()
