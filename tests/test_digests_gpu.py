"""Full-size parity (north_star: "bit-exact oracle agreement on all five configs"; SURVEY §8(d):
"no subsampling"): every output array of the CUDA path -- sorted_len, perm, cost, pipe, lb, mb, v,
ptime, makespan, key -- for EVERY candidate and iteration of BASELINE configs 1-6 (config 6:
token-budget batches), in the launch configuration bench.py times, against per-iteration digests
of the CPU oracle's outputs (tests/golden/digests_cfgN.npz, written by
tools/make_golden_digests.py, which imports only oracle/ and workload/).  A golden file that
covers fewer candidates or iterations than the configuration is checked on that prefix.  Digest = workload/digest.py (BLAKE2b of each iteration's slice)."""
import os

import numpy as np
import pytest

import workload as w
from workload.digest import iteration_digests

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def env():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_07894_b200 import assign, hyd

    hyd.lib()
    return dict(torch=torch, assign=assign)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5, 6])
def test_full_size_digests(env, cfg):
    g = np.load(os.path.join(GOLDEN, f"digests_cfg{cfg}.npz"))
    W = w.make_workload(cfg)
    assert str(g["workload"]) == W.name and int(g["n_cand_total"]) == W.n_cand
    It, Cn = int(g["n_iter"]), int(g["n_cand"])
    if It < W.n_iter or Cn < W.n_cand:  # config 5: the first Cn candidates x It iterations
        W = w.Workload(W.cfg, W.name, np.ascontiguousarray(W.lengths[:It]), W.schemes, W.cand[:Cn].copy(),
                       W.cand_np[:Cn].copy(), W.k_pad)
    assign = env["assign"]
    A = assign.Assigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad,
                        offsets=W.offsets if W.ragged else None)
    A.run(assign.lengths_to_device(W.lengths))
    out = A.numpy()
    del A
    env["torch"].cuda.empty_cache()
    dig = iteration_digests(out, It, offsets=W.offsets if W.ragged else None)
    for k, d in dig.items():
        bad = np.nonzero(d != g[k])[0]
        assert bad.size == 0, f"cfg{cfg} {k}: {bad.size} of {It} iterations differ, first {bad[:8].tolist()}"
    assert out["status"] == int(g["status"])
