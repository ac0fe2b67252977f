"""Probe: pack-stage statistics after Alg. 1 vs HYD-H1 dispatch at config 4 (diagnostic only)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import workload as w
from paper_2412_07894_b200 import assign

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
nc = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
W = w.make_workload(cfg, n_cand=nc)
for trials in ([0] if len(sys.argv) > 3 else [0, 100]):
    A = assign.Assigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad, trials=trials, seed=2024)
    L = assign.lengths_to_device(W.lengths)
    A.run(L)
    torch.cuda.synchronize()
    t0 = time.time()
    A.run(L)
    torch.cuda.synchronize()
    dt = time.time() - t0
    o = A.numpy()
    cnt = A.pack_counters()
    v = o["v"].astype(np.int64)
    st = A.stats.cpu().numpy().reshape(-1, 24)
    u = st[:, 0:4].copy().view(np.uint32).ravel()
    u = u[(u != 0xFFFFFFFF) & (u > 0)]
    print(f"trials={trials} run {dt*1e3:.1f} ms  evals={cnt['bin_evals']:.3e} queued={cnt['queued_tasks']}"
          f"  V*: mean {v[v>0].mean():.2f} p99 {np.percentile(v[v>0],99):.0f} max {v.max()}"
          f"  U: mean {u.mean():.1f} p99 {np.percentile(u,99):.0f} max {u.max()}  handoff {cnt['handoff']}")
