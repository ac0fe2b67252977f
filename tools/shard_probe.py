"""Per-shard step time of config 4 at G = 4 contiguous candidate blocks, one GPU (diagnostic)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import workload as w
from paper_2412_07894_b200 import assign

W = w.make_workload(4)
G = int(sys.argv[1]) if len(sys.argv) > 1 else 4
L = assign.lengths_to_device(W.lengths)
for mode in ("contiguous", "interleaved"):
    out = []
    for g in range(G):
        cs = np.arange(g * W.n_cand // G, (g + 1) * W.n_cand // G) if mode == "contiguous" else np.arange(g, W.n_cand, G)
        A = assign.Assigner(W.schemes, W.cand[cs], W.cand_np[cs], W.n_iter, W.batch, W.k_pad)
        for _ in range(2):
            A.run(L)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            A.run(L)
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) / 3)
        del A
    print(mode, [round(x, 2) for x in out], "max", round(max(out), 2), "mean", round(float(np.mean(out)), 2))
