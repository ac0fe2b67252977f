"""Pack-pass counters of one cfg step (diagnostic): hand-off reasons, phase-2 units, per-phase
SM cycles of thread 0 of every VMAX-16 CTA (include/hyd.h workspace header)."""
import sys

import torch

sys.path.insert(0, ".")
import workload as w
from paper_2412_07894_b200 import assign

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
nc = int(sys.argv[2]) if len(sys.argv) > 2 else None
W = w.make_workload(cfg, n_cand=nc)
A = assign.Assigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad, offsets=W.offsets)
L = assign.lengths_to_device(W.lengths)
A.run(L)
torch.cuda.synchronize()
pc = A.pack_counters()
h = pc["handoff"]
clk = {k: v for k, v in h.items() if k.startswith("clk")}
tot = sum(clk.values()) or 1
print("bin_evals", pc["bin_evals"], "queued", pc["queued_tasks"])
print({k: v for k, v in h.items() if not k.startswith("clk")})
print({k: round(v / tot, 3) for k, v in clk.items()})
