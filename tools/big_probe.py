import sys, torch, numpy as np
sys.path.insert(0,'.')
import workload as w
from paper_2412_07894_b200 import assign
for nc in (512, None):
    W=w.make_workload(4, n_cand=nc)
    A=assign.Assigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad)
    A.run(assign.lengths_to_device(W.lengths)); torch.cuda.synchronize()
    x=A.ws[0:256].cpu().numpy().view(np.uint64)
    m=int(x[19]); print(nc, "queued", int(x[0]), "max cyc", m>>32, "U", (m>>16)&0xFFFF, "nV", m&0xFFFF, "sum cyc", int(x[20]), "n>200k", int(x[21]), "vrange", int(x[22])>>32, int(x[22])&0xFFFFFFFF)
