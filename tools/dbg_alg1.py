import sys; sys.path.insert(0,'.')
import numpy as np, workload as w, oracle
from paper_2412_07894_b200 import assign
for trials in (0, 8):
    W = w.make_workload(2, n_cand=64, n_iter=3)
    A = assign.Assigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad, trials=trials, seed=1002)
    A.run(assign.lengths_to_device(W.lengths)); g = A.numpy()
    o = oracle.assign_batch(W, n_threads=0, trials=trials, seed=1002)
    for k in ("pipe","lb","mb","v","ptime","makespan","key"):
        bad = np.argwhere(g[k] != o[k])
        print(trials, k, len(bad), bad[:3].tolist())
    print(A.pack_counters())
    # per (c,t,j) mismatch of mb
    bad = np.argwhere(g["mb"] != o["mb"])
    if len(bad):
        c,t,i = bad[0]; j = o["pipe"][c,t,i]
        print("task", c,t,j, "v g/o", g["v"][c,t,j], o["v"][c,t,j], "U", (o["pipe"][c,t]==j).sum())
