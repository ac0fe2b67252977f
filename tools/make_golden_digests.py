#!/usr/bin/env python
"""Write tests/golden/digests_cfgN.npz: per-iteration digests (workload/digest.py) of EVERY output
array of the CPU oracle on the full BASELINE configurations (all candidates and iterations of
configs 1-4 and 6 = the token-budget workload).  Config 5 is cut to its first ``--cfg5-cands``
candidates x ``--cfg5-iters`` iterations: the oracle enumerates every V of App. D's range with
a fresh LPT run (no pruning), 13.6 s per candidate-iteration on one core at config 5's
8192-sequence, 16-pipeline shape, so all 16 384 x 2 would be ~124 CPU-hours.  Imports only
``oracle`` and ``workload``: no value here comes from the CUDA path.

    python tools/make_golden_digests.py [--configs 1 2 3 4 5 6] [--chunk 8] [--threads 0]
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import workload as w  # noqa: E402
from workload.digest import iteration_digests  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")


def sub_iters(W, t0, t1):
    if not W.ragged:
        return w.Workload(W.cfg, W.name, np.ascontiguousarray(W.lengths[t0:t1]), W.schemes, W.cand, W.cand_np,
                          W.k_pad)
    off = W.offsets.astype(np.int64)
    lens = np.ascontiguousarray(W.lengths[off[t0]:off[t1]])
    return w.Workload(W.cfg, W.name, lens, W.schemes, W.cand, W.cand_np, W.k_pad,
                      offsets=(off[t0:t1 + 1] - off[t0]).astype(np.uint32))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="*", default=[1, 2, 3, 4, 5, 6])
    ap.add_argument("--chunk", type=int, default=8, help="iterations per oracle call")
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--cfg5-iters", type=int, default=2)
    ap.add_argument("--cfg5-cands", type=int, default=1024)
    args = ap.parse_args()
    oracle.build()
    for cfg in args.configs:
        W = w.make_workload(cfg)
        It = min(W.n_iter, args.cfg5_iters) if cfg == 5 else W.n_iter
        if cfg == 5:
            W = w.Workload(W.cfg, W.name, W.lengths, W.schemes, W.cand[: args.cfg5_cands].copy(),
                           W.cand_np[: args.cfg5_cands].copy(), W.k_pad, meta=W.meta)
        parts, status = [], 0
        t_start = time.time()
        for t0 in range(0, It, args.chunk):
            t1 = min(It, t0 + args.chunk)
            S = sub_iters(W, t0, t1)
            o = oracle.assign_batch_ragged(S, n_threads=args.threads) if S.ragged else \
                oracle.assign_batch(S, n_threads=args.threads)
            status |= int(o["status"])
            parts.append(iteration_digests(o, t1 - t0, offsets=S.offsets))
            print(f"cfg{cfg}: iterations {t1}/{It}, {time.time() - t_start:.0f} s", flush=True)
        dig = {k: np.concatenate([p[k] for p in parts]) for k in parts[0]}
        path = os.path.join(GOLDEN, f"digests_cfg{cfg}.npz")
        np.savez_compressed(path, n_iter=np.int64(It), n_cand=np.int64(W.n_cand), status=np.int64(status),
                            n_cand_total=np.int64(w.CONFIGS[cfg]["C"]),
                            workload=np.array(W.name), seed=np.int64(W.meta.get("seed", -1)), **dig)
        print(f"wrote {path}: {It} iterations x {W.n_cand} candidates, status {status}, "
              f"{time.time() - t_start:.0f} s", flush=True)


if __name__ == "__main__":
    main()
