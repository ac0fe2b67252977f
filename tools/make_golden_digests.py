#!/usr/bin/env python
"""Write tests/golden/digests_cfgN.npz: per-iteration digests (workload/digest.py) of EVERY output
array of the CPU oracle on the full BASELINE configurations (all candidates and iterations of
configs 1-6; config 6 = the token-budget workload).  Config 5 (16 384 candidates x 16 iterations
of 8192 sequences on 16 pipelines, ~0.5 CPU-s per candidate-iteration with the heap LPT) is
written in iteration ranges on several hosts (--iter-range) and joined with --merge.  Imports
only ``oracle`` and ``workload``: no value here comes from the CUDA path.

    python tools/make_golden_digests.py [--configs 1 2 3 4 5 6] [--chunk 8] [--threads 0]
    python tools/make_golden_digests.py --configs 5 --iter-range 0 8 --out DIR   # then --merge
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
    ap.add_argument("--cfg5-iters", type=int, default=16)
    ap.add_argument("--cfg5-cands", type=int, default=16384)
    ap.add_argument("--out", default=GOLDEN, help="output directory")
    ap.add_argument("--iter-range", type=int, nargs=2, default=None,
                    help="only iterations [T0, T1): writes digests_cfgN_tT0-T1.npz (joined by --merge)")
    ap.add_argument("--merge", action="store_true", help="join the digests_cfgN_t*.npz parts in --out")
    args = ap.parse_args()
    if args.merge:
        for cfg in args.configs:
            merge(args.out, cfg)
        return
    oracle.build()
    for cfg in args.configs:
        W = w.make_workload(cfg)
        It = min(W.n_iter, args.cfg5_iters) if cfg == 5 else W.n_iter
        if cfg == 5:
            W = w.Workload(W.cfg, W.name, W.lengths, W.schemes, W.cand[: args.cfg5_cands].copy(),
                           W.cand_np[: args.cfg5_cands].copy(), W.k_pad, meta=W.meta)
        T0, T1 = (0, It) if args.iter_range is None else (args.iter_range[0], min(args.iter_range[1], W.n_iter))
        parts, status = [], 0
        t_start = time.time()
        for t0 in range(T0, T1, args.chunk):
            t1 = min(T1, t0 + args.chunk)
            S = sub_iters(W, t0, t1)
            o = oracle.assign_batch_ragged(S, n_threads=args.threads) if S.ragged else \
                oracle.assign_batch(S, n_threads=args.threads)
            status |= int(o["status"])
            parts.append(iteration_digests(o, t1 - t0, offsets=S.offsets))
            print(f"cfg{cfg}: iterations {t1}/{T1}, {time.time() - t_start:.0f} s", flush=True)
        dig = {k: np.concatenate([p[k] for p in parts]) for k in parts[0]}
        os.makedirs(args.out, exist_ok=True)
        whole = (T0, T1) == (0, It)
        path = os.path.join(args.out, f"digests_cfg{cfg}.npz" if whole else f"digests_cfg{cfg}_t{T0}-{T1}.npz")
        np.savez_compressed(path, n_iter=np.int64(T1 - T0), t0=np.int64(T0), n_cand=np.int64(W.n_cand), status=np.int64(status),
                            n_cand_total=np.int64(w.CONFIGS[cfg]["C"]),
                            workload=np.array(W.name), seed=np.int64(W.meta.get("seed", -1)), **dig)
        print(f"wrote {path}: {T1 - T0} iterations x {W.n_cand} candidates, status {status}, "
              f"{time.time() - t_start:.0f} s", flush=True)


def merge(out, cfg):
    """Join per-range parts (each written above from the oracle) into digests_cfgN.npz; the parts
    must tile [0, T) with the same workload and candidate count."""
    import glob

    parts = sorted((np.load(f) for f in glob.glob(os.path.join(out, f"digests_cfg{cfg}_t*.npz"))),
                   key=lambda g: int(g["t0"]))
    assert parts, f"no parts for config {cfg} in {out}"
    t = 0
    for g in parts:
        assert int(g["t0"]) == t, f"gap at iteration {t}"
        t += int(g["n_iter"])
        for k in ("workload", "n_cand", "n_cand_total", "seed"):
            assert parts[0][k] == g[k], k
    meta = ("n_iter", "t0", "n_cand", "status", "n_cand_total", "workload", "seed")
    dig = {k: np.concatenate([g[k] for g in parts]) for k in parts[0].files if k not in meta}
    status = int(np.bitwise_or.reduce([int(g["status"]) for g in parts]))
    path = os.path.join(out, f"digests_cfg{cfg}.npz")
    np.savez_compressed(path, n_iter=np.int64(t), t0=np.int64(0), n_cand=parts[0]["n_cand"], status=np.int64(status),
                        n_cand_total=parts[0]["n_cand_total"], workload=parts[0]["workload"],
                        seed=parts[0]["seed"], **dig)
    print(f"wrote {path}: {t} iterations from {len(parts)} parts", flush=True)


if __name__ == "__main__":
    main()
