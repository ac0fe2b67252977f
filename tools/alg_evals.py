#!/usr/bin/env python
"""Algorithmic work of the pack stage per candidate-iteration: the (sequence,
micro-batch) evaluations the EXACT pruned V search needs, independent of how a kernel schedules
it -- the numerator of bench.py's ALU roofline fraction.  Imports only ``oracle`` and ``workload``.

Per pipeline of a sampled (c, t) pair (HYD-H1 dispatch from the oracle):
  * every V of App. D's range gets LB(V) = max(ceil(sumT / V), tau_max) (PP - 1 + V)
    (<= obj(V), App. E.1's argument);
  * V are evaluated in ascending (LB(V), V) order, each as one full LPT(V) run costing U V
    evaluations, until LB(V) > best or (LB(V) = best and V > V_best) (SURVEY §8(c) "freedom");
  * if no V of the range is feasible, V_hi + 1, V_hi + 2, ... until one is (reading 5).
Writes profiles/r02/alg_evals.json: mean evaluations per c-i per config, with the sample size.

    python tools/alg_evals.py [--pairs 200] [--configs 1 2 3 4 5 6]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import workload as w  # noqa: E402


def pipeline_evals(ell, tau, sch):
    U = len(ell)
    if U == 0:
        return 0, 0
    M, P, UL = int(sch["max_len"]), int(sch["pp"]), int(sch["util_len"])
    S, sumT, tmax = int(sum(ell)), int(sum(tau)), int(tau[0])
    vlo = max(-(-S // M), 1)
    vhi = U if UL == 0 else min(S // UL, U)
    vhi = max(vhi, vlo)
    order = sorted(range(vlo, vhi + 1), key=lambda V: (max(-(-sumT // V), tmax) * (P - 1 + V), V))
    best, vbest, ev, runs = None, None, 0, 0
    for V in order:
        lbv = max(-(-sumT // V), tmax) * (P - 1 + V)
        if best is not None and (lbv > best or (lbv == best and V > vbest)):
            break
        ok, _, mx = oracle.lpt(ell, tau, V, M)
        ev += U * V
        runs += 1
        if ok:
            obj = mx * (P - 1 + V)
            if best is None or obj < best or (obj == best and V < vbest):
                best, vbest = obj, V
    V = vhi + 1
    while best is None and V <= U:
        ok, _, mx = oracle.lpt(ell, tau, V, M)
        ev += U * V
        runs += 1
        if ok:
            best = mx
        V += 1
    return ev, runs


def config_evals(cfg, n_pairs, seed=0):
    W = w.make_workload(cfg)
    rng = np.random.default_rng(seed)
    pc = rng.integers(0, W.n_cand, n_pairs)
    pt = rng.integers(0, W.n_iter, n_pairs)
    tot_ev, tot_runs, n_pipes, feas = 0, 0, 0, 0
    per_pair = []
    for c, t in zip(pc, pt):
        c, t = int(c), int(t)
        lens = W.iteration(t) if W.ragged else W.lengths[t]
        s, _, cst, _ = oracle.cost_table(lens, W.schemes, W.k_pad)
        row = [int(k) for k in W.cand[c, : W.cand_np[c]]]
        ok, pipe, _ = oracle.dispatch(s, cst, W.schemes, row)
        if not ok:
            per_pair.append(0)
            continue
        feas += 1
        ev_pair = 0
        for j, k in enumerate(row):
            idx = np.nonzero(pipe == j)[0]
            ev, runs = pipeline_evals(s[idx], cst[idx, k], W.schemes[k])
            ev_pair += ev
            tot_runs += runs
            n_pipes += 1 if idx.size else 0
        tot_ev += ev_pair
        per_pair.append(ev_pair)
    a = np.array(per_pair, np.float64)
    return {"evals_per_ci": float(a.mean()), "stderr": float(a.std(ddof=1) / math.sqrt(a.size)),
            "runs_per_pipeline": tot_runs / max(n_pipes, 1), "pairs": int(n_pairs), "feasible_pairs": feas,
            "workload": W.name}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pairs", type=int, default=200)
    ap.add_argument("--configs", type=int, nargs="*", default=[1, 2, 3, 4, 5, 6])
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "alg_evals.json"))
    args = ap.parse_args()
    out = {"what": "exact pruned V search, (sequence, micro-batch) evaluations per candidate-iteration "
                   "(tools/alg_evals.py; oracle LPT runs, ascending-LB order, full runs)", "configs": {}}
    for cfg in args.configs:
        n = args.pairs if cfg != 5 else max(8, args.pairs // 10)
        out["configs"][str(cfg)] = config_evals(cfg, n, seed=cfg)
        print(cfg, out["configs"][str(cfg)], flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(out, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
