#!/usr/bin/env python
"""Benchmark of the Hydraulis two-stage data assignment on B200.

Metric (BASELINE.json): candidate-iteration assignments per second -- one c-i is one
complete pipe + mb + ptime + makespan row for one (candidate, iteration) pair followed by
the per-iteration selection.  A step is one pass of the whole hot path a1-a6 over the
configuration's batch: sort + cost table, dispatch, pack, select, and (N > 1) the NCCL
allreduce-min of the keys.  Default workload: BASELINE config 4 (512 seqs x 1024 iterations
x 4096 candidates, LLaMA-70B-shaped cost models), strong-scaled over N GPUs by candidate.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]
  N > 1: python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workload as wl  # noqa: E402

METRIC = "candidate-iteration assignments/sec"
UNIT = "c-i/s"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=30.0, help="target CPU time of the oracle sample")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no e2e/cpu/clocks)")
    ap.add_argument("--trials", type=int, default=0,
                    help="NEXT-1: stage 1 = Alg. 1 with this many random trials per (c,t) (0: HYD-H1 dispatch)")
    ap.add_argument("--seed", type=int, default=2024, help="Alg. 1 permutation seed")
    ap.add_argument("--candidates", type=int, default=0, help="diagnostics: first N candidates only (0: all)")
    ap.add_argument("--gap", action="store_true",
                    help="NEXT-4: exact Eq. 3 optimum (branch-and-bound) vs the heuristics on B-sequence iterations")
    ap.add_argument("--gap-batch", type=int, default=20, help="--gap: sequences per iteration (<= 64)")
    ap.add_argument("--gap-cands", type=int, default=4096, help="--gap: candidates (config 4's first N)")
    ap.add_argument("--gap-iters", type=int, default=64, help="--gap: iterations")
    ap.add_argument("--gap-nodes", type=int, default=1 << 22, help="--gap: node budget per instance")
    ap.add_argument("--gap-no-eq1", action="store_true", help="--gap: skip the Eq. 1 packing study")
    ap.add_argument("--dp", action="store_true",
                    help="NEXT-3: time the strategy-proposal DP on the paper's grid (64 GPUs, 0.1 steps, 128-token "
                         "buckets to 32K) instead of the assignment path")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def newest_profile(name):
    """Newest committed profiles/rNN/<name> (rounds sort lexically), else None."""
    import glob

    paths = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", name)))
    return paths[-1] if paths else None


def alu_peak(pk, how):
    """Integer-instruction issue ceiling in G thread-instructions/s: the measured LPT-mix
    microbenchmark (tools/int_peak.py -> profiles/rNN/int_peak.json), else the nominal
    148 SM x 128 lanes x clock, saying which."""
    p = newest_profile("int_peak.json")
    if p:
        try:
            d = json.load(open(p))
            return float(d["peak_gops"]), f"measured: {os.path.relpath(p, ROOT)} ({d.get('peak_kind', 'mix')})"
        except Exception:
            pass
    sm_mhz = float(pk.get("sm_max_mhz", 1965.0))
    return 148 * 128 * sm_mhz * 1e6 / 1e9, f"nominal 148 SM x 128 INT32 lanes x {sm_mhz:.0f} MHz ({how} clock)"


def alg_evals_per_ci(cfg):
    """SURVEY §8(d) algorithmic pack work per c-i for this config (tools/alg_evals.py, oracle only)."""
    p = newest_profile("alg_evals.json")
    if not p:
        return None, None
    try:
        d = json.load(open(p))["configs"][str(cfg)]
        return float(d["evals_per_ci"]), os.path.relpath(p, ROOT)
    except Exception:
        return None, None


def cpu_info():
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.p = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_gpu{gpu_index}.csv")

    def start(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


def sub_workload(W, its, cs):
    """Iterations ``its`` x candidates ``cs`` of W (ragged workloads keep their CSR layout)."""
    if not W.ragged:
        return wl.Workload(W.cfg, W.name, W.lengths[its], W.schemes, W.cand[cs], W.cand_np[cs], W.k_pad)
    rows = [W.iteration(int(t)) for t in its]
    off = np.concatenate([[0], np.cumsum([r.size for r in rows])]).astype(np.uint32)
    return wl.Workload(W.cfg, W.name, np.concatenate(rows).astype(np.uint32), W.schemes, W.cand[cs], W.cand_np[cs],
                       W.k_pad, offsets=off)


def run_oracle(W, n_threads=0, **kw):
    import oracle

    if W.ragged:
        return oracle.assign_batch_ragged(W, n_threads=n_threads)
    return oracle.assign_batch(W, n_threads=n_threads, **kw)


# ----------------------------------------------------------------------------- CPU oracle leg
def oracle_sample(W, target_s, rng_seed=0, max_cand=None, trials=0, seed=0):
    """Time the oracle (as it stands) on a bounded slice of W: a1-a5 for C' candidates x It'
    iterations, sized from a calibration run to about ``target_s`` seconds of CPU time."""
    import oracle

    oracle.build()
    rng = np.random.default_rng(rng_seed)
    ncal, ical = min(W.n_cand, 4 * (os.cpu_count() or 4)), min(2, W.n_iter)
    its = np.sort(rng.choice(W.n_iter, ical, replace=False))
    sub = sub_workload(W, its, np.arange(ncal))
    t0 = time.perf_counter()
    run_oracle(sub, **({"trials": trials, "seed": seed} if trials else {}))
    per = (time.perf_counter() - t0) / (ncal * ical)  # wall seconds per c-i on all host threads
    want = max(1, int(target_s / max(per, 1e-9)))  # c-i in the sample
    cap = W.n_cand if max_cand is None else min(max_cand, W.n_cand)
    nc = max(1, min(cap, want))
    n_it = max(1, min(W.n_iter, -(-want // nc)))
    cs = np.sort(rng.choice(W.n_cand, nc, replace=False))
    its = np.sort(rng.choice(W.n_iter, n_it, replace=False))
    sub = sub_workload(W, its, cs)
    t0 = time.perf_counter()
    run_oracle(sub, **({"trials": trials, "seed": seed} if trials else {}))
    dt = time.perf_counter() - t0
    cores = os.cpu_count() or 1
    # the same oracle on ONE thread, on a slice of the sample sized to about a quarter of target_s
    per1 = dt * min(cores, nc) / (nc * n_it)  # ~ seconds per c-i on one thread
    n1 = max(1, min(nc, int(0.25 * target_s / max(per1, 1e-9))))
    sub1 = sub_workload(W, its[:1], cs[:n1])
    t1 = time.perf_counter()
    run_oracle(sub1, n_threads=1, **({"trials": trials, "seed": seed} if trials else {}))
    dt1 = time.perf_counter() - t1
    return {
        "value": (nc * n_it) / dt,
        "unit": UNIT,
        "cores": min(cores, nc),
        "kind": "oracle",
        "sample": f"{nc} candidates x {n_it} iterations of cfg{W.cfg} ({nc * n_it} c-i, steps a1-a5"
                  + (f", Alg. 1 with {trials} trials" if trials else "") + f"), {dt:.1f} s on {min(cores, nc)} threads",
        "value_1thread": n1 / dt1,
        "sample_1thread": f"{n1} candidates x 1 iteration ({n1} c-i) on 1 thread, {dt1:.1f} s",
        **cpu_info(),
        "seconds": dt,
    }


def run_reference(args):
    world, rank, _ = dist_env()
    if world > 1 and rank != 0:
        return 0
    W = wl.make_workload(args.config)
    import oracle

    oracle.build()
    rng = np.random.default_rng(1)
    per_step = 64  # candidates per step (x 2 iterations): a bounded sample of the workload
    times = []
    for s in range(args.warmup + args.steps):
        its = np.sort(rng.choice(W.n_iter, 2, replace=False))
        cs = np.sort(rng.choice(W.n_cand, per_step, replace=False))
        sub = sub_workload(W, its, cs)
        t0 = time.perf_counter()
        run_oracle(sub)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
    ms = 1000.0 * float(np.mean(times))
    val = (per_step * 2) / (ms / 1000.0)
    cores = os.cpu_count() or 1
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": val,
        "unit": UNIT,
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "int64",
        "data": "synthetic",
        "config": {"workload": W.name, "sample_per_step": f"{per_step} candidates x 2 iterations"},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": min(cores, per_step), "kind": "oracle",
                         "sample": f"{per_step} random candidates x 2 random iterations of cfg{W.cfg} per step",
                         **cpu_info()},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU leg
def dp_transitions(schemes, step, J, n_gpus, scale):
    """Algorithmic (k, d, l') transitions the DP evaluates: sum over states (n, l)."""
    g = [int(s["tp"]) * int(s["pp"]) * int(s["cp"]) for s in schemes]
    ml = [int(s["max_len"]) for s in schemes]
    NV = n_gpus * scale
    tot = 0
    for j in range(1, J + 1):
        ks = [k for k in range(len(schemes)) if ml[k] >= j * step]
        per_nu = sum(sum(nu // g[k] for k in ks) for nu in range(1, NV + 1))
        tot += per_nu * j
    return tot


def run_gap(args):
    """NEXT-4 bench line: exact Eq. 3 optima at scale and the heuristics' gap."""
    import torch

    from paper_2412_07894_b200 import assign, hyd

    B, It, Cn, node_limit = args.gap_batch, args.gap_iters, args.gap_cands, args.gap_nodes
    base = wl.make_workload(4, n_cand=Cn, n_iter=1)
    rng = np.random.default_rng(2024)
    L = wl.lengths_lognormal(rng, It * B, hi=32768).reshape(It, B)
    W = wl.Workload(0, f"gap-{B}seq", L, base.schemes, base.cand, base.cand_np, base.k_pad)
    Ld = assign.lengths_to_device(L)
    A = assign.Assigner(W.schemes, W.cand, W.cand_np, It, B, W.k_pad)
    A1 = assign.Assigner(W.schemes, W.cand, W.cand_np, It, B, W.k_pad, trials=100, seed=args.seed)
    pc = np.repeat(np.arange(Cn), It).astype(np.int32)
    pt = np.tile(np.arange(It), Cn).astype(np.int32)
    for _ in range(max(1, args.warmup)):
        A.eq3_exact(Ld, pc[:256], pt[:256], node_limit)
    torch.cuda.synchronize()
    l0 = hyd.kernel_launches()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    val, pipe, nodes, proved = A.eq3_exact(Ld, pc, pt, node_limit)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    launches = hyd.kernel_launches() - l0
    A.run(Ld)
    A1.run(Ld)
    lb = A.numpy()["lb"][pc, pt]
    lb1 = A1.numpy()["lb"][pc, pt]
    feas = (val != np.uint64(2**64 - 1)) & proved
    opt = val[feas].astype(np.float64)
    r_h1 = lb[feas].astype(np.float64) / opt
    r_a1 = lb1[feas].astype(np.float64) / opt
    # Alg. 1's O_max ties (reading 22): how often a trial's pick had more than one
    # pipeline at the minimal O_max is not observable here; the ratio distribution is reported
    q = lambda r, p: float(np.quantile(r, p)) if r.size else None
    line_gap_extra = {"hyd_h1_p99_ratio": q(r_h1, 0.99), "alg1_T100_p50_ratio": q(r_a1, 0.5),
                      "alg1_T100_p99_ratio": q(r_a1, 0.99)}
    if args.gap_no_eq1:
        line = {
            "metric": "exact Eq. 3 instances/sec", "value": pc.size / (ms / 1000.0), "unit": "instances/s",
            "n_gpus": 1, "steps": 1, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": f"NEXT-4 gap study: config-4 schemes and first {Cn} candidates (8 pipelines), "
                                   f"{B}-sequence lognormal iterations (cfg6 corpus shape, 32K context)",
                       "instances": int(pc.size), "node_limit": node_limit, "batch": B},
            "gap": {"proved_fraction": float(proved[val != np.uint64(2**64 - 1)].mean()),
                    "proved_instances": int(feas.sum()),
                    "hyd_h1_within_10pct": float((r_h1 <= 1.10).mean()), "hyd_h1_mean_ratio": float(r_h1.mean()),
                    "hyd_h1_max_ratio": float(r_h1.max()),
                    "alg1_T100_within_10pct": float((r_a1 <= 1.10).mean()), "alg1_T100_mean_ratio": float(r_a1.mean()),
                    "alg1_T100_max_ratio": float(r_a1.max()), **line_gap_extra,
                    "nodes_mean": float(nodes.astype(np.float64).mean()), "nodes_max": int(nodes.max())},
            "gpu_launches": int(launches),
        }
        print(json.dumps(line), flush=True)
        return 0
    # Eq. 1 (packing) at scale: 64-sequence iterations, candidates cut to their first 4
    # pipelines (~16 sequences per pipeline), the HYD-H1 dispatch's pipelines packed exactly
    B1, It1, C1 = 64, 16, 1024
    L1 = wl.lengths_lognormal(np.random.default_rng(2025), It1 * B1, hi=32768).reshape(It1, B1)
    cand1 = base.cand[:C1].copy()
    np1 = np.minimum(base.cand_np[:C1], 4).astype(np.uint8)
    for c in range(C1):
        cand1[c, np1[c]:] = 0xFF
    A2 = assign.Assigner(base.schemes, cand1, np1, It1, B1, base.k_pad, fused=False)  # eq1_exact reads members
    A2.run(assign.lengths_to_device(L1))
    g2 = A2.numpy()
    pc2, pt2, pj2 = [], [], []
    for c in range(C1):
        for t in range(It1):
            if g2["makespan"][t, c] != np.uint64(2**64 - 1):
                for j in range(int(np1[c])):
                    pc2.append(c), pt2.append(t), pj2.append(j)
    a2, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a2.record()
    v1, o1, n1, p1 = A2.eq1_exact(pc2, pt2, pj2, node_limit=1 << 22)
    b2.record()
    torch.cuda.synchronize()
    ms1 = a2.elapsed_time(b2)
    pc2, pt2, pj2 = np.array(pc2), np.array(pt2), np.array(pj2)
    heur = g2["ptime"][pc2, pt2, pj2]
    nz = p1 & (o1 > 0) & (v1 > 0)
    r_pack = heur[nz].astype(np.float64) / o1[nz].astype(np.float64)
    # two-stage: makespan with exact packing of the same dispatch vs the heuristic's
    exact_ms = np.zeros((It1, C1), np.float64)
    np.maximum.at(exact_ms, (pt2[p1], pc2[p1]), o1[p1].astype(np.float64))
    okpair = np.ones((It1, C1), bool)
    np.logical_and.at(okpair, (pt2, pc2), p1)
    feas2 = (g2["makespan"] != np.uint64(2**64 - 1)) & okpair
    r_ms = g2["makespan"][feas2].astype(np.float64) / exact_ms[feas2]
    line = {
        "metric": "exact Eq. 3 instances/sec", "value": pc.size / (ms / 1000.0), "unit": "instances/s", "n_gpus": 1,
        "steps": 1, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": "NEXT-4 gap study: config-4 schemes and candidates (8 pipelines), 20-sequence "
                               "lognormal iterations", "instances": int(pc.size), "node_limit": node_limit},
        "gap": {"proved_fraction": float(proved[val != np.uint64(2**64 - 1)].mean()),
                "hyd_h1_within_10pct": float((r_h1 <= 1.10).mean()), "hyd_h1_mean_ratio": float(r_h1.mean()),
                "hyd_h1_max_ratio": float(r_h1.max()),
                "alg1_T100_within_10pct": float((r_a1 <= 1.10).mean()), "alg1_T100_mean_ratio": float(r_a1.mean()),
                "alg1_T100_max_ratio": float(r_a1.max()),
                "nodes_mean": float(nodes.astype(np.float64).mean()), "nodes_max": int(nodes.max())},
        "eq1_gap": {"pipelines": int(pc2.size), "ms": ms1, "proved_fraction": float(p1.mean()),
                    "lpt_within_10pct": float((r_pack <= 1.10).mean()), "lpt_mean_ratio": float(r_pack.mean()),
                    "lpt_max_ratio": float(r_pack.max()), "makespan_mean_ratio_vs_exact_packing": float(r_ms.mean()),
                    "makespan_within_10pct": float((r_ms <= 1.10).mean()),
                    "workload": "64-sequence lognormal iterations x 1024 candidates cut to 4 pipelines"},
        "gpu_launches": int(launches),
    }
    print(json.dumps(line), flush=True)
    return 0


def dp_probes(schemes, step, J, n_gpus, scale):
    """(k, d) pairs the GPU evaluates, each by two binary searches over l' (~2 log2 j + 2 probes)."""
    import math

    g = [int(s["tp"]) * int(s["pp"]) * int(s["cp"]) for s in schemes]
    ml = [int(s["max_len"]) for s in schemes]
    NV = n_gpus * scale
    tot = 0
    for j in range(1, J + 1):
        ks = [k for k in range(len(schemes)) if ml[k] >= j * step]
        pairs = sum(sum(nu // g[k] for k in ks) for nu in range(1, NV + 1))
        tot += pairs * (2 * math.ceil(math.log2(j + 1)) + 2)
    return tot


def run_dp(args):
    """NEXT-3 bench line: one proposal = histogram + DP over the whole grid + strategies + rounding."""
    import torch

    from paper_2412_07894_b200 import assign, hyd

    W = wl.make_workload(6, n_cand=2, n_iter=1024)  # 100K-token iterations: a 1024-iteration length sample
    lens = np.ascontiguousarray(W.lengths)
    step, J, N, scale = 128, 256, 64, 10
    P = assign.Proposer(W.schemes, step, J, N, scale)
    L = assign.lengths_to_device(lens)
    for _ in range(args.warmup):
        P.run(L)
    torch.cuda.synchronize()
    clk = ClockSampler(0)
    clk.start()
    time.sleep(0.3)
    l0 = hyd.kernel_launches()
    evs = []
    for _ in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        P.run(L)
        b.record()
        evs.append((a, b))
    torch.cuda.synchronize()
    launches = hyd.kernel_launches() - l0
    clocks = clk.stop()
    ms = float(np.mean([a.elapsed_time(b) for a, b in evs]))
    trans = dp_transitions(W.schemes, step, J, N, scale)
    sel, cand, cnp = P.candidates()
    # oracle on a coarser grid (CPU minutes otherwise): same code, 1-GPU steps
    cpu = None
    if not args.no_cpu:
        import oracle

        oracle.build()
        t0 = time.perf_counter()
        oracle.dp_propose(lens, W.schemes, step, J, N, 1)
        dt = time.perf_counter() - t0
        ct = dp_transitions(W.schemes, step, J, N, 1)
        cpu = {"value": ct / dt, "unit": "transitions/s", "cores": 1, "kind": "oracle",
               "sample": f"integer DP (scale 1) on the same lengths and length grid, {ct} transitions in {dt:.1f} s"}
    pk, how = peaks()
    alu, alu_src = alu_peak(pk, how)
    probes = dp_probes(W.schemes, step, J, N, scale)
    ops = 24.0 * probes  # ~24 int ops per probe (two 64x64->128 products, compares)
    achieved = ops / (ms / 1000.0) / 1e9
    line = {
        "metric": "strategy-proposal DP transitions/sec", "value": trans / (ms / 1000.0), "unit": "transitions/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int64 (exact rationals, 128-bit products)",
        "data": "synthetic",
        "config": {"workload": "NEXT-3 proposal DP, cfg6 length sample", "n_sequences": int(lens.size),
                   "length_step": step, "buckets": J, "gpus": N, "gpu_step": 1 / scale, "transitions": trans,
                   "probes_evaluated": probes,
                   "proposed_candidates": int(len(sel))},
        "roofline": {"kernel": "k_dp_solve", "bound": "alu", "achieved": achieved, "peak": alu, "unit": "Gop/s",
                     "frac": achieved / alu, "traffic": None, "peak_source": alu_src},
        "gpu_launches": int(launches), "clocks": clocks,
    }
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.dp:
        return run_dp(args)
    if args.gap:
        return run_gap(args)
    import torch
    import torch.distributed as dist

    from paper_2412_07894_b200 import assign, hyd

    world, rank, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    W = wl.make_workload(args.config, n_cand=args.candidates or None)
    sh = assign.plan_shard(W.n_cand, W.n_iter, world, rank)
    cand = W.cand[sh.cand_lo:sh.cand_hi]
    cand_np = W.cand_np[sh.cand_lo:sh.cand_hi]
    if W.ragged:  # NEXT-2: token-budget batches; ranks split candidates only
        assert sh.by != "iter", "ragged workloads shard by candidates"
        lens = W.lengths
        It_local = W.n_iter
        A_rows = [W.iteration(t) for t in range(W.n_iter)]
    else:
        lens = W.lengths[sh.iter_lo:sh.iter_hi]
        It_local = lens.shape[0]
        A_rows = lens
    C_local = cand.shape[0]
    A = assign.Assigner(W.schemes, cand, cand_np, It_local, W.batch, W.k_pad, cand_offset=sh.cand_lo, device=dev,
                        trials=args.trials, seed=args.seed, offsets=W.offsets if W.ragged else None)
    len_dev = assign.lengths_to_device(lens, dev)
    A._lens_host = A_rows
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2

    names = ["sort_cost", "dispatch", "pack", "select", "allreduce"]

    def step(evs=None):
        It, B, K, kp, Cn = A.n_iter, A.batch, A.n_schemes, A.k_pad, A.n_cand
        if evs:
            evs[0].record(stream)
        if A.ragged:
            N = A.n_total
            hyd.cost_table_ragged(len_dev, It, A.off, N, B, A.schemes, K, kp, A.sorted_len, A.perm, A.cost, A.status)
            if evs:
                evs[1].record(stream)
            if A.fused:  # a3 + a4 in one kernel (timed as "pack"; "dispatch" is empty)
                if evs:
                    evs[2].record(stream)
                hyd.dispatch_pack_ragged(A.sorted_len, A.cost, It, A.off, N, B, kp, A.schemes, K, A.cand, A.cand_np,
                                         Cn, A.max_np, A.pipe, A.lb, A.mb, A.v, A.ptime, A.makespan, A.status,
                                         A.small_ws)
            else:
                hyd.dispatch_ragged(A.sorted_len, A.cost, It, A.off, N, B, kp, A.schemes, K, A.cand, A.cand_np, Cn,
                                    A.max_np, A.pipe, A.lb, A.stats, A.members, A.status, A.disp_ws)
                if evs:
                    evs[2].record(stream)
                hyd.pack_ragged(A.sorted_len, A.cost, It, A.off, N, B, kp, A.schemes, K, A.cand, A.cand_np, Cn,
                                A.max_np, A.pipe, A.stats, A.members, A.mb, A.v, A.ptime, A.makespan, A.status, A.ws)
            if evs:
                evs[3].record(stream)
            hyd.select_best(A.makespan, It, Cn, A.cand_offset, A.key, A.status)
            if evs:
                evs[4].record(stream)
            if sh.needs_reduce:
                assign.reduce_keys(A.key)
            if evs:
                evs[5].record(stream)
            return
        hyd.cost_table(len_dev, It, B, A.schemes, K, kp, A.sorted_len, A.perm, A.cost, A.status)
        if evs:
            evs[1].record(stream)
        if A.fused:  # a3 + a4 in one kernel (timed as "pack"; "dispatch" is empty)
            if evs:
                evs[2].record(stream)
            hyd.dispatch_pack(A.sorted_len, A.cost, It, B, kp, A.schemes, K, A.cand, A.cand_np, Cn, A.max_np, A.pipe,
                              A.lb, A.mb, A.v, A.ptime, A.makespan, A.status, A.small_ws)
            if evs:
                evs[3].record(stream)
            hyd.select_best(A.makespan, It, Cn, A.cand_offset, A.key, A.status)
            if evs:
                evs[4].record(stream)
            if sh.needs_reduce:
                assign.reduce_keys(A.key)
            if evs:
                evs[5].record(stream)
            return
        if A.trials:  # NEXT-1: Alg. 1 (permutations drawn every step, as Alg. 1 line 2 does)
            hyd.alg1_permutations(A.seed, It, B, A.trials, A.order)
            hyd.dispatch_alg1(A.sorted_len, A.cost, It, B, kp, A.schemes, K, A.cand, A.cand_np, Cn, A.max_np,
                              A.trials, A.order, A.best, A.pipe, A.lb, A.stats, A.members, A.status, A.alg1_ws)
        else:
            hyd.dispatch(A.sorted_len, A.cost, It, B, kp, A.schemes, K, A.cand, A.cand_np, Cn, A.max_np, A.pipe,
                         A.lb, A.stats, A.members, A.status, A.disp_ws)
        if evs:
            evs[2].record(stream)
        hyd.pack(A.sorted_len, A.cost, It, B, kp, A.schemes, K, A.cand, A.cand_np, Cn, A.max_np, A.pipe, A.stats,
                 A.members, A.mb, A.v, A.ptime, A.makespan, A.status, A.ws)
        if evs:
            evs[3].record(stream)
        hyd.select_best(A.makespan, It, Cn, A.cand_offset, A.key, A.status)
        if evs:
            evs[4].record(stream)
        if sh.needs_reduce:
            assign.reduce_keys(A.key)
        if evs:
            evs[5].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(dev.index) if not args.profile else None
    if clk:
        clk.start()
        time.sleep(0.3)
    per_step = []
    per_kernel = np.zeros(len(names))
    l0 = hyd.kernel_launches()
    for _ in range(args.steps):
        flush.zero_()  # L2 flush outside the timed events
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        step(evs)
        per_step.append(evs)
    torch.cuda.synchronize()
    launches = hyd.kernel_launches() - l0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = clk.stop() if clk else None
    step_ms = []
    for evs in per_step:
        step_ms.append(evs[0].elapsed_time(evs[5]))
        per_kernel += np.array([evs[i].elapsed_time(evs[i + 1]) for i in range(5)])
    ms_local = float(np.sum(step_ms)) / args.steps
    per_kernel /= args.steps
    t = torch.tensor([ms_local], dtype=torch.float64, device=dev)
    rank_ms = [ms_local]
    if world > 1:
        allt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        rank_ms = [float(x.item()) for x in allt]
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    total_ci = W.n_cand * W.n_iter
    value = total_ci / (ms / 1000.0)
    bits = A.status_bits()
    if bits:
        print(f"WARNING: device status {hyd.status_names(bits)}", file=sys.stderr)

    # ---- roofline of the dominant kernel (largest share of the step)
    pk, how = peaks()
    dom = int(np.argmax(per_kernel[:4]))
    roof = roofline(names[dom], per_kernel[dom], W, A, pk, how, local_ci=C_local * It_local, world=world)

    # ---- end-to-end through the public host-buffer API (hyd_assign_host)
    e2e, H = None, None
    if not args.no_e2e and not args.profile and not args.trials:  # hyd_assign_host runs HYD-H1 only
        e2e, H = run_e2e(args, W, sh, cand, cand_np, lens, world, dev)

    # ---- a6 on hardware (N > 1, outside the timed region): reduced keys and every rank's winner
    #      rows against a one-rank run over all candidates
    a6 = None
    if world > 1 and not args.profile and not args.trials:
        a6 = verify_multi(W, sh, A, H, world, rank, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and not args.profile:
        cpu = oracle_sample(W, args.cpu_seconds, trials=args.trials, seed=args.seed)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value,
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "int64",
            "data": "synthetic",
            "config": {
                "workload": W.name,
                "batch": (f"ragged: mean {W.n_total / W.n_iter:.1f}, max {W.batch} sequences "
                          f"({W.meta.get('tokens_per_iteration')} tokens/iteration)") if W.ragged else W.batch,
                "pipelines": int(W.cand_np.max()),
                "candidates": W.n_cand,
                "iterations": W.n_iter,
                "c_i_per_step": total_ci,
                "shard": sh.by,
                "parallelism": f"candidates/{world}" if sh.by == "cand" else (f"iterations/{world}" if sh.by == "iter" else "single"),
                "l2": "flushed: 256 MiB memset between steps, outside the timed events",
                "cost_model": W.meta.get("model"),
                "stage1": f"Alg. 1, {args.trials} random trials (NEXT-1)" if args.trials else "HYD-H1 LPT dispatch",
                "kernels": "a3+a4 fused (hyd_dispatch_pack, batch <= 128)" if A.fused else "hyd_dispatch + hyd_pack",
            },
            "kernel_ms": {n: float(x) for n, x in zip(names, per_kernel)},
            "rank_ms": rank_ms,
            "roofline": roof,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "status": hyd.status_names(bits),
        }
        if e2e is not None:
            line["e2e"] = e2e
        if a6 is not None:
            line["a6_check"] = a6
        if cpu is not None:
            line["cpu_baseline"] = {k: v for k, v in cpu.items() if k != "seconds"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if a6 is not None and not (a6["keys_equal_one_rank"] and a6["winner_rows_equal_one_rank"]):
        print("ERROR: multi-GPU result differs from the one-rank run", file=sys.stderr)
        return 3
    return 0


def verify_multi(W, sh, A, H, world, rank, dev):
    """Rank 0 runs the whole workload on one GPU; every rank compares its reduced keys (device
    path) and its hyd_assign_host outputs (keys + winner rows of every iteration it holds)."""
    import torch
    import torch.distributed as dist

    from paper_2412_07894_b200 import assign

    offs = W.offsets if W.ragged else None
    ref = None
    if rank == 0:
        F = assign.Assigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad, device=dev, offsets=offs)
        F.run(assign.lengths_to_device(W.lengths, dev))
        ref = {"key": F.key.cpu().numpy()}
        del F
        torch.cuda.empty_cache()
        if H is not None:
            HF = assign.HostAssigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad, offsets=offs)
            HF(torch.from_numpy(np.ascontiguousarray(W.lengths).view(np.int32)).pin_memory())
            for k in ("win_pipe", "win_mb", "win_v", "win_ptime"):
                ref[k] = getattr(HF, k).numpy().copy()
            assert np.array_equal(HF.key.numpy(), ref["key"])
            del HF
            torch.cuda.empty_cache()
    obj = [ref]
    dist.broadcast_object_list(obj, src=0)
    ref = obj[0]
    lo, hi = sh.iter_lo, sh.iter_hi
    keys_ok = bool(np.array_equal(A.key.cpu().numpy(), ref["key"][lo:hi]))
    rows_ok = True
    if H is not None:
        rows_ok = bool(np.array_equal(H.key.numpy(), ref["key"][lo:hi]))
        for k in ("win_pipe", "win_mb", "win_v", "win_ptime"):
            # ragged rows are [N_total] (candidate shards only: every rank holds every iteration)
            want = ref[k] if (W.ragged and k in ("win_pipe", "win_mb")) else ref[k][lo:hi]
            rows_ok = rows_ok and bool(np.array_equal(getattr(H, k).numpy(), want))
    flags = torch.tensor([int(keys_ok), int(rows_ok)], dtype=torch.int32, device=dev)
    dist.all_reduce(flags, op=dist.ReduceOp.MIN)
    return {"keys_equal_one_rank": bool(flags[0].item()), "winner_rows_equal_one_rank": bool(flags[1].item()),
            "ranks": world, "checked": "outside the timed region: device-path keys after the last step and the "
                                      "e2e call's keys + win_pipe/win_mb/win_v/win_ptime on every rank vs rank 0's "
                                      "one-GPU run over all candidates"}


def ncu_traffic(cfg, prefix):
    """DRAM bytes per launch of the kernels named ``prefix*`` from the newest committed
    `ncu --set full` summary of this config (profiles/rNN/ncu_cfgX_summary.json), else None."""
    import glob

    paths = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", f"ncu_cfg{cfg}_summary.json")))
    if not paths:
        return None, None
    try:
        d = json.load(open(paths[-1]))
        tot = sum(e["dram_bytes"] for e in d.get("full_capture", [])
                  if any(e["kernel"].replace("void ", "").startswith(p) for p in prefix) and e.get("dram_bytes"))
        return (tot or None), os.path.relpath(paths[-1], ROOT)
    except Exception:
        return None, None


def roofline(name, ms, W, A, pk, how, local_ci, world=1):
    """Algorithmic work per launch / CUDA-event duration."""
    B, D = (W.n_total / W.n_iter if W.ragged else W.batch), int(W.cand_np.max())
    alu, alu_src = alu_peak(pk, how)
    hbm = float(pk.get("hbm_gbs", 6650.0))
    if name == "pack":
        cnt = A.pack_counters()
        ops_exec = 6.0 * cnt["bin_evals"]  # ~6 int32 instructions per executed (item, bin) evaluation
        per_ci, alg_src = alg_evals_per_ci(W.cfg)
        ops = 6.0 * per_ci * local_ci if per_ci else ops_exec  # algorithmic: exact pruned search
        if A.fused:  # the fused kernel also does the dispatch: its evaluations count too
            dev_ops = 6.0 * A.dispatch_evals(A._lens_host)
            ops, ops_exec = ops + dev_ops, ops_exec + dev_ops
        achieved = ops / (ms / 1000.0) / 1e9
        traffic, src = ncu_traffic(W.cfg, ("k_assign_small",) if A.fused else ("k_pack_", "k_flag_list"))
        if world > 1:  # the committed ncu capture is of the N = 1 launch: not this shard's
            traffic, src = None, "n/a at N > 1 (ncu captures are single-GPU)"
        return {"kernel": "dispatch + pack fused (k_assign_small)" if A.fused else "pack (k_pack_lanes + k_pack_big)",
                "bound": "alu", "achieved": achieved,
                "peak": alu, "unit": "Gop/s", "frac": achieved / alu,
                "frac_executed": ops_exec / (ms / 1000.0) / 1e9 / alu,
                "traffic": traffic,
                "traffic_unit": "bytes/launch (dram read+write, ncu --set full)", "traffic_source": src,
                "algorithmic_bytes_per_launch": local_ci * (3 * B + 10 * D + 8),
                "algorithmic_ops_per_launch": ops, "algorithmic_evals_per_ci": per_ci,
                "algorithmic_source": alg_src or "none: executed evaluations used",
                "executed_ops_per_launch": ops_exec, "bin_evals_per_launch": cnt["bin_evals"],
                "executed_evals_per_ci": cnt["bin_evals"] / max(local_ci, 1),
                "queued_tasks": cnt["queued_tasks"], "handoff": cnt.get("handoff"),
                "hbm_algorithmic_GBps": local_ci * (3 * B + 10 * D + 8) / (ms / 1000.0) / 1e9,
                "hbm_frac_algorithmic": local_ci * (3 * B + 10 * D + 8) / (ms / 1000.0) / 1e9 / hbm,
                "peak_source": alu_src, "ops_model": "6 int32 instructions per (sequence, micro-batch) evaluation"}
    if name == "dispatch":
        ev = A.dispatch_evals(A._lens_host) * max(A.trials, 1)
        ops = (8.0 if A.trials else 6.0) * ev  # int ops per (sequence, feasible pipeline)
        achieved = ops / (ms / 1000.0) / 1e9
        return {"kernel": "dispatch" + (f" (Alg. 1, {A.trials} trials)" if A.trials else ""), "bound": "alu",
                "achieved": achieved, "peak": alu, "unit": "Gop/s",
                "frac": achieved / alu, "traffic": None, "algorithmic_ops_per_launch": ops,
                "peak_source": alu_src}
    byts = {"sort_cost": A.n_iter * B * (4 + 8 + 4 * A.k_pad), "select": A.n_iter * A.n_cand * 8 + 8 * A.n_iter}[name]
    achieved = byts / (ms / 1000.0) / 1e9
    return {"kernel": name, "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": None, "peak_source": how}


def run_e2e(args, W, sh, cand, cand_np, lens, world, dev):
    import torch
    import torch.distributed as dist

    from paper_2412_07894_b200 import assign

    H = assign.HostAssigner(W.schemes, cand, cand_np, W.n_iter if W.ragged else lens.shape[0], W.batch, W.k_pad,
                            cand_offset=sh.cand_lo, offsets=W.offsets if W.ragged else None,
                            reduce=sh.needs_reduce)
    lh = torch.from_numpy(np.ascontiguousarray(lens).view(np.int32)).pin_memory()
    stream = torch.cuda.current_stream()
    for _ in range(max(1, args.warmup)):
        H(lh)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    tot = 0.0
    n = max(1, min(args.steps, 5))
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        H(lh)  # H2D copies, kernels, (allreduce), gather, D2H, stream sync
        b.record(stream)
        b.synchronize()
        tot += a.elapsed_time(b)
    ms = tot / n
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    return {"value": W.n_cand * W.n_iter / (ms / 1000.0), "unit": UNIT,
            "h2d_bytes_per_step": int(lh.numel() * 4 + H.h2d_bytes_fixed), "d2h_bytes_per_step": int(H.d2h_bytes),
            "ms_per_step": ms, "api": ("hyd_assign_host_ragged" if W.ragged else "hyd_assign_host") + " (pinned host buffers)"
            + (", incl. the NCCL key allreduce-MIN and winner-row allreduce-SUM (every rank gets every plan)"
               if sh.needs_reduce else "")}, H


if __name__ == "__main__":
    sys.exit(main())
