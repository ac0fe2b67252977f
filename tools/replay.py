#!/usr/bin/env python
"""Replay dumps of the end-to-end call (SURVEY §5 "Checkpoint / resume": the path is stateless per
batch, so a batch's inputs and outputs dumped to .bin files replay it exactly).

  python tools/replay.py dump DIR --config 4 [--cands 64] [--iters 8]   # run hyd_assign_host, write DIR
  python tools/replay.py check DIR [--oracle]                          # re-run, compare bit for bit

DIR holds lengths.u32 [N] (+ offsets.u32 [It+1] for token-budget batches), schemes.bin (48-byte
hyd_scheme records), cand.u8 [C][32], cand_np.u8 [C], meta.json, and the outputs key.i64,
win_pipe.u8, win_mb.u16, win_v.u16, win_ptime.u64, status.u32.  ``--oracle`` also checks the
keys against the CPU oracle (test infrastructure)."""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workload as w  # noqa: E402

OUTS = (("key", np.int64), ("win_pipe", np.uint8), ("win_mb", np.uint16), ("win_v", np.uint16),
        ("win_ptime", np.uint64), ("status", np.uint32))


def run(W):
    import torch

    from paper_2412_07894_b200 import assign

    H = assign.HostAssigner(W.schemes, W.cand, W.cand_np, W.n_iter, W.batch, W.k_pad,
                            offsets=W.offsets if W.ragged else None)
    lh = torch.from_numpy(np.ascontiguousarray(W.lengths, np.uint32).view(np.int32)).pin_memory()
    H(lh)
    return {k: getattr(H, k).numpy().view(dt).copy() for k, dt in OUTS}


def dump(d, cfg, cands, iters):
    W = w.make_workload(cfg, n_cand=cands, n_iter=iters)
    os.makedirs(d, exist_ok=True)
    np.ascontiguousarray(W.lengths, np.uint32).tofile(os.path.join(d, "lengths.u32"))
    if W.ragged:
        np.ascontiguousarray(W.offsets, np.uint32).tofile(os.path.join(d, "offsets.u32"))
    np.ascontiguousarray(W.schemes).tofile(os.path.join(d, "schemes.bin"))
    W.cand.tofile(os.path.join(d, "cand.u8"))
    W.cand_np.tofile(os.path.join(d, "cand_np.u8"))
    json.dump({"config": cfg, "workload": W.name, "n_iter": W.n_iter, "batch": W.batch, "k_pad": W.k_pad,
               "ragged": W.ragged, "n_cand": W.n_cand}, open(os.path.join(d, "meta.json"), "w"))
    for k, a in run(W).items():
        a.tofile(os.path.join(d, f"{k}.bin"))
    print("dumped", d)


def load(d):
    m = json.load(open(os.path.join(d, "meta.json")))
    lens = np.fromfile(os.path.join(d, "lengths.u32"), np.uint32)
    off = np.fromfile(os.path.join(d, "offsets.u32"), np.uint32) if m["ragged"] else None
    if off is None:
        lens = lens.reshape(m["n_iter"], m["batch"])
    sch = np.fromfile(os.path.join(d, "schemes.bin"), w.SCHEME_DTYPE)
    cand = np.fromfile(os.path.join(d, "cand.u8"), np.uint8).reshape(-1, 32)
    cnp = np.fromfile(os.path.join(d, "cand_np.u8"), np.uint8)
    return w.Workload(m["config"], m["workload"], lens, sch, cand, cnp, m["k_pad"], offsets=off), m


def check(d, use_oracle):
    W, _ = load(d)
    got = run(W)
    for k, dt in OUTS:
        want = np.fromfile(os.path.join(d, f"{k}.bin"), dt).reshape(got[k].shape)
        assert np.array_equal(got[k], want), f"{k} differs from the dump"
    if use_oracle:
        import oracle

        o = oracle.assign_batch_ragged(W) if W.ragged else oracle.assign_batch(W)
        assert np.array_equal(got["key"], o["key"]), "keys differ from the oracle"
    print("REPLAY_OK", d)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["dump", "check"])
    ap.add_argument("dir")
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--cands", type=int, default=64)
    ap.add_argument("--iters", type=int, default=8)
    ap.add_argument("--oracle", action="store_true")
    a = ap.parse_args()
    dump(a.dir, a.config, a.cands, a.iters) if a.mode == "dump" else check(a.dir, a.oracle)


if __name__ == "__main__":
    main()
