#!/usr/bin/env python
"""Write configs/cfgN.json: each BASELINE configuration as data -- the integer scheme table
(tp, pp, cp, MaxLen, UtilLen and the Q32 cost coefficients a, b, c of T(l) = floor((a l^2 + b l + c)
/ 2^32)), the candidate table in canonical order, the sizes, the length generator and its seed
(SURVEY §5 "Config / flags").  The lengths themselves are regenerated from the seed by
``workload.make_workload`` (they are hundreds of MB); ``sha256_lengths`` pins them.
``tests/test_configs_cpu.py`` checks every file against ``workload.make_workload``.

    python tools/export_configs.py [--configs 1 2 3 4 5 6]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workload as w  # noqa: E402

GENERATORS = {
    1: "loguniform: floor(128 * 32^u), u ~ U[0,1)",
    2: "lognormal(6.9, 1.2), clamp [1, 32768]",
    3: "Pareto(1.1, x_min 256), clamp [1, 131072]",
    4: "lognormal(6.9, 1.2), clamp [1, 32768]",
    5: "70 % lognormal(6.9, 1.2) + 30 % Pareto(1.1, 256), clamp [64, 262144]",
    6: "token budget 100000 per iteration from a 10^6-sequence lognormal(6.9, 1.2) corpus, context 32768",
}


def config_dict(cfg: int) -> dict:
    W = w.make_workload(cfg)
    sch = [{k: int(s[k]) for k in ("tp", "pp", "cp", "max_len", "util_len", "a_q32", "b_q32", "c_q32")}
           for s in W.schemes]
    cand = [[int(k) for k in W.cand[c, : W.cand_np[c]]] for c in range(W.n_cand)]
    lens = np.ascontiguousarray(W.lengths, np.uint32)
    d = {"config": cfg, "workload": W.name, "n_iter": W.n_iter, "batch": W.batch if not W.ragged else None,
         "batch_max": W.batch, "n_total": W.n_total, "n_cand": W.n_cand, "k_pad": W.k_pad, "meta": W.meta,
         "lengths": {"generator": GENERATORS[cfg], "seed": int(W.meta.get("seed", -1)),
                     "sha256_lengths": hashlib.sha256(lens.tobytes()).hexdigest()},
         "schemes": sch, "candidates": cand}
    if W.ragged:
        d["lengths"]["sha256_offsets"] = hashlib.sha256(np.ascontiguousarray(W.offsets, np.uint32).tobytes()).hexdigest()
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="*", default=[1, 2, 3, 4, 5, 6])
    args = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "configs"), exist_ok=True)
    for cfg in args.configs:
        path = os.path.join(ROOT, "configs", f"cfg{cfg}.json")
        with open(path, "w") as f:
            json.dump(config_dict(cfg), f, indent=0, separators=(",", ":"))
        print("wrote", path)


if __name__ == "__main__":
    main()
