"""The committed goldens (tests/golden/digests_cfgN.npz, what test_digests_gpu.py compares the CUDA
path with) are complete and are what the oracle as it stands computes:

* every file covers its whole BASELINE configuration (all candidates, all iterations);
* the first iterations of configs 1, 2, 3, 4 and 6, recomputed here by
  tools/make_golden_digests.py (oracle/ and workload/ only), match the committed digests --
  an oracle change that was not followed by regenerating the goldens fails here;
* writing a range in two parts and joining them with --merge gives the single-range file.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import workload as w

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
TOOL = os.path.join(ROOT, "tools", "make_golden_digests.py")
META = ("n_iter", "t0", "n_cand", "status", "n_cand_total", "workload", "seed")


def _run(*args):
    subprocess.run([sys.executable, TOOL, *args], check=True, cwd=ROOT, stdout=subprocess.DEVNULL)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5, 6])
def test_golden_covers_whole_config(cfg):
    g = np.load(os.path.join(GOLDEN, f"digests_cfg{cfg}.npz"))
    c = w.CONFIGS[cfg]
    assert int(g["n_iter"]) == c["It"] and int(g["n_cand"]) == c["C"] == int(g["n_cand_total"])
    assert str(g["workload"]) == c["name"] and int(g["status"]) == 0
    for k in ("sorted_len", "perm", "cost", "pipe", "lb", "mb", "v", "ptime", "makespan", "key"):
        assert g[k].shape == (c["It"],), k


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 6])
def test_golden_prefix_recomputes(cfg, tmp_path):
    _run("--configs", str(cfg), "--iter-range", "0", "2", "--chunk", "2", "--out", str(tmp_path))
    part = np.load(tmp_path / f"digests_cfg{cfg}_t0-2.npz")
    g = np.load(os.path.join(GOLDEN, f"digests_cfg{cfg}.npz"))
    for k in part.files:
        if k not in META:
            assert np.array_equal(part[k], g[k][:2]), k


def test_merge_equals_single_range(tmp_path):
    a, b = tmp_path / "a", tmp_path / "b"
    _run("--configs", "2", "--iter-range", "0", "4", "--chunk", "4", "--out", str(a))
    _run("--configs", "2", "--iter-range", "0", "2", "--chunk", "2", "--out", str(b))
    _run("--configs", "2", "--iter-range", "2", "4", "--chunk", "2", "--out", str(b))
    _run("--configs", "2", "--merge", "--out", str(b))
    one, joined = np.load(a / "digests_cfg2_t0-4.npz"), np.load(b / "digests_cfg2.npz")
    assert int(joined["n_iter"]) == 4
    for k in one.files:
        if k not in META:
            assert np.array_equal(one[k], joined[k]), k
