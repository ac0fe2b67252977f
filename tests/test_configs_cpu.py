"""configs/cfgN.json (tools/export_configs.py) describe exactly the workloads the tests and bench.py
generate: scheme tables, candidate tables, sizes and the seeded lengths (SHA-256)."""
import os

import numpy as np
import pytest

import workload as w

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5, 6])
def test_config_json_matches_generator(cfg):
    W = w.make_workload(cfg)
    J = w.load_config(os.path.join(ROOT, "configs", f"cfg{cfg}.json"))
    assert J.name == W.name and J.k_pad == W.k_pad and J.n_iter == W.n_iter
    assert np.array_equal(J.schemes, W.schemes)
    assert np.array_equal(J.cand, W.cand) and np.array_equal(J.cand_np, W.cand_np)
    assert np.array_equal(J.lengths, W.lengths)
