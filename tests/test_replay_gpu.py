"""Replay dumps (tools/replay.py): a batch's inputs and hyd_assign_host outputs written to .bin
files replay bit for bit, and the replayed keys equal the oracle's (uniform and token-budget)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("cfg", [4, 6])
def test_dump_and_replay(tmp_path, cfg):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    tool = os.path.join(ROOT, "tools", "replay.py")
    d = str(tmp_path / f"cfg{cfg}")
    r = subprocess.run([sys.executable, tool, "dump", d, "--config", str(cfg), "--cands", "48", "--iters", "5"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    r = subprocess.run([sys.executable, tool, "check", d, "--oracle"], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "REPLAY_OK" in r.stdout, r.stdout + r.stderr
