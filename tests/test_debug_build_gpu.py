"""The bounds-checked build (libhyd_debug.so: -DHYD_DEBUG_CHECKS, and HYD_SPLIT_TASKS=0 so the warp
queue takes its sequential path, which the release build keeps for queues of more than 2 M
pipelines) runs every kernel family's cases of tools/sanitize_cases.py against the oracle in a
subprocess: no device check may fire and every result must match."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_debug_build_cases():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_07894_b200 import build

    lib = build.build_debug()
    env = dict(os.environ, HYD_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py")], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=1200)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "SANITIZE_CASES_OK" in r.stdout, out[-3000:]
    assert "HYD_CHECK failed" not in out
