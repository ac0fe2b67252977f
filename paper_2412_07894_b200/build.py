"""Build libhyd.so (sm_100a) in-tree with nvcc.  Usage: python -m paper_2412_07894_b200.build"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libhyd.so")
SOURCES = ["sort_cost.cu", "dispatch.cu", "alg1.cu", "pack.cu", "select.cu", "index.cu", "small.cu", "dp.cu", "bb.cu", "api.cu"]
HEADERS = ["hyd_internal.cuh", "search.cuh"]


def nvcc() -> str:
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(p):
        raise RuntimeError("nvcc not found")
    return p


FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
    "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include"),
]


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "hyd.h")]
    return any(os.path.getmtime(d) > t for d in deps)


DEBUG_LIB = os.path.join(HERE, "libhyd_debug.so")


def build_debug(force: bool = False) -> str:
    """libhyd_debug.so: the same sources with -DHYD_DEBUG_CHECKS (device bounds checks); loaded
    instead of libhyd.so when HYD_LIB points at it (tools/sanitize_cases.py)."""
    if not force and os.path.exists(DEBUG_LIB) and not _stale(DEBUG_LIB):
        return DEBUG_LIB
    # HYD_SPLIT_TASKS=0: the warp queue takes its sequential path, which the release build uses
    # only for queues of more than 2 M pipelines -- so the debug cases cover both paths
    return build(force=True, extra=["-DHYD_DEBUG_CHECKS", "-DHYD_SPLIT_TASKS=0"], out=DEBUG_LIB,
                 bdir_name="build_debug")


def build(force: bool = False, verbose: bool = False, extra: list[str] | None = None, out: str = LIB,
          bdir_name: str = "build") -> str:
    if not force and not _stale(out):
        return out
    bdir = os.path.join(HERE, bdir_name)
    os.makedirs(bdir, exist_ok=True)
    objs = []
    for src in SOURCES:
        obj = os.path.join(bdir, src.replace(".cu", ".o"))
        cmd = [nvcc(), *FLAGS, *(extra or []), "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        objs.append(obj)
    tmp = out + f".tmp{os.getpid()}"
    subprocess.check_call([nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", tmp])
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, extra=["-Xptxas", "-v"] if "--ptxas" in sys.argv else None)
    print(LIB)
