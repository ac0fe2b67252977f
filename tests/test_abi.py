"""C-ABI boundary checks that need no GPU: libhyd.so loads, exports every function that
include/hyd.h declares, and host-side validation answers synchronously."""
import ctypes
import os
import re

import numpy as np
import pytest

import workload as w

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def hyd():
    from paper_2412_07894_b200 import build, hyd

    build.build()
    return hyd


def declared_functions():
    src = open(os.path.join(ROOT, "include", "hyd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hyd_[a-z0-9_]+)\s*\(", src)) - {"hyd_reduce_fn"})


def test_exports_every_declared_symbol(hyd):
    L = hyd.lib()
    decl = declared_functions()
    assert len(decl) >= 13
    for name in decl:
        assert hasattr(L, name), name
    assert sorted(hyd.EXPORTS) == decl


def test_status_strings(hyd):
    L = hyd.lib()
    assert L.hyd_status_string(0) == b"ok"
    assert b"canonical" in L.hyd_status_string(-2)
    assert L.hyd_status_string(12345) == b"unknown status"


def test_host_validation_is_synchronous(hyd):
    L = hyd.lib()
    P = ctypes.c_void_p(1)  # never dereferenced: validation fails first
    assert L.hyd_cost_table(None, 1, 16, P, 1, 4, P, P, P, P, None) == -1
    assert L.hyd_cost_table(P, 1, 0, P, 1, 4, P, P, P, P, None) == -1  # batch 0
    assert L.hyd_cost_table(P, 1, 16, P, 5, 4, P, P, P, P, None) == -1  # k_pad < K
    assert L.hyd_cost_table(P, 1, 16, P, 3, 6, P, P, P, P, None) == -1  # k_pad % 4
    assert L.hyd_cost_table(P, 1, 16385, P, 1, 4, P, P, P, P, None) == -1  # batch limit
    assert L.hyd_dispatch(P, P, 1, 16, 4, P, 1, P, P, 1, 33, P, P, P, P, P, P, 4096, None) == -1  # max_np > 32
    assert L.hyd_dispatch(P, P, 1, 16, 4, P, 1, P, P, 1, 2, P, P, None, P, P, P, 4096, None) == -1  # stats null
    assert L.hyd_dispatch(P, P, 1, 16, 4, P, 1, P, P, 1, 2, P, P, P, P, P, None, 0, None) == -6  # no workspace
    assert L.hyd_dispatch_workspace(1024) >= 1024 * 8
    assert L.hyd_select_best(P, 4, 10, (1 << 20) - 5, P, P, None) == -1  # key range
    assert L.hyd_pack(P, P, 1, 16, 4, P, 1, P, P, 1, 2, P, P, P, P, P, P, P, P, None, 0, None) == -6
    # NEXT-1: trials in [1, HYD_MAX_TRIALS], workspace
    assert L.hyd_alg1_permutations(1, 1, 16, 0, P, None) == -1
    assert L.hyd_alg1_permutations(1, 1, 16, 257, P, None) == -1
    assert L.hyd_alg1_permutations(1, 1, 16, 4, None, None) == -1
    assert L.hyd_dispatch_alg1(P, P, 1, 16, 4, P, 1, P, P, 1, 2, 0, P, P, P, P, P, P, P, P, 4096, None) == -1
    assert L.hyd_dispatch_alg1(P, P, 1, 16, 4, P, 1, P, P, 1, 2, 4, P, P, P, P, P, P, P, None, 0, None) == -6
    assert L.hyd_alg1_workspace(1024) >= 1024 * 8
    # iterations map to a grid dimension: n_iter <= HYD_MAX_ITER (65535)
    assert L.hyd_cost_table(P, 65536, 16, P, 1, 4, P, P, P, P, None) == -1
    assert L.hyd_select_best(P, 65536, 10, 0, P, P, None) == -1
    # the fused small-batch kernel: batch <= 128, <= 16 pipelines, workspace
    Z = L.hyd_dispatch_pack_workspace()
    assert L.hyd_dispatch_pack(P, P, 1, 129, 4, P, 1, P, P, 1, 2, P, P, P, P, P, P, P, P, Z, None) == -1
    assert L.hyd_dispatch_pack(P, P, 1, 64, 4, P, 1, P, P, 1, 17, P, P, P, P, P, P, P, P, Z, None) == -1
    assert L.hyd_dispatch_pack(P, P, 1, 64, 4, P, 1, P, P, 1, 8, P, P, P, P, P, P, P, None, 0, None) == -6
    # hyd_pipe_index / hyd_dp_candidates argument checks
    assert L.hyd_pipe_index(P, P, 1, 16, 4, P, 1, P, P, 1, 33, P, P, P, P, P, None) == -1
    assert L.hyd_pipe_index(P, P, 1, 16, 4, P, 1, P, P, 1, 2, None, P, P, P, P, None) == -1
    assert L.hyd_dp_candidates(P, P, 0, P, 1, P, P, P, None) == -1


def test_workspace_sizes(hyd):
    n = hyd.pack_workspace(1024, 512, 4096, 8)
    assert n >= 1024 * 4096 * 8 * 8
    total = hyd.assign_workspace(1024, 512, 14, 16, 4096, 8)
    assert total > n + 4096 * 1024 * 512 * 3
    assert hyd.assign_key_offset(1024, 512, 14, 16, 4096, 8) % 256 == 0


def test_check_candidates(hyd):
    W = w.make_workload(4, n_cand=64, n_iter=1)
    assert hyd.check_candidates(W.cand, W.cand_np, W.schemes) == 8
    bad = W.cand.copy()
    bad[3, [0, 1]] = bad[3, [1, 0]]
    if W.schemes[bad[3, 0]]["max_len"] != W.schemes[bad[3, 1]]["max_len"] or bad[3, 0] != bad[3, 1]:
        with pytest.raises(hyd.HydError, match="canonical"):
            hyd.check_candidates(bad, W.cand_np, W.schemes)
    nz = W.cand_np.copy()
    nz[0] = 0
    with pytest.raises(hyd.HydError):
        hyd.check_candidates(W.cand, nz, W.schemes)
    oob = W.cand.copy()
    oob[0, 0] = 200
    with pytest.raises(hyd.HydError):
        hyd.check_candidates(oob, W.cand_np, W.schemes)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2412_07894_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "hydref" not in txt, f


def test_scheme_record_layout():
    assert w.SCHEME_DTYPE.itemsize == 48
    assert w.SCHEME_DTYPE.fields["a_q32"][1] == 24
    hdr = open(os.path.join(ROOT, "include", "hyd.h")).read()
    assert "uint64_t a_q32, b_q32, c_q32;" in hdr
    assert np.dtype(w.SCHEME_DTYPE).names[:5] == ("tp", "pp", "cp", "max_len", "util_len")
