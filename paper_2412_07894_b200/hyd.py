"""Thin ctypes binding of libhyd.so (include/hyd.h) -- argument marshalling only.

Every function here has the same name as its C entry point (minus the ``hyd_``
prefix) and forwards device pointers of torch tensors plus the CUDA stream handle.
All computation happens in the sm_100a kernels of libhyd.so.  There is no CPU
fallback: if the library is missing, loading raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# HYD_LIB: an alternative build of the same sources (libhyd_debug.so, device bounds checks)
LIB_PATH = os.environ.get("HYD_LIB") or os.path.join(HERE, "libhyd.so")

HYD_OK = 0
STATUS_BITS = {1: "OVERFLOW", 2: "ZERO_COST", 4: "BAD_LENGTH", 8: "KEY_RANGE", 16: "NOT_CANONICAL", 32: "BAD_PIPE"}
MAX_PIPES = 32
PIPE_STATS_BYTES = 24  # sizeof(hyd_pipe_stats)
KEY_SHIFT = 20
INT64_MAX = 2**63 - 1

# every function include/hyd.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "hyd_cost_table",
    "hyd_dispatch_workspace",
    "hyd_dispatch",
    "hyd_pack_workspace",
    "hyd_pack",
    "hyd_select_best",
    "hyd_gather_winners",
    "hyd_assign_workspace",
    "hyd_assign_key_offset",
    "hyd_assign_host",
    "hyd_check_candidates",
    "hyd_status_string",
    "hyd_last_cuda_error",
    "hyd_kernel_launches",
    "hyd_cost_table_ragged",
    "hyd_dispatch_ragged",
    "hyd_pack_ragged",
    "hyd_gather_winners_ragged",
    "hyd_assign_workspace_ragged",
    "hyd_assign_key_offset_ragged",
    "hyd_assign_host_ragged",
    "hyd_eq3_exact",
    "hyd_eq1_exact",
    "hyd_dp_workspace",
    "hyd_dp_propose",
    "hyd_alg1_workspace",
    "hyd_alg1_permutations",
    "hyd_dispatch_alg1",
    "hyd_pipe_index",
    "hyd_pipe_index_ragged",
    "hyd_dp_candidates",
    "hyd_dispatch_pack_workspace",
    "hyd_dispatch_pack",
    "hyd_dispatch_pack_ragged",
)


class HydError(RuntimeError):
    pass


# hyd_collective_fn(buf_dev, count, op, user, stream); op: COLL_MIN_I64 / COLL_SUM_I32
COLL_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p, C.c_void_p)
COLL_MIN_I64, COLL_SUM_I32 = 0, 1
_lib = None


def lib():
    """Load libhyd.so (never builds or substitutes anything at run time)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise HydError(f"{LIB_PATH} is missing: build it with `python -m paper_2412_07894_b200.build`")
    L = C.CDLL(LIB_PATH)
    I, P, Z, U64 = C.c_int, C.c_void_p, C.c_size_t, C.c_uint64
    sig = {
        "hyd_cost_table": ([P, I, I, P, I, I, P, P, P, P, P], I),
        "hyd_dispatch_workspace": ([I], Z),
        "hyd_dispatch": ([P, P, I, I, I, P, I, P, P, I, I, P, P, P, P, P, P, Z, P], I),
        "hyd_pack_workspace": ([I, I, I, I], Z),
        "hyd_pack": ([P, P, I, I, I, P, I, P, P, I, I, P, P, P, P, P, P, P, P, P, Z, P], I),
        "hyd_select_best": ([P, I, I, I, P, P, P], I),
        "hyd_gather_winners": ([P, P, P, P, P, P, I, I, I, I, P, P, P, P, P], I),
        "hyd_assign_workspace": ([I, I, I, I, I, I], Z),
        "hyd_assign_key_offset": ([I, I, I, I, I, I], Z),
        "hyd_assign_host": ([P, I, I, P, I, I, P, P, I, I, P, P, P, P, P, P, COLL_FN, P, P, Z, P], I),
        "hyd_check_candidates": ([P, P, I, P, I, C.POINTER(C.c_int)], I),
        "hyd_status_string": ([I], C.c_char_p),
        "hyd_last_cuda_error": ([], C.c_char_p),
        "hyd_kernel_launches": ([], I),
        "hyd_cost_table_ragged": ([P, I, P, I, I, P, I, I, P, P, P, P, P], I),
        "hyd_dispatch_ragged": ([P, P, I, P, I, I, I, P, I, P, P, I, I, P, P, P, P, P, P, Z, P], I),
        "hyd_pack_ragged": ([P, P, I, P, I, I, I, P, I, P, P, I, I, P, P, P, P, P, P, P, P, P, Z, P], I),
        "hyd_gather_winners_ragged": ([P, P, P, P, P, P, I, P, I, I, I, I, P, P, P, P, P], I),
        "hyd_assign_workspace_ragged": ([I, I, I, I, I, I, I], Z),
        "hyd_assign_key_offset_ragged": ([I, I, I, I, I, I, I], Z),
        "hyd_assign_host_ragged": ([P, I, P, I, P, I, I, P, P, I, I, P, P, P, P, P, P, COLL_FN, P, P, Z, P], I),
        "hyd_eq3_exact": ([P, P, I, I, I, P, I, P, P, I, P, P, I, C.c_uint64, P, P, P, P, P, P], I),
        "hyd_eq1_exact": ([P, P, I, I, I, P, I, P, I, I, P, P, P, P, I, C.c_uint64, P, P, P, P, P, P], I),
        "hyd_dp_workspace": ([I, I], Z),
        "hyd_dp_propose": ([P, I, P, I, I, I, I, I, P, P, P, P, P, P, P, P, P, Z, P], I),
        "hyd_alg1_workspace": ([I], Z),
        "hyd_alg1_permutations": ([U64, I, I, I, P, P], I),
        "hyd_dispatch_alg1": ([P, P, I, I, I, P, I, P, P, I, I, I, P, P, P, P, P, P, P, P, Z, P], I),
        "hyd_dispatch_pack_workspace": ([], Z),
        "hyd_dispatch_pack": ([P, P, I, I, I, P, I, P, P, I, I, P, P, P, P, P, P, P, P, Z, P], I),
        "hyd_dispatch_pack_ragged": ([P, P, I, P, I, I, I, P, I, P, P, I, I, P, P, P, P, P, P, P, P, Z, P], I),
        "hyd_dp_candidates": ([P, P, I, P, I, P, P, P, P], I),
        "hyd_pipe_index": ([P, P, I, I, I, P, I, P, P, I, I, P, P, P, P, P, P], I),
        "hyd_pipe_index_ragged": ([P, P, I, P, I, I, I, P, I, P, P, I, I, P, P, P, P, P, P], I),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    del U64
    _lib = L
    return L


def _check(rc: int, what: str):
    if rc != HYD_OK:
        L = lib()
        msg = L.hyd_status_string(rc).decode()
        if rc == -5:
            msg += ": " + L.hyd_last_cuda_error().decode()
        raise HydError(f"{what} failed ({rc}): {msg}")


def _dev(t):
    if t is None:
        return None
    if not t.is_cuda or not t.is_contiguous():
        raise HydError("expected a contiguous CUDA tensor")
    return t.data_ptr()


def _stream(stream):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def kernel_launches() -> int:
    return int(lib().hyd_kernel_launches())


def status_names(bits: int):
    return [n for b, n in STATUS_BITS.items() if bits & b]


def check_candidates(cand, cand_np, schemes) -> int:
    """Host validation of candidate tables (numpy); returns max_np."""
    import numpy as np

    cand = np.ascontiguousarray(cand, dtype=np.uint8)
    cand_np = np.ascontiguousarray(cand_np, dtype=np.uint8)
    schemes = np.ascontiguousarray(schemes)
    mx = C.c_int(0)
    rc = lib().hyd_check_candidates(cand.ctypes.data, cand_np.ctypes.data, cand.shape[0],
                                    schemes.ctypes.data, schemes.shape[0], C.byref(mx))
    _check(rc, "hyd_check_candidates")
    return int(mx.value)


def cost_table(len_, n_iter, batch, schemes, n_schemes, k_pad, sorted_len, perm, cost, status, stream=None):
    _check(lib().hyd_cost_table(_dev(len_), n_iter, batch, _dev(schemes), n_schemes, k_pad, _dev(sorted_len),
                                _dev(perm), _dev(cost), _dev(status), _stream(stream)), "hyd_cost_table")


def dispatch_workspace(n_iter) -> int:
    return int(lib().hyd_dispatch_workspace(n_iter))


def dispatch(sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, max_np, pipe, lb,
             stats, members, status, ws, stream=None):
    _check(lib().hyd_dispatch(_dev(sorted_len), _dev(cost), n_iter, batch, k_pad, _dev(schemes), n_schemes,
                              _dev(cand), _dev(cand_np), n_cand, max_np, _dev(pipe), _dev(lb), _dev(stats),
                              _dev(members), _dev(status), _dev(ws), ws.numel() * ws.element_size(),
                              _stream(stream)), "hyd_dispatch")


def pack_workspace(n_iter, batch, n_cand, max_np) -> int:
    return int(lib().hyd_pack_workspace(n_iter, batch, n_cand, max_np))


def pack(sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, max_np, pipe, stats,
         members, mb, v, ptime, makespan, status, ws, stream=None):
    _check(lib().hyd_pack(_dev(sorted_len), _dev(cost), n_iter, batch, k_pad, _dev(schemes), n_schemes, _dev(cand),
                          _dev(cand_np), n_cand, max_np, _dev(pipe), _dev(stats), _dev(members), _dev(mb), _dev(v),
                          _dev(ptime),
                          _dev(makespan), _dev(status), _dev(ws), ws.numel() * ws.element_size(),
                          _stream(stream)), "hyd_pack")


# ---- NEXT-2: ragged (token-budget) batches; ``off`` is the device CSR offsets tensor [It + 1]
def cost_table_ragged(len_, n_iter, off, n_total, batch_max, schemes, n_schemes, k_pad, sorted_len, perm, cost,
                      status, stream=None):
    _check(lib().hyd_cost_table_ragged(_dev(len_), n_iter, _dev(off), n_total, batch_max, _dev(schemes), n_schemes,
                                       k_pad, _dev(sorted_len), _dev(perm), _dev(cost), _dev(status),
                                       _stream(stream)), "hyd_cost_table_ragged")


def dispatch_ragged(sorted_len, cost, n_iter, off, n_total, batch_max, k_pad, schemes, n_schemes, cand, cand_np,
                    n_cand, max_np, pipe, lb, stats, members, status, ws, stream=None):
    _check(lib().hyd_dispatch_ragged(_dev(sorted_len), _dev(cost), n_iter, _dev(off), n_total, batch_max, k_pad,
                                     _dev(schemes), n_schemes, _dev(cand), _dev(cand_np), n_cand, max_np, _dev(pipe),
                                     _dev(lb), _dev(stats), _dev(members), _dev(status), _dev(ws),
                                     ws.numel() * ws.element_size(), _stream(stream)), "hyd_dispatch_ragged")


def pack_ragged(sorted_len, cost, n_iter, off, n_total, batch_max, k_pad, schemes, n_schemes, cand, cand_np, n_cand,
                max_np, pipe, stats, members, mb, v, ptime, makespan, status, ws, stream=None):
    _check(lib().hyd_pack_ragged(_dev(sorted_len), _dev(cost), n_iter, _dev(off), n_total, batch_max, k_pad,
                                 _dev(schemes), n_schemes, _dev(cand), _dev(cand_np), n_cand, max_np, _dev(pipe),
                                 _dev(stats), _dev(members), _dev(mb), _dev(v), _dev(ptime), _dev(makespan),
                                 _dev(status), _dev(ws), ws.numel() * ws.element_size(), _stream(stream)),
           "hyd_pack_ragged")


def assign_workspace_ragged(n_iter, n_total, batch_max, n_schemes, k_pad, n_cand, max_np) -> int:
    return int(lib().hyd_assign_workspace_ragged(n_iter, n_total, batch_max, n_schemes, k_pad, n_cand, max_np))


def assign_key_offset_ragged(n_iter, n_total, batch_max, n_schemes, k_pad, n_cand, max_np) -> int:
    return int(lib().hyd_assign_key_offset_ragged(n_iter, n_total, batch_max, n_schemes, k_pad, n_cand, max_np))


def assign_host_ragged(len_host_ptr, n_iter, off_host_ptr, batch_max, schemes_host_ptr, n_schemes, k_pad,
                       cand_host_ptr, cand_np_host_ptr, n_cand, cand_offset, key_host_ptr, win_pipe_ptr, win_mb_ptr,
                       win_v_ptr, win_ptime_ptr, status_ptr, coll_cb, ws, stream=None):
    cb = coll_cb if coll_cb is not None else COLL_FN(0)
    _check(lib().hyd_assign_host_ragged(len_host_ptr, n_iter, off_host_ptr, batch_max, schemes_host_ptr, n_schemes,
                                        k_pad, cand_host_ptr, cand_np_host_ptr, n_cand, cand_offset, key_host_ptr,
                                        win_pipe_ptr, win_mb_ptr, win_v_ptr, win_ptime_ptr, status_ptr, cb, None,
                                        _dev(ws), ws.numel() * ws.element_size(), _stream(stream)),
           "hyd_assign_host_ragged")


BB_MAX_BATCH = 64


def eq3_exact(sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, pair_c, pair_t,
              node_limit, value, pipe, nodes, proved, status, stream=None):
    _check(lib().hyd_eq3_exact(_dev(sorted_len), _dev(cost), n_iter, batch, k_pad, _dev(schemes), n_schemes,
                               _dev(cand), _dev(cand_np), n_cand, _dev(pair_c), _dev(pair_t), int(pair_c.numel()),
                               int(node_limit), _dev(value), _dev(pipe), _dev(nodes), _dev(proved), _dev(status),
                               _stream(stream)), "hyd_eq3_exact")


def eq1_exact(sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, n_cand, max_np, members, pair_c,
              pair_t, pair_j, node_limit, v, obj, nodes, proved, status, stream=None):
    _check(lib().hyd_eq1_exact(_dev(sorted_len), _dev(cost), n_iter, batch, k_pad, _dev(schemes), n_schemes,
                               _dev(cand), n_cand, max_np, _dev(members), _dev(pair_c), _dev(pair_t), _dev(pair_j),
                               int(pair_c.numel()), int(node_limit), _dev(v), _dev(obj), _dev(nodes), _dev(proved),
                               _dev(status), _stream(stream)), "hyd_eq1_exact")


DP_MAX_ROUND = 64


def dp_workspace(n_schemes, J) -> int:
    return int(lib().hyd_dp_workspace(n_schemes, J))


def dp_propose(lengths, n_seq, schemes, n_schemes, step, J, n_gpus, scale, t_num, t_den, choice, counts, rows, valid,
               keep, status, ws, stream=None):
    _check(lib().hyd_dp_propose(_dev(lengths), n_seq, _dev(schemes), n_schemes, step, J, n_gpus, scale, _dev(t_num),
                                _dev(t_den), _dev(choice), _dev(counts), _dev(rows), _dev(valid), _dev(keep),
                                _dev(status), _dev(ws), ws.numel() * ws.element_size(), _stream(stream)),
           "hyd_dp_propose")


def dp_candidates(rows, keep, J, schemes, n_schemes, cand, cand_np, n_out, stream=None):
    _check(lib().hyd_dp_candidates(_dev(rows), _dev(keep), J, _dev(schemes), n_schemes, _dev(cand), _dev(cand_np),
                                   _dev(n_out), _stream(stream)), "hyd_dp_candidates")


def alg1_workspace(n_iter) -> int:
    return int(lib().hyd_alg1_workspace(n_iter))


def alg1_permutations(seed, n_iter, batch, trials, order, stream=None):
    _check(lib().hyd_alg1_permutations(int(seed) & 0xFFFFFFFFFFFFFFFF, n_iter, batch, trials, _dev(order),
                                       _stream(stream)), "hyd_alg1_permutations")


def dispatch_alg1(sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, max_np, trials,
                  order, best, pipe, lb, stats, members, status, ws, stream=None):
    _check(lib().hyd_dispatch_alg1(_dev(sorted_len), _dev(cost), n_iter, batch, k_pad, _dev(schemes), n_schemes,
                                   _dev(cand), _dev(cand_np), n_cand, max_np, trials, _dev(order), _dev(best),
                                   _dev(pipe), _dev(lb), _dev(stats), _dev(members), _dev(status), _dev(ws),
                                   ws.numel() * ws.element_size(), _stream(stream)), "hyd_dispatch_alg1")


def pipe_index(sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, max_np, pipe, lb,
               stats, members, status, stream=None):
    _check(lib().hyd_pipe_index(_dev(sorted_len), _dev(cost), n_iter, batch, k_pad, _dev(schemes), n_schemes,
                                _dev(cand), _dev(cand_np), n_cand, max_np, _dev(pipe), _dev(lb), _dev(stats),
                                _dev(members), _dev(status), _stream(stream)), "hyd_pipe_index")


def pipe_index_ragged(sorted_len, cost, n_iter, off, n_total, batch_max, k_pad, schemes, n_schemes, cand, cand_np,
                      n_cand, max_np, pipe, lb, stats, members, status, stream=None):
    _check(lib().hyd_pipe_index_ragged(_dev(sorted_len), _dev(cost), n_iter, _dev(off), n_total, batch_max, k_pad,
                                       _dev(schemes), n_schemes, _dev(cand), _dev(cand_np), n_cand, max_np,
                                       _dev(pipe), _dev(lb), _dev(stats), _dev(members), _dev(status),
                                       _stream(stream)), "hyd_pipe_index_ragged")


SMALL_MAX_BATCH = 128


def dispatch_pack_workspace() -> int:
    return int(lib().hyd_dispatch_pack_workspace())


def dispatch_pack(sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, max_np, pipe, lb,
                  mb, v, ptime, makespan, status, ws, stream=None):
    _check(lib().hyd_dispatch_pack(_dev(sorted_len), _dev(cost), n_iter, batch, k_pad, _dev(schemes), n_schemes,
                                   _dev(cand), _dev(cand_np), n_cand, max_np, _dev(pipe), _dev(lb), _dev(mb), _dev(v),
                                   _dev(ptime), _dev(makespan), _dev(status), _dev(ws), ws.numel() * ws.element_size(),
                                   _stream(stream)), "hyd_dispatch_pack")


def dispatch_pack_ragged(sorted_len, cost, n_iter, off, n_total, batch_max, k_pad, schemes, n_schemes, cand, cand_np,
                         n_cand, max_np, pipe, lb, mb, v, ptime, makespan, status, ws, stream=None):
    _check(lib().hyd_dispatch_pack_ragged(_dev(sorted_len), _dev(cost), n_iter, _dev(off), n_total, batch_max, k_pad,
                                          _dev(schemes), n_schemes, _dev(cand), _dev(cand_np), n_cand, max_np,
                                          _dev(pipe), _dev(lb), _dev(mb), _dev(v), _dev(ptime), _dev(makespan),
                                          _dev(status), _dev(ws), ws.numel() * ws.element_size(), _stream(stream)),
           "hyd_dispatch_pack_ragged")


def select_best(makespan, n_iter, n_cand, cand_offset, key, status, stream=None):
    _check(lib().hyd_select_best(_dev(makespan), n_iter, n_cand, cand_offset, _dev(key), _dev(status),
                                 _stream(stream)), "hyd_select_best")


def gather_winners(key, perm, pipe, mb, v, ptime, n_iter, batch, n_cand, cand_offset, win_pipe, win_mb, win_v,
                   win_ptime, stream=None):
    _check(lib().hyd_gather_winners(_dev(key), _dev(perm), _dev(pipe), _dev(mb), _dev(v), _dev(ptime), n_iter,
                                    batch, n_cand, cand_offset, _dev(win_pipe), _dev(win_mb), _dev(win_v),
                                    _dev(win_ptime), _stream(stream)), "hyd_gather_winners")


def assign_workspace(n_iter, batch, n_schemes, k_pad, n_cand, max_np) -> int:
    return int(lib().hyd_assign_workspace(n_iter, batch, n_schemes, k_pad, n_cand, max_np))


def assign_key_offset(n_iter, batch, n_schemes, k_pad, n_cand, max_np) -> int:
    return int(lib().hyd_assign_key_offset(n_iter, batch, n_schemes, k_pad, n_cand, max_np))


def assign_host(len_host_ptr, n_iter, batch, schemes_host_ptr, n_schemes, k_pad, cand_host_ptr, cand_np_host_ptr,
                n_cand, cand_offset, key_host_ptr, win_pipe_ptr, win_mb_ptr, win_v_ptr, win_ptime_ptr,
                status_ptr, coll_cb, ws, stream=None):
    """hyd_assign_host with HOST pointers (ints); ``coll_cb`` is a COLL_FN or None (one rank)."""
    cb = coll_cb if coll_cb is not None else COLL_FN(0)
    _check(lib().hyd_assign_host(len_host_ptr, n_iter, batch, schemes_host_ptr, n_schemes, k_pad, cand_host_ptr,
                                 cand_np_host_ptr, n_cand, cand_offset, key_host_ptr, win_pipe_ptr, win_mb_ptr,
                                 win_v_ptr, win_ptime_ptr, status_ptr, cb, None, _dev(ws),
                                 ws.numel() * ws.element_size(), _stream(stream)), "hyd_assign_host")
