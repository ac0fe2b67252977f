"""CPU oracle of the Hydraulis two-stage assignment (HYD-H1) -- ctypes wrapper.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` leg may import this package.
The product path (``paper_2412_07894_b200``) never imports it and shares no code
with it; the two meet only in ``workload`` (seeded inputs, no method arithmetic).

The arithmetic lives in ``oracle/hydref.c`` (plain C11, cited to PAPER.md).
This wrapper only marshals numpy arrays.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRCS = [os.path.join(_HERE, "hydref.c"), os.path.join(_HERE, "alg1ref.c"), os.path.join(_HERE, "dpref.c"),
         os.path.join(_HERE, "bbref.c")]
_HDR = os.path.join(_HERE, "hydref.h")
_LIB = os.path.join(_HERE, "libhydref.so")


def build(force: bool = False) -> str:
    """Compile oracle/libhydref.so with gcc (idempotent)."""
    newest = max(os.path.getmtime(f) for f in _SRCS + [_HDR])
    stale = not os.path.exists(_LIB) or newest > os.path.getmtime(_LIB)
    if force or stale:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-std=gnu11", "-O2", "-g", "-Wall", "-Wextra", "-shared", "-fPIC", "-pthread", *_SRCS, "-o", tmp]
        )
        os.replace(tmp, _LIB)
    return _LIB


_lib = None

_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_voidp = C.c_void_p


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        I, U32P = C.c_int, C.POINTER(C.c_uint32)
        L.hydref_cost.argtypes = [_voidp, C.c_uint32, U32P]
        L.hydref_cost.restype = C.c_uint32
        L.hydref_sort.argtypes = [_u32p, I, _u32p, _u32p]
        L.hydref_cost_table.argtypes = [_u32p, I, _voidp, I, I, _u32p, _u32p, _u32p, U32P]
        L.hydref_dispatch.argtypes = [_u32p, _u32p, I, I, _voidp, _u8p, I, _u8p, C.POINTER(C.c_uint64)]
        L.hydref_dispatch.restype = I
        L.hydref_lpt.argtypes = [_u32p, _u32p, I, I, C.c_uint32, _u16p, C.POINTER(C.c_uint64)]
        L.hydref_lpt.restype = I
        L.hydref_lpt_heap.argtypes = [_u32p, _u32p, I, I, C.c_uint32, _u16p, C.POINTER(C.c_uint64)]
        L.hydref_lpt_heap.restype = I
        L.hydref_pack_pipeline.argtypes = [
            _u32p, _u32p, I, _voidp, C.POINTER(C.c_uint16), C.POINTER(C.c_uint64), _u16p, U32P,
        ]
        L.hydref_assign_pair.argtypes = [
            _u32p, _u32p, I, I, _voidp, _u8p, I, _u8p, C.POINTER(C.c_uint64), _u16p, _u16p, _u64p, U32P,
        ]
        L.hydref_assign_pair.restype = C.c_uint64
        L.hydref_pack_pair.argtypes = [
            _u32p, _u32p, I, I, _voidp, _u8p, I, _u8p, _u16p, _u16p, _u64p, U32P,
        ]
        L.hydref_pack_pair.restype = C.c_uint64
        L.hydref_select.argtypes = [_u64p, I, I, U32P]
        L.hydref_select.restype = C.c_int64
        L.hydref_assign_batch.argtypes = [
            _u32p, I, I, _voidp, I, I, _u8p, _u8p, I, I, _u32p, _u32p, _u32p,
            _u8p, _u64p, _u16p, _u16p, _u64p, _u64p, _i64p, U32P, I,
        ]
        L.hydref_assign_pairs.argtypes = [
            _u32p, _u32p, I, I, I, _voidp, _u8p, _u8p, _i32p, _i32p, I,
            _u8p, _u64p, _u16p, _u16p, _u64p, _u64p, U32P, I,
        ]
        # NEXT-1 (alg1ref.c)
        U64 = C.c_uint64
        L.hydref_philox4x32_10.argtypes = [_u32p, _u32p, _u32p]
        L.hydref_alg1_permutation.argtypes = [U64, I, I, I, _u32p]
        L.hydref_alg1_trial.argtypes = [_u32p, _u32p, I, I, _voidp, _u8p, I, _u32p, _u8p]
        L.hydref_alg1_trial.restype = U64
        L.hydref_alg1_dispatch.argtypes = [
            _u32p, _u32p, I, I, _voidp, _u8p, I, U64, I, I, _u8p, C.POINTER(U64), C.POINTER(C.c_int32),
        ]
        L.hydref_alg1_dispatch.restype = I
        L.hydref_assign_batch_ex.argtypes = [
            _u32p, I, I, _voidp, I, I, _u8p, _u8p, I, I, I, U64, _u32p, _u32p, _u32p,
            _u8p, _u64p, _u16p, _u16p, _u64p, _u64p, _i64p, _i32p, U32P, I,
        ]
        L.hydref_assign_pairs_ex.argtypes = [
            _u32p, _u32p, I, I, I, _voidp, _u8p, _u8p, _i32p, _i32p, I, I, U64,
            _u8p, _u64p, _u16p, _u16p, _u64p, _u64p, _i32p, U32P, I,
        ]
        # NEXT-4 (bbref.c)
        L.hydref_eq3_exact.argtypes = [_u32p, _u32p, I, I, _voidp, _u8p, I, C.c_uint64, _u8p,
                                       C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.hydref_eq3_exact.restype = I
        L.hydref_eq1_exact.argtypes = [_u32p, _u32p, I, _voidp, C.c_uint64, C.POINTER(C.c_uint32),
                                       C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.hydref_eq1_exact.restype = I
        # NEXT-3 (dpref.c)
        L.hydref_dp_prefix.argtypes = [_u32p, I, _voidp, I, I, I, _u64p, U32P]
        L.hydref_dp_solve.argtypes = [_u64p, _voidp, I, I, I, I, I, _u64p, _u64p, _i32p]
        L.hydref_dp_solve.restype = I
        L.hydref_dp_strategy.argtypes = [_i32p, _u64p, _voidp, I, I, I, I, I, _u32p, U32P]
        L.hydref_dp_strategy.restype = I
        _lib = L
    return _lib


def _sch_ptr(schemes):
    assert schemes.dtype.itemsize == 48 and schemes.flags.c_contiguous
    return schemes.ctypes.data


def cost(scheme_row, l):
    """T(l, P) of one scheme (structured array of length 1 or a record)."""
    s = np.ascontiguousarray(np.atleast_1d(scheme_row))
    st = C.c_uint32(0)
    v = lib().hydref_cost(_sch_ptr(s), C.c_uint32(int(l)), C.byref(st))
    return int(v), int(st.value)


def sort(lengths):
    x = np.ascontiguousarray(lengths, dtype=np.uint32)
    s = np.empty_like(x)
    p = np.empty_like(x)
    lib().hydref_sort(x, x.size, s, p)
    return s, p


def cost_table(lengths_row, schemes, k_pad):
    x = np.ascontiguousarray(lengths_row, dtype=np.uint32)
    B = x.size
    s, p = np.empty(B, np.uint32), np.empty(B, np.uint32)
    cst = np.empty(B * k_pad, np.uint32)
    st = C.c_uint32(0)
    lib().hydref_cost_table(x, B, _sch_ptr(schemes), len(schemes), k_pad, s, p, cst, C.byref(st))
    return s, p, cst.reshape(B, k_pad), int(st.value)


def dispatch(sorted_len, cost_tab, schemes, cand_row):
    B, k_pad = cost_tab.shape
    row = np.full(32, 0xFF, np.uint8)
    row[: len(cand_row)] = cand_row
    pipe = np.empty(B, np.uint8)
    lb = C.c_uint64(0)
    ok = lib().hydref_dispatch(
        np.ascontiguousarray(sorted_len, np.uint32), np.ascontiguousarray(cost_tab, np.uint32).ravel(),
        B, k_pad, _sch_ptr(schemes), row, len(cand_row), pipe, C.byref(lb),
    )
    return bool(ok), pipe, int(lb.value)


def lpt(ell, tau, v, max_len, heap=False):
    """LPT(V) with capacity: the plain scan (hydref_lpt) or the heap form (hydref_lpt_heap)
    that hydref_pack_pipeline's V enumeration uses."""
    ell = np.ascontiguousarray(ell, np.uint32)
    tau = np.ascontiguousarray(tau, np.uint32)
    mb = np.zeros(max(ell.size, 1), np.uint16)
    mx = C.c_uint64(0)
    fn = lib().hydref_lpt_heap if heap else lib().hydref_lpt
    ok = fn(ell, tau, ell.size, int(v), int(max_len), mb, C.byref(mx))
    return bool(ok), mb[: ell.size], int(mx.value)


def pack_pipeline(ell, tau, scheme_row):
    ell = np.ascontiguousarray(ell, np.uint32)
    tau = np.ascontiguousarray(tau, np.uint32)
    s = np.ascontiguousarray(np.atleast_1d(scheme_row))
    mb = np.zeros(max(ell.size, 1), np.uint16)
    v, pt, st = C.c_uint16(0), C.c_uint64(0), C.c_uint32(0)
    lib().hydref_pack_pipeline(ell, tau, ell.size, _sch_ptr(s), C.byref(v), C.byref(pt), mb, C.byref(st))
    return int(v.value), int(pt.value), mb[: ell.size], int(st.value)


def is_assignment(sorted_len, schemes, cand_row, pipe):
    """Whether ``pipe`` is a stage-1 result of Eq. 3 for this (c, t): every sequence
    i on exactly one pipeline j of the candidate with MaxLen(P_j) >= l_i (J_i); for an
    infeasible pair (l_0 > MaxLen_0) the only result is the all-0xFF row.  Returns
    (valid, feasible)."""
    ml = [int(schemes["max_len"][k]) for k in cand_row]
    feasible = int(sorted_len[0]) <= ml[0]
    if not feasible:
        return all(int(p) == 0xFF for p in pipe), False
    ok = all(int(p) < len(cand_row) and ml[int(p)] >= int(l) for p, l in zip(pipe, sorted_len))
    return ok, True


def eq2_lb(sorted_len, cost_tab, schemes, cand_row, pipe):
    """Eq. 2 of an assignment: max_j (sum_i m_ij T(l_i, P_j) + T(max l, P_j)(PP_j - 1));
    under sorted order the first member of j is its longest (T non-decreasing in l)."""
    best = 0
    for j, k in enumerate(cand_row):
        idx = [i for i in range(len(pipe)) if int(pipe[i]) == j]
        if not idx:
            continue
        tau = [int(cost_tab[i][k]) for i in idx]
        best = max(best, sum(tau) + max(tau) * (int(schemes["pp"][k]) - 1))
    return best


def pack_pair(sorted_len, cost_tab, schemes, cand_row, pipe):
    """Steps 5-6 of HYD-H1 for one (c, t) whose stage-1 result ``pipe`` [B] is given (any
    assignment, e.g. Alg. 1's or a caller's): (makespan, mb [B], v [32], ptime [32], lb, valid).
    A row that is not an assignment (``is_assignment``) is handled as an infeasible pair:
    makespan and lb UINT64_MAX, mb 0xFFFF, v = ptime = 0."""
    B, k_pad = cost_tab.shape
    ok, feas = is_assignment(sorted_len, schemes, cand_row, pipe)
    v = np.zeros(32, np.uint16)
    pt = np.zeros(32, np.uint64)
    if not (ok and feas):
        return 2**64 - 1, np.full(B, 0xFFFF, np.uint16), v, pt, 2**64 - 1, ok
    row = np.full(32, 0xFF, np.uint8)
    row[: len(cand_row)] = cand_row
    mb = np.empty(B, np.uint16)
    st = C.c_uint32(0)
    ms = lib().hydref_pack_pair(
        np.ascontiguousarray(sorted_len, np.uint32), np.ascontiguousarray(cost_tab, np.uint32).ravel(), B, k_pad,
        _sch_ptr(schemes), row, len(cand_row), np.ascontiguousarray(pipe, np.uint8), mb, v, pt, C.byref(st),
    )
    return int(ms), mb, v, pt, eq2_lb(sorted_len, cost_tab, schemes, cand_row, pipe), True


def select(makespan, cand_offset=0):
    m = np.ascontiguousarray(makespan, np.uint64)
    st = C.c_uint32(0)
    k = lib().hydref_select(m, m.size, int(cand_offset), C.byref(st))
    return int(k), int(st.value)


def assign_batch(W, n_threads=0, cand_offset=0, trials=0, seed=0):
    """All outputs of steps 1-7 for a ``workload.Workload``; dict of numpy arrays.

    ``trials`` > 0 replaces the HYD-H1 dispatch by Alg. 1 with that many random trials
    (NEXT-1, seeded by ``seed``); ``best_trial`` [C][It] is then part of the result."""
    It, B, Cn, kp = W.n_iter, W.batch, W.n_cand, W.k_pad
    o = dict(
        sorted_len=np.empty((It, B), np.uint32),
        perm=np.empty((It, B), np.uint32),
        cost=np.empty((It, B, kp), np.uint32),
        pipe=np.empty((Cn, It, B), np.uint8),
        lb=np.empty((Cn, It), np.uint64),
        mb=np.empty((Cn, It, B), np.uint16),
        v=np.empty((Cn, It, 32), np.uint16),
        ptime=np.empty((Cn, It, 32), np.uint64),
        makespan=np.empty((It, Cn), np.uint64),
        key=np.empty(It, np.int64),
        best_trial=np.full((Cn, It), -1, np.int32),
    )
    st = C.c_uint32(0)
    lib().hydref_assign_batch_ex(
        np.ascontiguousarray(W.lengths, np.uint32), It, B, _sch_ptr(W.schemes), W.n_schemes, kp,
        np.ascontiguousarray(W.cand), np.ascontiguousarray(W.cand_np), Cn, int(cand_offset), int(trials),
        int(seed), o["sorted_len"], o["perm"], o["cost"], o["pipe"], o["lb"], o["mb"], o["v"], o["ptime"],
        o["makespan"], o["key"], o["best_trial"], C.byref(st), int(n_threads),
    )
    o["status"] = int(st.value)
    if not trials:
        del o["best_trial"]
    return o


def cost_tables(W):
    """Steps 1-2 for every iteration of ``W``: (sorted [It][B], perm, cost [It][B][k_pad], status)."""
    It, B, kp = W.n_iter, W.batch, W.k_pad
    s = np.empty((It, B), np.uint32)
    p = np.empty((It, B), np.uint32)
    cst = np.empty((It, B, kp), np.uint32)
    status = 0
    for t in range(It):
        st = C.c_uint32(0)
        lib().hydref_cost_table(
            np.ascontiguousarray(W.lengths[t]), B, _sch_ptr(W.schemes), W.n_schemes, kp, s[t], p[t],
            cst[t].reshape(-1), C.byref(st),
        )
        status |= int(st.value)
    return s, p, cst, status


def assign_pairs(W, pairs_c, pairs_t, tables=None, n_threads=0, trials=0, seed=0):
    """Outputs for selected (c,t) pairs only; rows indexed by pair (``trials`` as assign_batch)."""
    if tables is None:
        tables = cost_tables(W)
    s, _, cst, status = tables
    pc = np.ascontiguousarray(pairs_c, np.int32)
    pt = np.ascontiguousarray(pairs_t, np.int32)
    n, B = pc.size, W.batch
    o = dict(
        pipe=np.empty((n, B), np.uint8),
        lb=np.empty(n, np.uint64),
        mb=np.empty((n, B), np.uint16),
        v=np.empty((n, 32), np.uint16),
        ptime=np.empty((n, 32), np.uint64),
        makespan=np.empty(n, np.uint64),
        best_trial=np.full(n, -1, np.int32),
    )
    st = C.c_uint32(0)
    lib().hydref_assign_pairs_ex(
        s, cst.reshape(-1), W.n_iter, B, W.k_pad, _sch_ptr(W.schemes), np.ascontiguousarray(W.cand),
        np.ascontiguousarray(W.cand_np), pc, pt, n, int(trials), int(seed), o["pipe"], o["lb"], o["mb"],
        o["v"], o["ptime"], o["makespan"], o["best_trial"], C.byref(st), int(n_threads),
    )
    o["status"] = status | int(st.value)
    if not trials:
        del o["best_trial"]
    return o


# ------------------------------------------------------------------ NEXT-1 (alg1ref.c)
def philox4x32_10(ctr, key):
    c = np.ascontiguousarray(ctr, np.uint32)
    k = np.ascontiguousarray(key, np.uint32)
    out = np.empty(4, np.uint32)
    lib().hydref_philox4x32_10(c, k, out)
    return out


def alg1_permutation(seed, t, trial, batch):
    order = np.empty(max(batch, 1), np.uint32)
    lib().hydref_alg1_permutation(int(seed), int(t), int(trial), int(batch), order)
    return order[:batch]


def alg1_trial(sorted_len, cost_tab, schemes, cand_row, order):
    B, k_pad = cost_tab.shape
    row = np.full(32, 0xFF, np.uint8)
    row[: len(cand_row)] = cand_row
    pipe = np.empty(B, np.uint8)
    o = lib().hydref_alg1_trial(
        np.ascontiguousarray(sorted_len, np.uint32), np.ascontiguousarray(cost_tab, np.uint32).ravel(), B, k_pad,
        _sch_ptr(schemes), row, len(cand_row), np.ascontiguousarray(order, np.uint32), pipe,
    )
    return int(o), pipe


def alg1_dispatch(sorted_len, cost_tab, schemes, cand_row, seed, t, trials):
    B, k_pad = cost_tab.shape
    row = np.full(32, 0xFF, np.uint8)
    row[: len(cand_row)] = cand_row
    pipe = np.empty(B, np.uint8)
    lb = C.c_uint64(0)
    bt = C.c_int32(0)
    ok = lib().hydref_alg1_dispatch(
        np.ascontiguousarray(sorted_len, np.uint32), np.ascontiguousarray(cost_tab, np.uint32).ravel(), B, k_pad,
        _sch_ptr(schemes), row, len(cand_row), int(seed), int(t), int(trials), pipe, C.byref(lb), C.byref(bt),
    )
    return bool(ok), pipe, int(lb.value), int(bt.value)


# ------------------------------------------------------------------ NEXT-2 (ragged batches)
def _iteration_workload(W, t):
    """Iteration t of a ragged workload as a one-iteration uniform workload."""
    import workload as wl

    return wl.Workload(W.cfg, W.name, np.ascontiguousarray(W.iteration(t))[None, :], W.schemes, W.cand,
                       W.cand_np, W.k_pad)


def assign_batch_ragged(W, n_threads=0, cand_offset=0):
    """Steps 1-7 on token-budget batches (CSR ``W.offsets``): by definition the uniform method
    applied to each iteration separately (include/hyd.h NEXT-2).  Row layouts as the GPU's:
    sorted_len/perm [N], cost [N][k_pad], pipe/mb [C][N], lb [C][It], v/ptime [C][It][32],
    makespan [It][C], key [It]."""
    It, N, Cn, kp = W.n_iter, W.n_total, W.n_cand, W.k_pad
    off = W.offsets.astype(np.int64)
    o = dict(
        sorted_len=np.empty(N, np.uint32), perm=np.empty(N, np.uint32), cost=np.empty((N, kp), np.uint32),
        pipe=np.empty((Cn, N), np.uint8), lb=np.empty((Cn, It), np.uint64), mb=np.empty((Cn, N), np.uint16),
        v=np.empty((Cn, It, 32), np.uint16), ptime=np.empty((Cn, It, 32), np.uint64),
        makespan=np.empty((It, Cn), np.uint64), key=np.empty(It, np.int64), status=0,
    )
    for t in range(It):
        a, b = off[t], off[t + 1]
        r = assign_batch(_iteration_workload(W, t), n_threads=n_threads, cand_offset=cand_offset)
        o["sorted_len"][a:b] = r["sorted_len"][0]
        o["perm"][a:b] = r["perm"][0]
        o["cost"][a:b] = r["cost"][0]
        o["pipe"][:, a:b] = r["pipe"][:, 0]
        o["mb"][:, a:b] = r["mb"][:, 0]
        o["lb"][:, t] = r["lb"][:, 0]
        o["v"][:, t] = r["v"][:, 0]
        o["ptime"][:, t] = r["ptime"][:, 0]
        o["makespan"][t] = r["makespan"][0]
        o["key"][t] = r["key"][0]
        o["status"] |= r["status"]
    return o


def assign_pairs_ragged(W, pairs_c, pairs_t, n_threads=0):
    """Outputs for selected (c,t) pairs of a ragged workload; row r has the pair's B_t entries."""
    pc = np.asarray(pairs_c, np.int64)
    pt = np.asarray(pairs_t, np.int64)
    out = [None] * pc.size
    for t in np.unique(pt):
        idx = np.nonzero(pt == t)[0]
        Wt = _iteration_workload(W, int(t))
        r = assign_pairs(Wt, pc[idx], np.zeros(idx.size, np.int64), n_threads=n_threads)
        for q, i in enumerate(idx):
            out[i] = {k: r[k][q] for k in ("pipe", "lb", "mb", "v", "ptime", "makespan")}
    return out


# ------------------------------------------------------------------ NEXT-3 (dpref.c)
def dp_prefix(lengths, schemes, step, J):
    x = np.ascontiguousarray(lengths, np.uint32)
    K = len(schemes)
    pre = np.empty((K, J + 1), np.uint64)
    st = C.c_uint32(0)
    lib().hydref_dp_prefix(x, x.size, _sch_ptr(schemes), K, int(step), int(J), pre.reshape(-1), C.byref(st))
    return pre, int(st.value)


def dp_solve(pre, schemes, step, J, n_gpus, scale):
    """The DP table: (t_num, t_den, choice), each [(n_gpus * scale + 1)][J + 1]."""
    NV = n_gpus * scale
    shape = (NV + 1, J + 1)
    tn, td = np.empty(shape, np.uint64), np.empty(shape, np.uint64)
    ch = np.empty(shape, np.int32)
    lib().hydref_dp_solve(np.ascontiguousarray(pre, np.uint64).reshape(-1), _sch_ptr(schemes), len(schemes),
                          int(step), int(J), int(n_gpus), int(scale), tn.reshape(-1), td.reshape(-1),
                          ch.reshape(-1))
    return tn, td, ch


def dp_strategy(choice, t_den, schemes, J, n_gpus, scale, j):
    """S[N][j step]: (feasible, per-scheme d in 1/scale units, scheme of the longest interval)."""
    K = len(schemes)
    counts = np.zeros(K, np.uint32)
    top = C.c_uint32(0)
    ok = lib().hydref_dp_strategy(np.ascontiguousarray(choice, np.int32).reshape(-1),
                                  np.ascontiguousarray(t_den, np.uint64).reshape(-1), _sch_ptr(schemes), K, int(J),
                                  int(n_gpus), int(scale), int(j), counts, C.byref(top))
    return bool(ok), counts, int(top.value)


def dp_round(counts, top_k, schemes, n_gpus, scale, max_round=64):
    """Integer candidates near a relaxed strategy (reading 27): each scheme
    whose d_k (= counts[k] / scale) is not an integer takes floor or ceil -- combination m takes
    the ceiling for the q-th such scheme (ascending k) iff bit q of m is set, m = 0 .. 2^f - 1;
    a combination is kept if it fits in N GPUs and the scheme of the longest interval keeps a
    pipeline.  More than log2(max_round) non-integer schemes: nothing (flagged).  Returns a list
    of (m, per-scheme pipeline counts) for the kept combinations."""
    K = len(counts)
    g = [int(schemes[k]["tp"]) * int(schemes[k]["pp"]) * int(schemes[k]["cp"]) for k in range(K)]
    fr = [k for k in range(K) if int(counts[k]) % scale != 0]
    if 2 ** len(fr) > max_round:
        return None
    out = []
    for m in range(2 ** len(fr)):
        n = [int(counts[k]) // scale for k in range(K)]
        for q, k in enumerate(fr):
            n[k] += (m >> q) & 1
        if sum(n[k] * g[k] for k in range(K)) <= n_gpus and n[top_k] >= 1:
            out.append((m, tuple(n)))
    return out


def dp_propose(lengths, schemes, step, J, n_gpus, scale):
    """The proposed subset: the union over l = step .. J step of the roundings of S[N][l],
    in first-occurrence order over (l, m).  Returns (rows, tables, status)."""
    pre, st = dp_prefix(lengths, schemes, step, J)
    tn, td, ch = dp_solve(pre, schemes, step, J, n_gpus, scale)
    rows = []
    for j in range(1, J + 1):
        ok, counts, top = dp_strategy(ch, td, schemes, J, n_gpus, scale, j)
        if not ok:
            continue
        r = dp_round(counts, top, schemes, n_gpus, scale)
        if r is None:
            st |= 1  # HYDREF_F_OVERFLOW
            continue
        for _, row in r:
            if row not in rows:
                rows.append(row)
    return rows, (pre, tn, td, ch), st


# ------------------------------------------------------------------ NEXT-4 (bbref.c)
def eq3_exact(sorted_len, cost_tab, schemes, cand_row, node_limit=1 << 40):
    """Exact Eq. 3 optimum: (proved, value, pipe, nodes)."""
    B, k_pad = cost_tab.shape
    row = np.full(32, 0xFF, np.uint8)
    row[: len(cand_row)] = cand_row
    pipe = np.zeros(max(B, 1), np.uint8)
    v, n = C.c_uint64(0), C.c_uint64(0)
    ok = lib().hydref_eq3_exact(np.ascontiguousarray(sorted_len, np.uint32),
                                np.ascontiguousarray(cost_tab, np.uint32).ravel(), B, k_pad, _sch_ptr(schemes), row,
                                len(cand_row), int(node_limit), pipe, C.byref(v), C.byref(n))
    return bool(ok), int(v.value), pipe[:B], int(n.value)


def eq1_exact(ell, tau, scheme_row, node_limit=1 << 40):
    """Exact Eq. 1 optimum of one pipeline: (proved, V, obj, nodes)."""
    ell = np.ascontiguousarray(ell, np.uint32)
    tau = np.ascontiguousarray(tau, np.uint32)
    sch = np.ascontiguousarray(np.atleast_1d(scheme_row))
    v, o, n = C.c_uint32(0), C.c_uint64(0), C.c_uint64(0)
    ok = lib().hydref_eq1_exact(ell, tau, ell.size, _sch_ptr(sch), int(node_limit), C.byref(v), C.byref(o), C.byref(n))
    return bool(ok), int(v.value), int(o.value), int(n.value)
