"""Pure-Python exhaustive solvers for tiny instances (test-only, independent of oracle/).

These compute the TRUE optima of the paper's problems, by enumeration:
  * Eq. 1: for one pipeline and a V range, the min over all
    partitions of its sequences into V non-empty micro-batches with
    sum(l) <= MaxLen of  max_b sum T(l) * (PP - 1 + V).
  * Two-stage optimum: min over every dispatch m_ij respecting MaxLen
    of max_j [Eq. 1 optimum of pipeline j over V in App. D's range, P:1097].
  * Eq. 3: min over dispatches of max_j LowerBound_j (Eq. 2).
Costs use Python big integers on the closed form of App. C.2.
"""
from __future__ import annotations

import itertools
from functools import lru_cache


def _rec(scheme):
    return scheme[0] if getattr(scheme, "ndim", 0) > 0 else scheme


def T(scheme, l):
    """floor((a l^2 + b l + c) / 2^32), exact (App. C.2, Q32 reading)."""
    scheme = _rec(scheme)
    return (int(scheme["a_q32"]) * l * l + int(scheme["b_q32"]) * l + int(scheme["c_q32"])) >> 32


def set_partitions(items, v):
    """All partitions of ``items`` (tuple) into exactly ``v`` non-empty blocks."""
    n = len(items)
    if v < 1 or v > n:
        return
    # restricted growth strings
    def rec(i, labels, m):
        if i == n:
            if m == v:
                blocks = [[] for _ in range(v)]
                for it, lab in zip(items, labels):
                    blocks[lab].append(it)
                yield blocks
            return
        if v - m > n - i:
            return
        for lab in range(min(m + 1, v)):
            labels.append(lab)
            yield from rec(i + 1, labels, max(m, lab + 1))
            labels.pop()

    yield from rec(0, [], 0)


def v_range(lengths, scheme):
    """App. D range with SURVEY §8(c) reading 5 (ceil/floor, clamp)."""
    scheme = _rec(scheme)
    U = len(lengths)
    S = sum(lengths)
    M = int(scheme["max_len"])
    lo = max(-(-S // M), 1)
    ul = int(scheme["util_len"])
    hi = U if ul == 0 else min(S // ul, U)
    return lo, max(hi, lo)


def pack_opt(lengths, scheme, vs):
    """min over V in ``vs`` and capacity-feasible partitions of Eq. 1's objective; None if none."""
    scheme = _rec(scheme)
    M, P = int(scheme["max_len"]), int(scheme["pp"])
    best = None
    items = tuple(lengths)
    for v in vs:
        for blocks in set_partitions(items, v):
            if any(sum(b) > M for b in blocks):
                continue
            obj = max(sum(T(scheme, l) for l in b) for b in blocks) * (P - 1 + v)
            if best is None or obj < best:
                best = obj
    return best


def lower_bound(lengths, scheme):
    """Eq. 2: sum T(l) + T(max l) (PP - 1); 0 for an empty set."""
    scheme = _rec(scheme)
    if not lengths:
        return 0
    return sum(T(scheme, l) for l in lengths) + T(scheme, max(lengths)) * (int(scheme["pp"]) - 1)


def two_stage_opt(lengths, schemes, cand_row, full_v=False):
    """Exhaustive optimum of dispatch + packing (the problem the heuristic approximates).

    With ``full_v`` the V range is [1, U] instead of App. D's pruned range.
    Returns (opt_makespan, opt_eq3) where opt_eq3 is the Eq. 3 optimum.
    """
    D = len(cand_row)
    sch = [schemes[k] for k in cand_row]

    @lru_cache(maxsize=None)
    def pipe_cost(j, subset):
        ls = list(subset)
        if not ls:
            return 0
        if full_v:
            vs = range(1, len(ls) + 1)
        else:
            lo, hi = v_range(ls, sch[j])
            vs = list(range(lo, hi + 1))
            r = pack_opt(ls, sch[j], vs)
            if r is None:  # reading 5: extend upward on infeasibility
                vs = range(hi + 1, len(ls) + 1)
            else:
                return r
        r = pack_opt(ls, sch[j], vs)
        return r if r is not None else float("inf")

    best = float("inf")
    best_lb = float("inf")
    B = len(lengths)
    for assign in itertools.product(range(D), repeat=B):
        if any(lengths[i] > int(sch[assign[i]]["max_len"]) for i in range(B)):
            continue
        groups = [tuple(sorted(lengths[i] for i in range(B) if assign[i] == j)) for j in range(D)]
        ms = max(pipe_cost(j, groups[j]) for j in range(D))
        lb = max(lower_bound(list(groups[j]), sch[j]) for j in range(D))
        best = min(best, ms)
        best_lb = min(best_lb, lb)
    return best, best_lb


def makespan_opt_identical(costs, m):
    """Exact multiprocessor scheduling optimum on ``m`` identical machines."""
    best = float("inf")
    for assign in itertools.product(range(m), repeat=len(costs)):
        loads = [0] * m
        for c, a in zip(costs, assign):
            loads[a] += c
        best = min(best, max(loads))
    return best


def eq3_opt(lengths, schemes, cand_row):
    """Eq. 3 optimum: min over every dispatch respecting MaxLen of
    max_j LowerBound_j (Eq. 2), by enumeration of all D^B assignments."""
    D = len(cand_row)
    sch = [schemes[k] for k in cand_row]
    B = len(lengths)
    best = float("inf")
    for assign in itertools.product(range(D), repeat=B):
        if any(lengths[i] > int(sch[assign[i]]["max_len"]) for i in range(B)):
            continue
        o = max(lower_bound([lengths[i] for i in range(B) if assign[i] == j], sch[j]) for j in range(D))
        best = min(best, o)
    return best
