"""Pins of the NEXT-3 oracle (oracle/dpref.c): the strategy-proposal DP of §5.

* the prefix sums against direct sums of the closed-form cost (App. C.2) per interval;
* t[n][l] against exhaustive enumeration of every split of (0, l] into consecutive length
  intervals with a (scheme, d) per interval (the restricted problem the DP solves),
  for the integer DP and the 0.1-step relaxation;
* one scheme of one GPU per pipeline: t[n][L] = W / n (mediant argument) exactly;
* monotonicity in n and l; the relaxation is never worse than the integer DP;
* the recovered strategy S[N][l] uses at most N GPUs and reproduces t[N][l];
* rounding (reading 27) keeps every candidate within N GPUs.
"""
import itertools
from fractions import Fraction

import numpy as np
import pytest

import oracle
import workload as w
from tests import bruteforce as bf


def gpus(s):
    return int(s["tp"]) * int(s["pp"]) * int(s["cp"])


def tiny_instance(rng, K=3, J=4, step=64):
    sch = np.zeros(K, dtype=w.SCHEME_DTYPE)
    for k in range(K):
        sch[k]["tp"] = int(rng.integers(1, 3))
        sch[k]["pp"] = int(rng.integers(1, 3))
        sch[k]["cp"] = 1
        sch[k]["max_len"] = int(rng.choice([step, 2 * step, J * step, J * step + 5]))
        sch[k]["a_q32"] = int(rng.integers(0, 4)) << 24
        sch[k]["b_q32"] = int(rng.integers(1, 5)) << 32
        sch[k]["c_q32"] = int(rng.integers(0, 30)) << 32
    sch[0]["max_len"] = J * step  # someone holds the longest lengths
    lens = rng.integers(1, J * step + 50, int(rng.integers(3, 25))).astype(np.uint32)
    return sch, lens


def brute_t(lens, sch, step, j_top, n_gpus, scale, J):
    """min over splits of (0, j_top step] and (k, mu) per interval of max_i scale W_i / mu_i
    (lengths truncated to the context J step)."""
    Lmax = J * step
    best = None
    for cuts in itertools.product([0, 1], repeat=j_top - 1):
        bounds = [0] + [b + 1 for b, c in enumerate(cuts) if c] + [j_top]
        ivs = list(zip(bounds[:-1], bounds[1:]))
        opts = []
        for a, b in ivs:
            o = []
            for k in range(len(sch)):
                if int(sch[k]["max_len"]) < b * step:
                    continue
                Wk = sum(bf.T(sch[k], min(int(x), Lmax)) for x in lens
                         if a * step < min(int(x), Lmax) <= b * step)
                for mu in range(1, n_gpus * scale // gpus(sch[k]) + 1):
                    o.append((k, mu, Fraction(scale * Wk, mu)))
            opts.append(o)
        for choice in itertools.product(*opts):
            if sum(mu * gpus(sch[k]) for k, mu, _ in choice) > n_gpus * scale:
                continue
            v = max(val for _, _, val in choice)
            if best is None or v < best:
                best = v
    return best


def frac(tn, td):
    return None if int(td) == 0 else Fraction(int(tn), int(td))


def test_prefix_sums_are_interval_sums():
    rng = np.random.default_rng(1)
    sch, lens = tiny_instance(rng, K=4, J=6)
    pre, st = oracle.dp_prefix(lens, sch, 64, 6)
    assert st == 0
    Lmax = 6 * 64
    for k in range(4):
        for j in range(7):
            direct = sum(bf.T(sch[k], min(int(x), Lmax)) for x in lens if min(int(x), Lmax) <= j * 64)
            assert int(pre[k, j]) == direct


@pytest.mark.parametrize("scale", [1, 10])
def test_dp_equals_exhaustive_interval_search(scale):
    rng = np.random.default_rng(7 + scale)
    n_cases = 0
    for _ in range(6 if scale == 1 else 3):
        J = int(rng.integers(2, 4))
        sch, lens = tiny_instance(rng, K=2, J=J)
        N = int(rng.integers(1, 4)) if scale == 1 else 2
        pre, _ = oracle.dp_prefix(lens, sch, 64, J)
        tn, td, ch = oracle.dp_solve(pre, sch, 64, J, N, scale)
        for n in range(1, N + 1):
            for j in range(1, J + 1):
                assert frac(tn[n * scale, j], td[n * scale, j]) == brute_t(lens, sch, 64, j, n, scale, J), (n, j)
        n_cases += 1
    assert n_cases >= 3


def test_single_unit_scheme_closed_form():
    rng = np.random.default_rng(3)
    for _ in range(5):
        sch = w.make_scheme(pp=1, max_len=4096, a_q32=int(rng.integers(0, 9)) << 20,
                            b_q32=int(rng.integers(1, 9)) << 32, c_q32=int(rng.integers(0, 99)) << 32)
        lens = rng.integers(1, 4096, 200).astype(np.uint32)
        pre, _ = oracle.dp_prefix(lens, sch, 256, 16)
        W = sum(bf.T(sch, int(x)) for x in lens)
        for scale in (1, 10):
            tn, td, _ = oracle.dp_solve(pre, sch, 256, 16, 6, scale)
            for n in range(1, 7):
                assert frac(tn[n * scale, 16], td[n * scale, 16]) == Fraction(W, n)


def test_monotone_and_relaxation_not_worse():
    W = w.make_workload(4, n_cand=2, n_iter=4)
    lens = W.lengths.reshape(-1)
    J, step, N = 16, 2048, 16
    pre, _ = oracle.dp_prefix(lens, W.schemes, step, J)
    tn1, td1, _ = oracle.dp_solve(pre, W.schemes, step, J, N, 1)
    tn10, td10, _ = oracle.dp_solve(pre, W.schemes, step, J, N, 10)
    INF = None
    for n in range(1, N + 1):
        for j in range(1, J + 1):
            a = frac(tn1[n, j], td1[n, j])
            b = frac(tn10[10 * n, j], td10[10 * n, j])
            assert a is INF or (b is not INF and b <= a)  # finer grid contains the integer one
            if n > 1:
                p = frac(tn1[n - 1, j], td1[n - 1, j])
                assert a is INF or (p is INF or a <= p)  # more GPUs never hurt
            if j > 1:
                q = frac(tn1[n, j - 1], td1[n, j - 1])
                assert a is INF or (q is not INF and q <= a)  # more sequences never help


def test_strategy_reproduces_objective_and_rounding_budget():
    W = w.make_workload(4, n_cand=2, n_iter=6)
    lens = W.lengths.reshape(-1)
    J, step, N = 16, 2048, 64
    for scale in (1, 10):
        rows, (pre, tn, td, ch), st = oracle.dp_propose(lens, W.schemes, step, J, N, scale)
        assert st == 0 and rows
        g = np.array([gpus(s) for s in W.schemes])
        for j in range(1, J + 1):
            ok, counts, top = oracle.dp_strategy(ch, td, W.schemes, J, N, scale, j)
            assert ok
            assert int((counts * g).sum()) <= N * scale
            assert int(W.schemes[top]["max_len"]) >= j * step
            # replay the recorded choices: the intervals' max (1/d) W equals t[N][l], the GPUs fit
            nu, jj, vals, used = N * scale, j, [], 0
            while jj > 0:
                c = int(ch[nu, jj])
                if c == -1:
                    nu -= 1
                    continue
                k, mu, jp = c >> 24, (c >> 12) & 0xFFF, c & 0xFFF
                assert int(W.schemes[k]["max_len"]) >= jj * step
                vals.append(Fraction(scale * (int(pre[k, jj]) - int(pre[k, jj - jp])), mu))
                used += mu * g[k]
                nu -= mu * g[k]
                jj -= jp
            assert max(vals) == frac(tn[N * scale, j], td[N * scale, j]) and used <= N * scale
        for r in rows:
            assert int((np.array(r) * g).sum()) <= N and sum(r) >= 1


def test_round_hand_worked():
    """Reading 27 ("round and adjust to include all nearby integer solutions") by hand.
    Schemes: k0 = <2,1,1> (2 GPUs), k1 = <4,1,1> (4 GPUs), k2 = <1,1,1> (1 GPU); scale 10.
    d = (1.5, 2.3, 1.0): k0 and k1 are non-integer (q = 0, 1), k2 stays 1.  Combinations
      m=0 floor/floor (1,2,1): 2+8+1 = 11 GPUs;  m=1 ceil k0 (2,2,1): 13;
      m=2 ceil k1 (1,3,1): 15;  m=3 both (2,3,1): 17.
    With N = 16 GPUs and top scheme k1: m = 0, 1, 2 kept, m = 3 over budget.
    d = (1.5, 0.7, 1.0), top k1: floor(0.7) = 0 drops the top scheme (m = 0, 1); m=2 (1,1,1) = 7
    and m=3 (2,1,1) = 9 GPUs -> N = 8 keeps only m = 2, N = 9 keeps m = 2, 3.
    Seven non-integer schemes need 2^7 = 128 > 64 combinations: nothing (flagged)."""
    sch = np.concatenate([w.make_scheme(tp=2, max_len=4096, b_q32=1 << 32), w.make_scheme(tp=4, max_len=8192, b_q32=1 << 32),
                          w.make_scheme(tp=1, max_len=2048, b_q32=1 << 32)])
    got = oracle.dp_round([15, 23, 10], 1, sch, 16, 10)
    assert got == [(0, (1, 2, 1)), (1, (2, 2, 1)), (2, (1, 3, 1))]
    assert oracle.dp_round([15, 7, 10], 1, sch, 8, 10) == [(2, (1, 1, 1))]
    assert oracle.dp_round([15, 7, 10], 1, sch, 9, 10) == [(2, (1, 1, 1)), (3, (2, 1, 1))]
    sch7 = np.concatenate([w.make_scheme(max_len=1000 + k, b_q32=1 << 32) for k in range(7)])
    assert oracle.dp_round([5] * 7, 0, sch7, 64, 10) is None
