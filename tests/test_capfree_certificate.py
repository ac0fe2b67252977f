"""The capacity-free certificate of the pack lanes, checked on its own terms.

Claim: with alpha = min_i tau_i / l_i over the sequences a scheme can hold and
cap = floor(alpha * MaxLen), an LPT(V) run whose abort threshold thr satisfies thr <= cap makes
the same choices with and without the MaxLen mask, and fails (running maximum bin time > thr, or
no micro-batch fits) at the same sequence.  Plain Python runs of both rules (Eq. 1's LPT, P:604-607,
as in the oracle) on random instances with tight MaxLen; the negative control shows the two rules
do differ once thr exceeds cap, so the equality is not vacuous.
"""
import numpy as np


def lpt_abort(ell, tau, V, M, thr, capped):
    """LPT over the sequences in the given order: least-time bin (smallest index on ties) among
    those whose tokens stay within M (capped) or among all bins; abort when the running maximum
    exceeds thr.  Returns (status, step, assignment prefix)."""
    t = [0] * V
    tok = [0] * V
    mx = 0
    out = []
    for q, (l, ta) in enumerate(zip(ell, tau)):
        best = -1
        for b in range(V):
            if capped and tok[b] + l > M:
                continue
            if best < 0 or t[b] < t[best]:
                best = b
        if best < 0:
            return "fail", q, out
        t[best] += ta
        tok[best] += l
        mx = max(mx, t[best])
        out.append(best)
        if mx > thr:
            return "fail", q, out
    return "done", len(ell), out


def instance(rng):
    M = int(rng.integers(200, 2000))
    a, b, c = int(rng.integers(0, 3)), int(rng.integers(1, 9)), int(rng.integers(0, 400))
    n = int(rng.integers(4, 40))
    ell = sorted((int(x) for x in rng.integers(1, M + 1, n)), reverse=True)
    tau = [(a * l * l) // 64 + b * l + c for l in ell]
    alpha_num, alpha_den = min(((tu, l) for tu, l in zip(tau, ell)), key=lambda p: p[0] / p[1])
    cap = alpha_num * M // alpha_den
    V = int(rng.integers(1, 9))
    return ell, tau, M, V, cap


def test_capfree_equals_masked_below_cap():
    rng = np.random.default_rng(2412)
    checked = 0
    for _ in range(3000):
        ell, tau, M, V, cap = instance(rng)
        for thr in (cap, cap - 1, cap // 2, int(rng.integers(0, cap + 1))):
            if thr < 0:
                continue
            st_c, q_c, a_c = lpt_abort(ell, tau, V, M, thr, True)
            st_f, q_f, a_f = lpt_abort(ell, tau, V, M, thr, False)
            # same outcome at the same sequence, same choices before it (a failed run's own last
            # placement is never used: the lanes discard failed runs, and only runs that complete
            # write micro-batch ids)
            assert (st_c, q_c, a_c[:q_c]) == (st_f, q_f, a_f[:q_f])
            checked += 1
    assert checked > 10000


def lpt_mixed(ell, tau, V, M, thr, masked_steps):
    """A capacity-free unit whose warp runs some steps on the masked path: the masked steps test
    and update the bins' token counts, the capacity-free ones leave them stale."""
    t = [0] * V
    rem = [M] * V
    mx = 0
    out = []
    for q, (l, ta) in enumerate(zip(ell, tau)):
        best = -1
        for b in range(V):
            if masked_steps[q] and rem[b] < l:
                continue
            if best < 0 or t[b] < t[best]:
                best = b
        if best < 0:
            return "fail", q, out
        t[best] += ta
        if masked_steps[q]:
            rem[best] -= l
        mx = max(mx, t[best])
        out.append(best)
        if mx > thr:
            return "fail", q, out
    return "done", len(ell), out


def test_stale_token_counts_are_harmless_below_cap():
    """A warp takes the masked path when any of its units needs it; the capacity-free units then
    run masked steps on token counts that missed their capacity-free steps (never smaller than the
    true ones), which still picks the same bins below cap."""
    rng = np.random.default_rng(11)
    for _ in range(2000):
        ell, tau, M, V, cap = instance(rng)
        thr = int(rng.integers(0, cap + 1))
        modes = [bool(x) for x in rng.integers(0, 2, len(ell))]
        st_c, q_c, a_c = lpt_abort(ell, tau, V, M, thr, True)
        st_m, q_m, a_m = lpt_mixed(ell, tau, V, M, thr, modes)
        assert (st_c, q_c, a_c[:q_c]) == (st_m, q_m, a_m[:q_m])


def test_rules_differ_above_cap():
    """Negative control: with no threshold (thr = infinity) the capacity mask matters."""
    rng = np.random.default_rng(7)
    differ = 0
    for _ in range(3000):
        ell, tau, M, V, cap = instance(rng)
        if lpt_abort(ell, tau, V, M, 1 << 62, True) != lpt_abort(ell, tau, V, M, 1 << 62, False):
            differ += 1
    assert differ > 0
