/* oracle/dpref.c -- CPU ORACLE of NEXT-3: the strategy-proposal dynamic programme (§5).
 *
 * TEST INFRASTRUCTURE ONLY (see hydref.h): loaded by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg only; never by the product path.
 *
 * Follows the paper's DP in its notation:
 *   t[n][l] = min( t[n-1][l], min_{(k,d) in Cond_{n,l}, l' < l} T_{k,d,l'} ),
 *   T_{k,d,l'} = max( t[n - d N(P_k)][l - l'], (1/d) sum_{x in D(l-l', l]} T(x, P_k) ),
 *   Cond_{n,l} = {(k, d) : MaxLen(P_k) >= l, d N(P_k) <= n},
 *   t[n][0] = 0 (n >= 0), t[0][l] = inf (l > 0);
 * with lengths on a grid of `step` tokens (l = j step, P:713 footnote: 128) and n, d on a grid
 * of 1/scale GPU (scale 1: the integer DP; scale 10: the continuous relaxation).  All
 * values are exact rationals num/den (num = scale * W, den = d * scale), compared by
 * cross-multiplication in 128 bits.  Readings: the sub-dataset of an interval
 * (l - l', l] is the sequences with lengths in it (lengths above the context are truncated to
 * it); ties keep the earlier option in the order carry (t[n-1][l]), then k, d, l'
 * ascending; the strategy S[n][l] is recovered by following the recorded choices. */
#include <stdlib.h>
#include <string.h>

#include "hydref.h"

typedef unsigned __int128 u128;

/* a < b for rationals (den 0 = infinity) */
static int q_less(uint64_t an, uint64_t ad, uint64_t bn, uint64_t bd) {
  if (bd == 0) return ad != 0;
  if (ad == 0) return 0;
  return (u128)an * bd < (u128)bn * ad;
}

void hydref_dp_prefix(const uint32_t* lengths, int n_seq, const hydref_scheme* schemes, int K,
                      int step, int J, uint64_t* pre, uint32_t* status) {
  /* pre[k][j] = sum over sequences x with min(x, J step) <= j step of T(min(x, J step), P_k) */
  const uint32_t lmax = (uint32_t)J * (uint32_t)step;
  memset(pre, 0, sizeof(uint64_t) * (size_t)K * (size_t)(J + 1));
  for (int k = 0; k < K; ++k) {
    uint64_t* p = pre + (size_t)k * (J + 1);
    for (int i = 0; i < n_seq; ++i) {
      const uint32_t x = lengths[i] < lmax ? lengths[i] : lmax; /* truncated to the context */
      const int j = (int)((x + (uint32_t)step - 1u) / (uint32_t)step); /* x in ((j-1)step, j step] */
      p[j] += hydref_cost(&schemes[k], x, status);
    }
    for (int j = 1; j <= J; ++j) p[j] += p[j - 1];
  }
}

int hydref_dp_solve(const uint64_t* pre, const hydref_scheme* schemes, int K, int step, int J,
                    int n_gpus, int scale, uint64_t* t_num, uint64_t* t_den, int32_t* choice) {
  const int NV = n_gpus * scale; /* n = nu / scale, d = mu / scale */
  uint32_t gk[64];
  for (int k = 0; k < K; ++k) gk[k] = schemes[k].tp * schemes[k].pp * schemes[k].cp; /* N(P_k) */
#define T_AT(nu, j) ((size_t)(nu) * (size_t)(J + 1) + (size_t)(j))
  for (int nu = 0; nu <= NV; ++nu) {
    t_num[T_AT(nu, 0)] = 0;
    t_den[T_AT(nu, 0)] = 1;
    choice[T_AT(nu, 0)] = -2; /* base state */
  }
  for (int j = 1; j <= J; ++j) {
    t_num[T_AT(0, j)] = 1;
    t_den[T_AT(0, j)] = 0; /* infinity */
    choice[T_AT(0, j)] = -2;
  }
  for (int nu = 1; nu <= NV; ++nu) {
    for (int j = 1; j <= J; ++j) {
      /* option t[n-1][l]: "up to n GPUs" */
      uint64_t bn = t_num[T_AT(nu - 1, j)], bd = t_den[T_AT(nu - 1, j)];
      int32_t bc = -1;
      const uint32_t l = (uint32_t)j * (uint32_t)step;
      for (int k = 0; k < K; ++k) {
        if (schemes[k].max_len < l) continue; /* MaxLen(P_k) >= l */
        for (int mu = 1; (uint64_t)mu * gk[k] <= (uint64_t)nu; ++mu) {
          const int nrest = nu - mu * (int)gk[k];
          for (int jp = 1; jp <= j; ++jp) {
            const uint64_t W = pre[(size_t)k * (J + 1) + j] - pre[(size_t)k * (J + 1) + (j - jp)];
            /* (1/d) W = scale W / mu */
            uint64_t vn = (uint64_t)scale * W, vd = (uint64_t)mu;
            const uint64_t rn = t_num[T_AT(nrest, j - jp)], rd = t_den[T_AT(nrest, j - jp)];
            if (q_less(vn, vd, rn, rd)) { /* max(t[rest], W/d) */
              vn = rn;
              vd = rd;
            }
            if (q_less(vn, vd, bn, bd)) {
              bn = vn;
              bd = vd;
              bc = (int32_t)(((uint32_t)k << 24) | ((uint32_t)mu << 12) | (uint32_t)jp);
            }
          }
        }
      }
      t_num[T_AT(nu, j)] = bn;
      t_den[T_AT(nu, j)] = bd;
      choice[T_AT(nu, j)] = bc;
    }
  }
#undef T_AT
  return 0;
}

int hydref_dp_strategy(const int32_t* choice, const uint64_t* t_den, const hydref_scheme* schemes,
                       int K, int J, int n_gpus, int scale, int j, uint32_t* counts,
                       uint32_t* top_k) {
  /* S[N][l = j step]: per scheme, the summed d (in units of 1/scale) over its intervals;
   * *top_k = the scheme of the interval holding the longest lengths.  Returns 0 if t = inf. */
  int nu = n_gpus * scale;
  for (int k = 0; k < K; ++k) counts[k] = 0;
  *top_k = 0xFFFFFFFFu;
  if (t_den[(size_t)nu * (J + 1) + j] == 0) return 0;
  while (j > 0) {
    const int32_t c = choice[(size_t)nu * (J + 1) + j];
    if (c == -1) {
      nu -= 1;
      continue;
    }
    const uint32_t k = (uint32_t)c >> 24, mu = ((uint32_t)c >> 12) & 0xFFFu, jp = (uint32_t)c & 0xFFFu;
    if (*top_k == 0xFFFFFFFFu) *top_k = k;
    counts[k] += mu;
    nu -= (int)(mu * schemes[k].tp * schemes[k].pp * schemes[k].cp);
    j -= (int)jp;
  }
  return 1;
}
