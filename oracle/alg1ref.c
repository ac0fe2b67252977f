/* oracle/alg1ref.c -- CPU ORACLE of NEXT-1: the paper's randomized greedy dispatcher (Alg. 1).
 *
 * TEST INFRASTRUCTURE ONLY (see hydref.h): loaded by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg only; never by the product path.
 *
 * Follows Alg. 1 (described at P:1201) line by line:
 *   for trial = 1..T:  random permutation pi (line 2); C_j = E_j = m_ij = 0 (line 3);
 *     for k = 1..B: i = pi_k (line 5); for j = 1..J_i (line 6):
 *       l_max = max(l_i, max_i' m_i'j l_i')                  (line 7; "l_j" read as l_i, reading 8)
 *       C_j' = C_j + T(l_i, P_j)                               (line 8)
 *       E_j' = T(l_max, P_j) (PP(P_j) - 1)                     (line 9)
 *       O_max = max(C_j' + E_j', C_k + E_k for k != j)         (line 10; all k, empty = 0, reading 9)
 *       if O_max < O_min: O_min = O_max, j* = j                (lines 11-12: strict, first j wins)
 *     m_ij* = 1, C_j* = C_j*', E_j* = E_j*'                    (line 13)
 *   O_trial = max_j (C_j + E_j); keep the trial if O_trial < O_best (lines 15-17: strict, so
 *   the smallest trial index wins ties).
 * The random permutation is the counter-based Fisher-Yates of hydref.h (reading 21).
 * Parity pins: tests/test_alg1_oracle.py (Philox known-answer vectors, a literal Python
 * transcription of the pseudo-code, brute-force optimum dominance, T-monotonicity). */
#include <stdlib.h>
#include <string.h>

#include "hydref.h"

/* ---------------------------------------------------------------- Philox4x32-10
 * Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy as 1, 2, 3" (SC'11):
 * round: (hi0, lo0) = M0 * x0, (hi1, lo1) = M1 * x2;
 *        x' = (hi1 ^ x1 ^ k0, lo1, hi0 ^ x3 ^ k1, lo0); key bumped by the Weyl constants
 *        between rounds. */
#define PHILOX_M0 0xD2511F53u
#define PHILOX_M1 0xCD9E8D57u
#define PHILOX_W0 0x9E3779B9u
#define PHILOX_W1 0xBB67AE85u

void hydref_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t x0 = ctr[0], x1 = ctr[1], x2 = ctr[2], x3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) {
      k0 += PHILOX_W0;
      k1 += PHILOX_W1;
    }
    uint64_t p0 = (uint64_t)PHILOX_M0 * x0;
    uint64_t p1 = (uint64_t)PHILOX_M1 * x2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t y0 = hi1 ^ x1 ^ k0, y1 = lo1, y2 = hi0 ^ x3 ^ k1, y3 = lo0;
    x0 = y0;
    x1 = y1;
    x2 = y2;
    x3 = y3;
  }
  out[0] = x0;
  out[1] = x1;
  out[2] = x2;
  out[3] = x3;
}

/* ---------------------------------------------------------------- line 2: permutation */
void hydref_alg1_permutation(uint64_t seed, int t, int trial, int batch, uint32_t* order) {
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  for (int i = 0; i < batch; ++i) order[i] = (uint32_t)i;
  for (int k = batch - 1; k >= 1; --k) {
    const uint32_t ctr[4] = {(uint32_t)k / 4u, (uint32_t)t, (uint32_t)trial, 0u};
    uint32_t r[4];
    hydref_philox4x32_10(ctr, key, r);
    const uint32_t j = (uint32_t)(((uint64_t)r[k % 4] * (uint64_t)(k + 1)) >> 32);
    const uint32_t tmp = order[k];
    order[k] = order[j];
    order[j] = tmp;
  }
}

/* ---------------------------------------------------------------- lines 3-15: one trial */
uint64_t hydref_alg1_trial(const uint32_t* sorted, const uint32_t* cost, int batch, int k_pad,
                           const hydref_scheme* schemes, const uint8_t* cand_row, int np,
                           const uint32_t* order, uint8_t* pipe) {
  uint64_t C[32], E[32];
  uint32_t lmax[32]; /* max_i m_ij l_i: the longest sequence already on pipeline j (0: none) */
  uint32_t st = 0;
  for (int j = 0; j < np; ++j) {
    C[j] = 0;
    E[j] = 0;
    lmax[j] = 0;
  }
  for (int k = 0; k < batch; ++k) {
    const uint32_t i = order[k];
    const uint32_t l = sorted[i];
    int jstar = -1;
    uint64_t omin = UINT64_MAX, cs = 0, es = 0;
    uint32_t ls = 0;
    for (int j = 0; j < np; ++j) {
      const hydref_scheme* P = &schemes[cand_row[j]];
      if (P->max_len < l) continue; /* j > J_i: MaxLen(P_j) < l_i */
      const uint32_t lm = lmax[j] > l ? lmax[j] : l;
      const uint64_t cj = C[j] + cost[(size_t)i * k_pad + cand_row[j]];
      const uint64_t ej = (uint64_t)hydref_cost(P, lm, &st) * (uint64_t)(P->pp - 1u);
      uint64_t omax = cj + ej;
      for (int q = 0; q < np; ++q)
        if (q != j && C[q] + E[q] > omax) omax = C[q] + E[q];
      if (omax < omin) {
        omin = omax;
        jstar = j;
        cs = cj;
        es = ej;
        ls = lm;
      }
    }
    /* jstar >= 0 whenever l <= MaxLen(P_0), which the caller checked for sorted[0] */
    pipe[i] = (uint8_t)jstar;
    C[jstar] = cs;
    E[jstar] = es;
    lmax[jstar] = ls;
  }
  uint64_t o = 0;
  for (int j = 0; j < np; ++j)
    if (C[j] + E[j] > o) o = C[j] + E[j];
  return o;
}

/* ---------------------------------------------------------------- lines 1-18: T trials */
int hydref_alg1_dispatch(const uint32_t* sorted, const uint32_t* cost, int batch, int k_pad,
                         const hydref_scheme* schemes, const uint8_t* cand_row, int np,
                         uint64_t seed, int t, int trials, uint8_t* pipe, uint64_t* lb,
                         int32_t* best_trial) {
  if (batch > 0 && sorted[0] > schemes[cand_row[0]].max_len) {
    memset(pipe, 0xFF, (size_t)batch);
    *lb = UINT64_MAX;
    if (best_trial) *best_trial = -1;
    return 0;
  }
  size_t n = (size_t)(batch > 0 ? batch : 1);
  uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint8_t* trial_pipe = (uint8_t*)malloc(n);
  uint64_t obest = UINT64_MAX;
  int tbest = -1;
  for (int trial = 0; trial < trials; ++trial) {
    hydref_alg1_permutation(seed, t, trial, batch, order);
    const uint64_t o = hydref_alg1_trial(sorted, cost, batch, k_pad, schemes, cand_row, np, order,
                                         trial_pipe);
    if (o < obest) { /* line 16: strict */
      obest = o;
      tbest = trial;
      memcpy(pipe, trial_pipe, (size_t)batch);
    }
  }
  free(order);
  free(trial_pipe);
  *lb = obest;
  if (best_trial) *best_trial = tbest;
  return 1;
}

/* ---------------------------------------------------------------- steps 4-6 with Alg. 1 */
uint64_t hydref_alg1_assign_pair(const uint32_t* sorted, const uint32_t* cost, int batch,
                                 int k_pad, const hydref_scheme* schemes, const uint8_t* cand_row,
                                 int np, uint64_t seed, int t, int trials, uint8_t* pipe,
                                 uint64_t* lb, uint16_t* mb, uint16_t* v, uint64_t* ptime,
                                 int32_t* best_trial, uint32_t* status) {
  for (int j = 0; j < 32; ++j) {
    v[j] = 0;
    ptime[j] = 0;
  }
  if (!hydref_alg1_dispatch(sorted, cost, batch, k_pad, schemes, cand_row, np, seed, t, trials,
                            pipe, lb, best_trial)) {
    for (int i = 0; i < batch; ++i) mb[i] = 0xFFFF;
    return UINT64_MAX;
  }
  return hydref_pack_pair(sorted, cost, batch, k_pad, schemes, cand_row, np, pipe, mb, v, ptime,
                          status);
}
