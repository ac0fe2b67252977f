/* oracle/bbref.c -- CPU ORACLE of NEXT-4: the exact optimum of Eq. 3 for small instances.
 *
 * TEST INFRASTRUCTURE ONLY (see hydref.h): loaded by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg only; never by the product path.
 *
 * Eq. 3: minimise over dispatch matrices m_ij (each sequence on one pipeline with
 * MaxLen(P_j) >= l_i) the largest pipeline lower bound
 *   LB_j = sum_{i on j} T(l_i, P_j) + T(max_{i on j} l_i, P_j) (PP_j - 1)      (Eq. 2).
 * Plain depth-first enumeration of every assignment, sequences in the given order, pruned only
 * by "the partial maximum already reaches the incumbent" (partial LB_j never decrease as
 * sequences are added, so pruning cannot lose an optimum).  E_j uses the largest length
 * assigned so far, computed from the closed-form cost.  The returned assignment is the first
 * optimum found in lexicographic (pipeline index) order. */
#include <stdlib.h>
#include <string.h>

#include "hydref.h"

typedef struct {
  const uint32_t* sorted;
  const uint32_t* cost;
  int B, k_pad, np;
  const hydref_scheme* P[32];
  uint32_t k[32];
  uint64_t C[32];
  uint32_t lmax[32];
  uint8_t cur[64], best_pipe[64];
  uint64_t best;
  uint64_t nodes, limit;
  int exhausted;
} bb_t;

static uint64_t lb_of(bb_t* s, int j, uint64_t C, uint32_t lmax) {
  uint32_t st = 0;
  if (lmax == 0) return 0;
  return C + (uint64_t)hydref_cost(s->P[j], lmax, &st) * (uint64_t)(s->P[j]->pp - 1u);
}

static void dfs(bb_t* s, int i, uint64_t partial_max) {
  if (s->exhausted) return;
  if (++s->nodes > s->limit) {
    s->exhausted = 1;
    return;
  }
  if (i == s->B) {
    if (partial_max < s->best) {
      s->best = partial_max;
      memcpy(s->best_pipe, s->cur, (size_t)s->B);
    }
    return;
  }
  const uint32_t l = s->sorted[i];
  for (int j = 0; j < s->np; ++j) {
    if (s->P[j]->max_len < l) continue;
    const uint64_t C0 = s->C[j];
    const uint32_t m0 = s->lmax[j];
    const uint64_t C1 = C0 + s->cost[(size_t)i * s->k_pad + s->k[j]];
    const uint32_t m1 = l > m0 ? l : m0;
    const uint64_t v = lb_of(s, j, C1, m1);
    const uint64_t nm = v > partial_max ? v : partial_max;
    if (nm >= s->best) continue; /* cannot improve the incumbent */
    s->C[j] = C1;
    s->lmax[j] = m1;
    s->cur[i] = (uint8_t)j;
    dfs(s, i + 1, nm);
    s->C[j] = C0;
    s->lmax[j] = m0;
  }
}

int hydref_eq3_exact(const uint32_t* sorted, const uint32_t* cost, int batch, int k_pad,
                     const hydref_scheme* schemes, const uint8_t* cand_row, int np,
                     uint64_t node_limit, uint8_t* pipe, uint64_t* value, uint64_t* nodes) {
  bb_t* s = (bb_t*)calloc(1, sizeof(bb_t));
  s->sorted = sorted;
  s->cost = cost;
  s->B = batch;
  s->k_pad = k_pad;
  s->np = np;
  for (int j = 0; j < np; ++j) {
    s->k[j] = cand_row[j];
    s->P[j] = &schemes[cand_row[j]];
  }
  s->best = UINT64_MAX;
  s->limit = node_limit;
  int ok = 1;
  if (batch > 64 || (batch > 0 && sorted[0] > s->P[0]->max_len)) ok = 0; /* too large / infeasible */
  if (ok) dfs(s, 0, 0);
  if (ok && s->best != UINT64_MAX) memcpy(pipe, s->best_pipe, (size_t)batch);
  *value = ok ? s->best : UINT64_MAX;
  *nodes = s->nodes;
  const int proved = ok && !s->exhausted;
  free(s);
  return proved; /* 1: value is the exact optimum; 0: infeasible, too large or node limit hit */
}

/* ---------------------------------------------------------------- Eq. 1 exact
 * Eq. 1 for one pipeline: min over V in App. D's range (reading 5, extended upward
 * while no V is feasible) and over every split of the items into V micro-batches with
 * sum l <= MaxLen of (max micro-batch time) (PP - 1 + V); ties to the smaller V.  Plain
 * depth-first enumeration: item by item (given order), every bin, pruned only by "the partial
 * maximum already reaches the best for this V" (bin times never decrease). */
typedef struct {
  const uint32_t* ell;
  const uint32_t* tau;
  int u, v;
  uint32_t M;
  uint64_t t[64];
  uint32_t tok[64];
  uint64_t best;
  uint64_t nodes, limit;
  int exhausted;
} pk_t;

static void pk_dfs(pk_t* s, int i, uint64_t pmax) {
  if (s->exhausted) return;
  if (++s->nodes > s->limit) {
    s->exhausted = 1;
    return;
  }
  if (i == s->u) {
    int empty = 0;
    for (int b = 0; b < s->v; ++b) empty |= s->tok[b] == 0; /* V non-empty micro-batches */
    if (!empty && pmax < s->best) s->best = pmax;
    return;
  }
  for (int b = 0; b < s->v; ++b) {
    if (s->tok[b] + s->ell[i] > s->M) continue;
    const uint64_t nt = s->t[b] + s->tau[i];
    const uint64_t nm = nt > pmax ? nt : pmax;
    if (nm >= s->best) continue;
    s->t[b] = nt;
    s->tok[b] += s->ell[i];
    pk_dfs(s, i + 1, nm);
    s->t[b] -= s->tau[i];
    s->tok[b] -= s->ell[i];
  }
}

int hydref_eq1_exact(const uint32_t* ell, const uint32_t* tau, int u, const hydref_scheme* sch,
                     uint64_t node_limit, uint32_t* v_out, uint64_t* obj_out, uint64_t* nodes) {
  *v_out = 0;
  *obj_out = 0;
  *nodes = 0;
  if (u == 0) return 1;
  if (u > 64) return 0;
  uint64_t S = 0;
  for (int i = 0; i < u; ++i) S += ell[i];
  const uint32_t M = sch->max_len, P = sch->pp;
  uint32_t vlo = (uint32_t)((S + M - 1) / M);
  if (vlo < 1) vlo = 1;
  uint32_t vhi = (uint32_t)u;
  if (sch->util_len) {
    const uint64_t q = S / sch->util_len;
    vhi = q < (uint64_t)u ? (uint32_t)q : (uint32_t)u;
  }
  if (vhi < vlo) vhi = vlo;
  pk_t* s = (pk_t*)calloc(1, sizeof(pk_t));
  s->ell = ell;
  s->tau = tau;
  s->u = u;
  s->M = M;
  s->limit = node_limit;
  uint64_t best = UINT64_MAX;
  uint32_t vbest = 0;
  int proved = 1;
  for (uint32_t V = vlo; V <= (uint32_t)u; ++V) {
    if (V > vhi && vbest != 0) break; /* extension only while nothing in range is feasible */
    if (V > 64) break;
    s->v = (int)V;
    memset(s->t, 0, sizeof(s->t));
    memset(s->tok, 0, sizeof(s->tok));
    s->best = UINT64_MAX;
    s->exhausted = 0;
    pk_dfs(s, 0, 0);
    if (s->exhausted) proved = 0;
    if (s->best != UINT64_MAX) {
      const uint64_t obj = s->best * (uint64_t)(P - 1u + V);
      if (obj < best) {
        best = obj;
        vbest = V;
      }
    }
  }
  *nodes = s->nodes;
  free(s);
  *v_out = vbest;
  *obj_out = best;
  return proved && vbest != 0;
}
