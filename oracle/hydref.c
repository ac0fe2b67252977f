/* oracle/hydref.c -- CPU ORACLE of the Hydraulis two-stage assignment (HYD-H1).
 *
 * TEST INFRASTRUCTURE ONLY (see hydref.h).  Plain scalar C11; no blocking, fusion,
 * pruning or reordering beyond what the paper / SURVEY.md §8(c) states.  Each
 * function cites the passage it follows (P:<line> = /root/reference/PAPER.md).
 *
 * Pins (tests/test_oracle_*.py): cost closed form vs Python big ints; sort vs
 * Python sorted(); dispatch vs a literal transcription of Alg. 1
 * and vs Graham's LPT bound on identical machines; Eq. 2 / Eq. 1 recomputed from
 * the outputs; capacity, conservation, non-empty micro-batches; brute-force
 * optimum on tiny instances (heuristic >= OPT); the hand-worked example of
 * SURVEY §8(c) (tests/golden/worked_example.json); SPEC S:313-314 examples.
 */
#include "hydref.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

typedef unsigned __int128 u128;

#define LEN_LIMIT (1u << 24)
#define KEY_SHIFT 20
#define MAKESPAN_LIMIT (1ull << 43)

/* ---------------------------------------------------------------- step 1: cost
 * App. C.2: T(l, P_k) = a_k l^2 + b_k l + c_k.  Reading 3:
 * coefficients are Q32 fixed point, T = floor((a l^2 + b l + c) / 2^32) ticks,
 * required to lie in [1, 2^32-1].  Lengths must lie in [1, 2^24]. */
uint32_t hydref_cost(const hydref_scheme* s, uint32_t l, uint32_t* status) {
  if (l == 0 || l > LEN_LIMIT) {
    *status |= HYDREF_F_BAD_LENGTH;
    return 0xFFFFFFFFu;
  }
  u128 ll = (u128)l;
  u128 num = (u128)s->a_q32 * ll * ll + (u128)s->b_q32 * ll + (u128)s->c_q32;
  u128 t = num >> 32;
  if (t > 0xFFFFFFFFu) {
    *status |= HYDREF_F_OVERFLOW;
    return 0xFFFFFFFFu;
  }
  if (t == 0) {
    *status |= HYDREF_F_ZERO_COST;
    return 0;
  }
  return (uint32_t)t;
}

/* ---------------------------------------------------------------- step 2: sort
 * Order positions by (length descending, original index ascending).  The paper
 * dispatches in a random order (Alg. 1 line 2); HYD-H1 uses this single
 * deterministic longest-first order (reading 7). */
typedef struct {
  uint32_t len;
  uint32_t idx;
} len_idx;

static int cmp_len_idx(const void* pa, const void* pb) {
  const len_idx* a = (const len_idx*)pa;
  const len_idx* b = (const len_idx*)pb;
  if (a->len != b->len) return a->len > b->len ? -1 : 1;
  return a->idx < b->idx ? -1 : (a->idx > b->idx ? 1 : 0);
}

void hydref_sort(const uint32_t* len, int batch, uint32_t* sorted, uint32_t* perm) {
  len_idx* tmp = (len_idx*)malloc(sizeof(len_idx) * (size_t)(batch > 0 ? batch : 1));
  for (int i = 0; i < batch; ++i) {
    tmp[i].len = len[i];
    tmp[i].idx = (uint32_t)i;
  }
  qsort(tmp, (size_t)batch, sizeof(len_idx), cmp_len_idx);
  for (int i = 0; i < batch; ++i) {
    sorted[i] = tmp[i].len;
    perm[i] = tmp[i].idx;
  }
  free(tmp);
}

void hydref_cost_table(const uint32_t* len, int batch, const hydref_scheme* schemes, int n_schemes,
                       int k_pad, uint32_t* sorted, uint32_t* perm, uint32_t* cost, uint32_t* status) {
  hydref_sort(len, batch, sorted, perm);
  for (int i = 0; i < batch; ++i)
    for (int k = 0; k < k_pad; ++k)
      cost[(size_t)i * k_pad + k] = k < n_schemes ? hydref_cost(&schemes[k], sorted[i], status) : 0u;
}

/* ---------------------------------------------------------------- step 4: dispatch
 * Stage 1 (§6.2).  Pipelines j = 0..np-1 of the candidate, in canonical order
 * (MaxLen non-increasing).  Sequence i may go to pipeline j iff
 * MaxLen(P_j) >= l_i (the horizon J_i of P:626, inclusive).
 *
 * Greedy in the sorted order: for each sequence, for each
 * feasible j, tau = T(l_i, P_j); the extra (bubble) term of Eq. 2 is
 * T(max assigned l, P_j) * (PP_j - 1): since sequences arrive longest first, the
 * first sequence a pipeline receives is its longest, so
 *   e_j = (pipeline j empty) ? tau * (PP_j - 1) : extra_j
 *   new_j = C_j + tau + e_j          (C_j, E_j are Alg. 1's accumulators)
 * and j* = argmin_j (new_j, j).  This is Alg. 1's min-O_max choice
 * with ties in O_max broken by smaller own new load, then smaller j (reading 10).
 * LB = max_j (C_j + E_j) is the Eq. 3 objective of the final assignment. */
int hydref_dispatch(const uint32_t* sorted, const uint32_t* cost, int batch, int k_pad,
                    const hydref_scheme* schemes, const uint8_t* cand_row, int np, uint8_t* pipe,
                    uint64_t* lb) {
  uint64_t C[32], E[32];
  int cnt[32];
  if (batch > 0 && sorted[0] > schemes[cand_row[0]].max_len) {
    memset(pipe, 0xFF, (size_t)batch);
    *lb = UINT64_MAX;
    return 0;
  }
  for (int j = 0; j < np; ++j) {
    C[j] = 0;
    E[j] = 0;
    cnt[j] = 0;
  }
  for (int i = 0; i < batch; ++i) {
    uint32_t l = sorted[i];
    int jstar = -1;
    uint64_t best = 0, best_tau = 0, best_e = 0;
    for (int j = 0; j < np; ++j) {
      const hydref_scheme* s = &schemes[cand_row[j]];
      if (s->max_len < l) continue; /* j > J_i */
      uint64_t tau = cost[(size_t)i * k_pad + cand_row[j]];
      uint64_t e = cnt[j] == 0 ? tau * (uint64_t)(s->pp - 1) : E[j];
      uint64_t nw = C[j] + tau + e;
      if (jstar < 0 || nw < best) {
        jstar = j;
        best = nw;
        best_tau = tau;
        best_e = e;
      }
    }
    /* jstar >= 0: l <= sorted[0] <= MaxLen(P_0) */
    C[jstar] += best_tau;
    E[jstar] = best_e;
    cnt[jstar] += 1;
    pipe[i] = (uint8_t)jstar;
  }
  uint64_t m = 0;
  for (int j = 0; j < np; ++j)
    if (C[j] + E[j] > m) m = C[j] + E[j];
  *lb = m;
  return 1;
}

/* ---------------------------------------------------------------- step 5: pack
 * LPT(V) with capacity: V empty bins; items in the given
 * (longest-first) order; item goes to the bin of least time among bins whose token
 * count stays <= MaxLen (constraint of Eq. 1, inclusive), ties to the
 * smallest bin index.  No bin fits -> bottom. */
int hydref_lpt(const uint32_t* ell, const uint32_t* tau, int u, int v, uint32_t max_len,
               uint16_t* mb_q, uint64_t* maxbin) {
  uint64_t* time = (uint64_t*)calloc((size_t)v, sizeof(uint64_t));
  uint64_t* tok = (uint64_t*)calloc((size_t)v, sizeof(uint64_t));
  int ok = 1;
  for (int q = 0; q < u && ok; ++q) {
    int bstar = -1;
    for (int b = 0; b < v; ++b) {
      if (tok[b] + ell[q] > max_len) continue;
      if (bstar < 0 || time[b] < time[bstar]) bstar = b;
    }
    if (bstar < 0) {
      ok = 0;
      break;
    }
    time[bstar] += tau[q];
    tok[bstar] += ell[q];
    mb_q[q] = (uint16_t)bstar;
  }
  if (ok) {
    uint64_t m = 0;
    for (int b = 0; b < v; ++b)
      if (time[b] > m) m = time[b];
    *maxbin = m;
  }
  free(time);
  free(tok);
  return ok;
}

/* The same LPT(V), with the argmin taken from a binary min-heap of the bins ordered by
 * (time_b, b) instead of a scan: bins leave the heap in increasing (time, b) order, so the
 * first one whose token count stays <= MaxLen is the scan's b* (least time among fitting bins,
 * ties to the smallest index).  Bins popped before it do not fit and go back unchanged.
 * O(U log V) instead of O(U V) per run, which is what lets the V enumeration below cover
 * config 5 (U up to ~2800, V up to U).  Pinned against hydref_lpt (tests/test_oracle_pins.py). */
static int heap_less(const uint64_t* time, uint32_t a, uint32_t b) {
  return time[a] < time[b] || (time[a] == time[b] && a < b);
}

static void heap_push(uint32_t* h, int* n, const uint64_t* time, uint32_t b) {
  int i = (*n)++;
  h[i] = b;
  while (i > 0 && heap_less(time, h[i], h[(i - 1) / 2])) {
    uint32_t x = h[i];
    h[i] = h[(i - 1) / 2];
    h[(i - 1) / 2] = x;
    i = (i - 1) / 2;
  }
}

static uint32_t heap_pop(uint32_t* h, int* n, const uint64_t* time) {
  uint32_t top = h[0];
  h[0] = h[--(*n)];
  int i = 0;
  for (;;) {
    int l = 2 * i + 1, r = l + 1, m = i;
    if (l < *n && heap_less(time, h[l], h[m])) m = l;
    if (r < *n && heap_less(time, h[r], h[m])) m = r;
    if (m == i) break;
    uint32_t x = h[i];
    h[i] = h[m];
    h[m] = x;
    i = m;
  }
  return top;
}

int hydref_lpt_heap(const uint32_t* ell, const uint32_t* tau, int u, int v, uint32_t max_len,
                    uint16_t* mb_q, uint64_t* maxbin) {
  uint64_t* time = (uint64_t*)calloc((size_t)v, sizeof(uint64_t));
  uint64_t* tok = (uint64_t*)calloc((size_t)v, sizeof(uint64_t));
  uint32_t* heap = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)v);
  uint32_t* skipped = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)v);
  int n = 0, ok = 1;
  for (int b = 0; b < v; ++b) heap_push(heap, &n, time, (uint32_t)b);
  for (int q = 0; q < u && ok; ++q) {
    int bstar = -1, n_skip = 0;
    while (n > 0) {
      uint32_t b = heap_pop(heap, &n, time);
      if (tok[b] + ell[q] <= max_len) {
        bstar = (int)b;
        break;
      }
      skipped[n_skip++] = b;
    }
    for (int s = 0; s < n_skip; ++s) heap_push(heap, &n, time, skipped[s]);
    if (bstar < 0) {
      ok = 0;
      break;
    }
    time[bstar] += tau[q];
    tok[bstar] += ell[q];
    mb_q[q] = (uint16_t)bstar;
    heap_push(heap, &n, time, (uint32_t)bstar);
  }
  if (ok) {
    uint64_t m = 0;
    for (int b = 0; b < v; ++b)
      if (time[b] > m) m = time[b];
    *maxbin = m;
  }
  free(time);
  free(tok);
  free(heap);
  free(skipped);
  return ok;
}

/* Eq. 1: objective = (max_b sum_{i in b} T(l_i)) * (PP - 1 + V).
 * V enumeration restricted to App. D's range:
 *   V_lo = max(ceil(S / MaxLen), 1),  V_hi = min(floor(S / UtilLen), U)
 * (reading 5: ceil/floor, UtilLen = 0 means no upper pruning, V_hi < V_lo -> V_hi = V_lo).
 * V* = argmin (obj(V), V) over feasible V in range (reading 6: smaller V on ties);
 * if no V in range is feasible, V* = the smallest feasible V in (V_hi, U]. */
void hydref_pack_pipeline(const uint32_t* ell, const uint32_t* tau, int u, const hydref_scheme* s,
                          uint16_t* v_out, uint64_t* ptime_out, uint16_t* mb_q, uint32_t* status) {
  if (u == 0) { /* reading 12: an empty pipeline has V = 0, time 0 */
    *v_out = 0;
    *ptime_out = 0;
    return;
  }
  uint64_t S = 0;
  for (int q = 0; q < u; ++q) S += ell[q];
  uint64_t M = s->max_len;
  uint64_t v_lo = (S + M - 1) / M;
  if (v_lo < 1) v_lo = 1;
  uint64_t v_hi = s->util_len == 0 ? (uint64_t)u : S / s->util_len;
  if (v_hi > (uint64_t)u) v_hi = (uint64_t)u;
  if (v_hi < v_lo) v_hi = v_lo;

  uint16_t* cur = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)u);
  int have = 0;
  u128 best = 0;
  uint64_t best_v = 0;
  for (uint64_t v = v_lo; v <= v_hi; ++v) {
    uint64_t maxbin;
    if (!hydref_lpt_heap(ell, tau, u, (int)v, s->max_len, cur, &maxbin)) continue;
    u128 obj = (u128)maxbin * (u128)(s->pp - 1 + v);
    if (!have || obj < best) {
      have = 1;
      best = obj;
      best_v = v;
      memcpy(mb_q, cur, sizeof(uint16_t) * (size_t)u);
    }
  }
  for (uint64_t v = v_hi + 1; !have && v <= (uint64_t)u; ++v) {
    uint64_t maxbin;
    if (!hydref_lpt_heap(ell, tau, u, (int)v, s->max_len, cur, &maxbin)) continue;
    have = 1;
    best = (u128)maxbin * (u128)(s->pp - 1 + v);
    best_v = v;
    memcpy(mb_q, cur, sizeof(uint16_t) * (size_t)u);
  }
  free(cur);
  if (!have) { /* an item longer than MaxLen: cannot come from hydref_dispatch */
    *v_out = 0;
    *ptime_out = UINT64_MAX;
    for (int q = 0; q < u; ++q) mb_q[q] = 0xFFFF;
    *status |= HYDREF_F_OVERFLOW;
    return;
  }
  *v_out = (uint16_t)best_v;
  if (best > (u128)UINT64_MAX - 1) {
    *status |= HYDREF_F_OVERFLOW;
    *ptime_out = UINT64_MAX - 1;
  } else {
    *ptime_out = (uint64_t)best;
  }
}

/* ---------------------------------------------------------------- steps 5-6 for one (c,t)
 * Given a stage-1 assignment pipe[B] (sorted positions), pack every pipeline (step 5) and
 * return the makespan max_j ptime_j (step 6). */
uint64_t hydref_pack_pair(const uint32_t* sorted, const uint32_t* cost, int batch, int k_pad,
                          const hydref_scheme* schemes, const uint8_t* cand_row, int np,
                          const uint8_t* pipe, uint16_t* mb, uint16_t* v, uint64_t* ptime,
                          uint32_t* status) {
  uint32_t* ell = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(batch > 0 ? batch : 1));
  uint32_t* tau = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(batch > 0 ? batch : 1));
  int* pos = (int*)malloc(sizeof(int) * (size_t)(batch > 0 ? batch : 1));
  uint16_t* mbq = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)(batch > 0 ? batch : 1));
  uint64_t makespan = 0; /* step 6: max over pipelines of the Eq. 1 objective */
  for (int j = 0; j < np; ++j) {
    int u = 0;
    for (int i = 0; i < batch; ++i)
      if (pipe[i] == j) {
        ell[u] = sorted[i];
        tau[u] = cost[(size_t)i * k_pad + cand_row[j]];
        pos[u] = i;
        ++u;
      }
    hydref_pack_pipeline(ell, tau, u, &schemes[cand_row[j]], &v[j], &ptime[j], mbq, status);
    for (int q = 0; q < u; ++q) mb[pos[q]] = mbq[q];
    if (ptime[j] > makespan) makespan = ptime[j];
  }
  free(ell);
  free(tau);
  free(pos);
  free(mbq);
  return makespan;
}

/* ---------------------------------------------------------------- steps 4-6 for one (c,t) */
uint64_t hydref_assign_pair(const uint32_t* sorted, const uint32_t* cost, int batch, int k_pad,
                            const hydref_scheme* schemes, const uint8_t* cand_row, int np,
                            uint8_t* pipe, uint64_t* lb, uint16_t* mb, uint16_t* v, uint64_t* ptime,
                            uint32_t* status) {
  for (int j = 0; j < 32; ++j) {
    v[j] = 0;
    ptime[j] = 0;
  }
  if (!hydref_dispatch(sorted, cost, batch, k_pad, schemes, cand_row, np, pipe, lb)) {
    for (int i = 0; i < batch; ++i) mb[i] = 0xFFFF;
    return UINT64_MAX;
  }
  return hydref_pack_pair(sorted, cost, batch, k_pad, schemes, cand_row, np, pipe, mb, v, ptime,
                          status);
}

/* ---------------------------------------------------------------- step 7: select
 * Step ④ of the per-iteration loop ("select the optimal one" P:567):
 * winner = argmin over feasible c of (makespan, c); key = makespan * 2^20 + c_global,
 * which needs makespan < 2^43 and c_global < 2^20 - 1 (reading 18: 2^20 - 1
 * with makespan 2^43 - 1 would equal the INT64_MAX "none" sentinel); else KEY_RANGE and
 * the candidate is excluded; INT64_MAX if no candidate remains. */
int64_t hydref_select(const uint64_t* makespan, int n_cand, int cand_offset, uint32_t* status) {
  int64_t best = INT64_MAX;
  for (int c = 0; c < n_cand; ++c) {
    uint64_t m = makespan[c];
    if (m == UINT64_MAX) continue;
    if (m >= MAKESPAN_LIMIT || (uint64_t)(c + cand_offset) >= (1ull << KEY_SHIFT) - 1) {
      *status |= HYDREF_F_KEY_RANGE;
      continue;
    }
    int64_t key = (int64_t)((m << KEY_SHIFT) | (uint64_t)(c + cand_offset));
    if (key < best) best = key;
  }
  return best;
}

/* ---------------------------------------------------------------- batch drivers */
typedef struct {
  const uint32_t* sorted;
  const uint32_t* cost;
  int n_iter, batch, k_pad, n_cand;
  const hydref_scheme* schemes;
  const uint8_t* cand;
  const uint8_t* cand_np;
  const int32_t* pair_c;
  const int32_t* pair_t;
  int n_pairs;
  uint8_t* pipe;
  uint64_t* lb;
  uint16_t* mb;
  uint16_t* v;
  uint64_t* ptime;
  uint64_t* makespan;
  int trials;         /* > 0: stage 1 is Alg. 1 with this many random trials (NEXT-1) */
  uint64_t seed;
  int32_t* best_trial; /* [C][It] (batch) or [n_pairs] (pairs) when trials > 0 */
  int tid, nthreads;
  uint32_t status;
} job;

static uint64_t job_pair(job* J, int c, int t, size_t orow, int32_t* best) {
  const uint32_t* sorted = J->sorted + (size_t)t * J->batch;
  const uint32_t* cost = J->cost + (size_t)t * J->batch * J->k_pad;
  if (J->trials > 0)
    return hydref_alg1_assign_pair(sorted, cost, J->batch, J->k_pad, J->schemes,
                                   J->cand + (size_t)c * 32, J->cand_np[c], J->seed, t, J->trials,
                                   J->pipe + orow * J->batch, J->lb + orow,
                                   J->mb + orow * J->batch, J->v + orow * 32,
                                   J->ptime + orow * 32, best, &J->status);
  return hydref_assign_pair(sorted, cost, J->batch, J->k_pad, J->schemes, J->cand + (size_t)c * 32,
                            J->cand_np[c], J->pipe + orow * J->batch, J->lb + orow,
                            J->mb + orow * J->batch, J->v + orow * 32, J->ptime + orow * 32,
                            &J->status);
}

static void* batch_worker(void* arg) {
  job* J = (job*)arg;
  for (int c = J->tid; c < J->n_cand; c += J->nthreads)
    for (int t = 0; t < J->n_iter; ++t) {
      size_t row = (size_t)c * J->n_iter + t;
      J->makespan[(size_t)t * J->n_cand + c] =
          job_pair(J, c, t, row, J->best_trial ? J->best_trial + row : NULL);
    }
  return NULL;
}

static void* pairs_worker(void* arg) {
  job* J = (job*)arg;
  for (int p = J->tid; p < J->n_pairs; p += J->nthreads)
    J->makespan[p] =
        job_pair(J, J->pair_c[p], J->pair_t[p], (size_t)p, J->best_trial ? J->best_trial + p : NULL);
  return NULL;
}

static int resolve_threads(int n) {
  if (n > 0) return n;
  long h = sysconf(_SC_NPROCESSORS_ONLN);
  return h > 0 ? (int)h : 1;
}

static uint32_t run_jobs(job* proto, int nthreads, void* (*fn)(void*)) {
  job* jobs = (job*)malloc(sizeof(job) * (size_t)nthreads);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  for (int k = 0; k < nthreads; ++k) {
    jobs[k] = *proto;
    jobs[k].tid = k;
    jobs[k].nthreads = nthreads;
    jobs[k].status = 0;
    pthread_create(&th[k], NULL, fn, &jobs[k]);
  }
  uint32_t st = 0;
  for (int k = 0; k < nthreads; ++k) {
    pthread_join(th[k], NULL);
    st |= jobs[k].status;
  }
  free(jobs);
  free(th);
  return st;
}

void hydref_assign_batch(const uint32_t* len, int n_iter, int batch, const hydref_scheme* schemes,
                         int n_schemes, int k_pad, const uint8_t* cand, const uint8_t* cand_np,
                         int n_cand, int cand_offset, uint32_t* sorted, uint32_t* perm,
                         uint32_t* cost, uint8_t* pipe, uint64_t* lb, uint16_t* mb, uint16_t* v,
                         uint64_t* ptime, uint64_t* makespan, int64_t* key, uint32_t* status,
                         int n_threads) {
  hydref_assign_batch_ex(len, n_iter, batch, schemes, n_schemes, k_pad, cand, cand_np, n_cand,
                         cand_offset, 0, 0, sorted, perm, cost, pipe, lb, mb, v, ptime, makespan,
                         key, NULL, status, n_threads);
}

void hydref_assign_batch_ex(const uint32_t* len, int n_iter, int batch,
                            const hydref_scheme* schemes, int n_schemes, int k_pad,
                            const uint8_t* cand, const uint8_t* cand_np, int n_cand,
                            int cand_offset, int trials, uint64_t seed, uint32_t* sorted,
                            uint32_t* perm, uint32_t* cost, uint8_t* pipe, uint64_t* lb,
                            uint16_t* mb, uint16_t* v, uint64_t* ptime, uint64_t* makespan,
                            int64_t* key, int32_t* best_trial, uint32_t* status, int n_threads) {
  for (int t = 0; t < n_iter; ++t)
    hydref_cost_table(len + (size_t)t * batch, batch, schemes, n_schemes, k_pad,
                      sorted + (size_t)t * batch, perm + (size_t)t * batch,
                      cost + (size_t)t * batch * k_pad, status);
  job proto;
  memset(&proto, 0, sizeof(proto));
  proto.sorted = sorted;
  proto.cost = cost;
  proto.n_iter = n_iter;
  proto.batch = batch;
  proto.k_pad = k_pad;
  proto.n_cand = n_cand;
  proto.schemes = schemes;
  proto.cand = cand;
  proto.cand_np = cand_np;
  proto.pipe = pipe;
  proto.lb = lb;
  proto.mb = mb;
  proto.v = v;
  proto.ptime = ptime;
  proto.makespan = makespan;
  proto.trials = trials;
  proto.seed = seed;
  proto.best_trial = best_trial;
  int nt = resolve_threads(n_threads);
  if (nt > n_cand) nt = n_cand > 0 ? n_cand : 1;
  *status |= run_jobs(&proto, nt, batch_worker);
  for (int t = 0; t < n_iter; ++t)
    key[t] = hydref_select(makespan + (size_t)t * n_cand, n_cand, cand_offset, status);
}

void hydref_assign_pairs(const uint32_t* sorted, const uint32_t* cost, int n_iter, int batch,
                         int k_pad, const hydref_scheme* schemes, const uint8_t* cand,
                         const uint8_t* cand_np, const int32_t* pair_c, const int32_t* pair_t,
                         int n_pairs, uint8_t* pipe, uint64_t* lb, uint16_t* mb, uint16_t* v,
                         uint64_t* ptime, uint64_t* makespan, uint32_t* status, int n_threads) {
  hydref_assign_pairs_ex(sorted, cost, n_iter, batch, k_pad, schemes, cand, cand_np, pair_c,
                         pair_t, n_pairs, 0, 0, pipe, lb, mb, v, ptime, makespan, NULL, status,
                         n_threads);
}

void hydref_assign_pairs_ex(const uint32_t* sorted, const uint32_t* cost, int n_iter, int batch,
                            int k_pad, const hydref_scheme* schemes, const uint8_t* cand,
                            const uint8_t* cand_np, const int32_t* pair_c, const int32_t* pair_t,
                            int n_pairs, int trials, uint64_t seed, uint8_t* pipe, uint64_t* lb,
                            uint16_t* mb, uint16_t* v, uint64_t* ptime, uint64_t* makespan,
                            int32_t* best_trial, uint32_t* status, int n_threads) {
  job proto;
  memset(&proto, 0, sizeof(proto));
  proto.sorted = sorted;
  proto.cost = cost;
  proto.n_iter = n_iter;
  proto.batch = batch;
  proto.k_pad = k_pad;
  proto.schemes = schemes;
  proto.cand = cand;
  proto.cand_np = cand_np;
  proto.pair_c = pair_c;
  proto.pair_t = pair_t;
  proto.n_pairs = n_pairs;
  proto.pipe = pipe;
  proto.lb = lb;
  proto.mb = mb;
  proto.v = v;
  proto.ptime = ptime;
  proto.makespan = makespan;
  proto.trials = trials;
  proto.seed = seed;
  proto.best_trial = best_trial;
  int nt = resolve_threads(n_threads);
  if (nt > n_pairs) nt = n_pairs > 0 ? n_pairs : 1;
  *status |= run_jobs(&proto, nt, pairs_worker);
}
