/* oracle/hydref.h -- CPU ORACLE of the Hydraulis two-stage assignment (HYD-H1).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load or call this library.  The product
 * path (paper_2412_07894_b200/, libhyd.so) never links, imports or executes it,
 * and shares no code, header, helper or constant generator with it.
 *
 * Plain, scalar, obviously-correct C11.  Every function follows the paper
 * (PAPER.md, cited P:<line>) step by step in the paper's order and notation, with
 * the readings of SURVEY.md §8(c) / DESIGN.md §2 where the paper is silent.
 * All arithmetic is integer (unsigned __int128 where a product may exceed 64 bits).
 */
#ifndef HYDREF_H
#define HYDREF_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* one parallel scheme P = <TP,PP,CP> with its profiled cost model (48 bytes) */
typedef struct {
  uint32_t tp, pp, cp;
  uint32_t max_len;  /* MaxLen(P), App. C.1 */
  uint32_t util_len; /* UtilLen(P), App. D; 0 = no upper bound on V */
  uint32_t pad_;
  uint64_t a_q32, b_q32, c_q32; /* T(l,P) = a l^2 + b l + c, App. C.2, Q32 */
} hydref_scheme;

/* status bits (same meaning as the product's, defined independently) */
#define HYDREF_F_OVERFLOW 1u
#define HYDREF_F_ZERO_COST 2u
#define HYDREF_F_BAD_LENGTH 4u
#define HYDREF_F_KEY_RANGE 8u

/* Step 1 -- T(l,P) in Q32 fixed point, floored, as u32 ticks. */
uint32_t hydref_cost(const hydref_scheme* s, uint32_t l, uint32_t* status);

/* Step 2 -- order by (length desc, index asc).  sorted[i] = len[perm[i]]. */
void hydref_sort(const uint32_t* len, int batch, uint32_t* sorted, uint32_t* perm);

/* Steps 1+2 for one iteration: sorted lengths, perm, cost[i*k_pad + k]. */
void hydref_cost_table(const uint32_t* len, int batch, const hydref_scheme* schemes, int n_schemes,
                       int k_pad, uint32_t* sorted, uint32_t* perm, uint32_t* cost, uint32_t* status);

/* Step 4 -- stage 1 dispatch of one (candidate, iteration) (Eq. 2/3 P:636-650, Alg. 1).
 * Returns 1 if feasible, 0 if the candidate cannot hold sorted[0] (pipe=0xFF.., lb=UINT64_MAX). */
int hydref_dispatch(const uint32_t* sorted, const uint32_t* cost, int batch, int k_pad,
                    const hydref_scheme* schemes, const uint8_t* cand_row, int np, uint8_t* pipe,
                    uint64_t* lb);

/* LPT(V) with capacity for one pipeline's items (in the given order).  Returns 1 if
 * feasible (bin ids in mb_q[0..u)), 0 if some item fits no bin (LPT(V) = bottom).
 * *maxbin = max bin time on success. */
int hydref_lpt(const uint32_t* ell, const uint32_t* tau, int u, int v, uint32_t max_len,
               uint16_t* mb_q, uint64_t* maxbin);
/* The same LPT(V) with the argmin read from a (time, b) min-heap (O(U log V)); identical
 * results (pinned against hydref_lpt).  hydref_pack_pipeline's V enumeration uses it. */
int hydref_lpt_heap(const uint32_t* ell, const uint32_t* tau, int u, int v, uint32_t max_len,
                    uint16_t* mb_q, uint64_t* maxbin);

/* Step 5 -- stage 2 pack of one pipeline (Eq. 1, V enumeration P:616,
 * App. D range P:1097).  ell/tau: the pipeline's items in increasing sorted position.
 * Writes V*, ptime = obj(V*) and the micro-batch id of each item. */
void hydref_pack_pipeline(const uint32_t* ell, const uint32_t* tau, int u, const hydref_scheme* s,
                          uint16_t* v_out, uint64_t* ptime_out, uint16_t* mb_q, uint32_t* status);

/* Steps 5-6 for one (c,t) given its stage-1 assignment pipe[B]: pack every pipeline,
 * return the makespan. */
uint64_t hydref_pack_pair(const uint32_t* sorted, const uint32_t* cost, int batch, int k_pad,
                          const hydref_scheme* schemes, const uint8_t* cand_row, int np,
                          const uint8_t* pipe, uint16_t* mb, uint16_t* v, uint64_t* ptime,
                          uint32_t* status);

/* Steps 4-6 for one (c,t): dispatch, pack every pipeline, makespan.  Outputs are
 * rows: pipe[B], mb[B], v[32], ptime[32]; returns makespan (UINT64_MAX if infeasible). */
uint64_t hydref_assign_pair(const uint32_t* sorted, const uint32_t* cost, int batch, int k_pad,
                            const hydref_scheme* schemes, const uint8_t* cand_row, int np,
                            uint8_t* pipe, uint64_t* lb, uint16_t* mb, uint16_t* v, uint64_t* ptime,
                            uint32_t* status);

/* Step 7 -- selection for one iteration over n_cand makespans (stride 1). */
int64_t hydref_select(const uint64_t* makespan, int n_cand, int cand_offset, uint32_t* status);

/* Whole batch (steps 1-7), threads over candidates (n_threads <= 0: hardware count).
 * Layouts as include/hyd.h: sorted/perm [It][B], cost [It][B][k_pad], pipe/mb [C][It][B],
 * lb [C][It], v/ptime [C][It][32], makespan [It][C], key [It]. */
void hydref_assign_batch(const uint32_t* len, int n_iter, int batch, const hydref_scheme* schemes,
                         int n_schemes, int k_pad, const uint8_t* cand, const uint8_t* cand_np,
                         int n_cand, int cand_offset, uint32_t* sorted, uint32_t* perm,
                         uint32_t* cost, uint8_t* pipe, uint64_t* lb, uint16_t* mb, uint16_t* v,
                         uint64_t* ptime, uint64_t* makespan, int64_t* key, uint32_t* status,
                         int n_threads);

/* Selected (c,t) pairs only (sampled parity at full size).  Requires sorted/cost for
 * every t (from hydref_cost_table).  Row outputs are [n_pairs][B] / [n_pairs][32]. */
void hydref_assign_pairs(const uint32_t* sorted, const uint32_t* cost, int n_iter, int batch,
                         int k_pad, const hydref_scheme* schemes, const uint8_t* cand,
                         const uint8_t* cand_np, const int32_t* pair_c, const int32_t* pair_t,
                         int n_pairs, uint8_t* pipe, uint64_t* lb, uint16_t* mb, uint16_t* v,
                         uint64_t* ptime, uint64_t* makespan, uint32_t* status, int n_threads);

/* ------------------------------------------------------------------ NEXT-1 (alg1ref.c)
 * Paper-faithful Alg. 1: T random-permutation trials, best by (O, trial). */

/* Philox4x32-10 (Salmon et al., SC'11): 10 rounds of the Philox S-P network on a 128-bit
 * counter under a 64-bit key. */
void hydref_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* Trial permutation of the B sorted positions for (seed, iteration t, trial): Fisher-Yates
 * (Durstenfeld), for k = B-1 down to 1: r = Philox(ctr = (k / 4, t, trial, 0),
 * key = (seed lo, seed hi))[k % 4], j = (r * (k + 1)) >> 32, swap(order[k], order[j]).
 * DESIGN.md reading 21: one permutation per (t, trial), shared by every candidate. */
void hydref_alg1_permutation(uint64_t seed, int t, int trial, int batch, uint32_t* order);

/* One trial: Alg. 1 lines 3-14 over the sequences in `order` (sorted positions).  Writes
 * pipe[i] for each sorted position i; returns O_trial = max_j (C_j + E_j) (line 15). */
uint64_t hydref_alg1_trial(const uint32_t* sorted, const uint32_t* cost, int batch, int k_pad,
                           const hydref_scheme* schemes, const uint8_t* cand_row, int np,
                           const uint32_t* order, uint8_t* pipe);

/* Alg. 1 with T = trials: the trial with the smallest (O_trial, trial) wins (lines 16-17,
 * strict <).  Returns 1 if feasible (pipe, lb = O_best, *best_trial), 0 if the candidate
 * cannot hold sorted[0] (pipe = 0xFF.., lb = UINT64_MAX, *best_trial = -1). */
int hydref_alg1_dispatch(const uint32_t* sorted, const uint32_t* cost, int batch, int k_pad,
                         const hydref_scheme* schemes, const uint8_t* cand_row, int np,
                         uint64_t seed, int t, int trials, uint8_t* pipe, uint64_t* lb,
                         int32_t* best_trial);

/* Steps 4-6 with Alg. 1 as stage 1 (best_trial may be NULL). */
uint64_t hydref_alg1_assign_pair(const uint32_t* sorted, const uint32_t* cost, int batch,
                                 int k_pad, const hydref_scheme* schemes, const uint8_t* cand_row,
                                 int np, uint64_t seed, int t, int trials, uint8_t* pipe,
                                 uint64_t* lb, uint16_t* mb, uint16_t* v, uint64_t* ptime,
                                 int32_t* best_trial, uint32_t* status);

/* Batch / pairs drivers with a stage-1 choice: trials = 0 -> HYD-H1 dispatch, else Alg. 1
 * with that many trials; best_trial [C][It] / [n_pairs] may be NULL. */
void hydref_assign_batch_ex(const uint32_t* len, int n_iter, int batch,
                            const hydref_scheme* schemes, int n_schemes, int k_pad,
                            const uint8_t* cand, const uint8_t* cand_np, int n_cand,
                            int cand_offset, int trials, uint64_t seed, uint32_t* sorted,
                            uint32_t* perm, uint32_t* cost, uint8_t* pipe, uint64_t* lb,
                            uint16_t* mb, uint16_t* v, uint64_t* ptime, uint64_t* makespan,
                            int64_t* key, int32_t* best_trial, uint32_t* status, int n_threads);
void hydref_assign_pairs_ex(const uint32_t* sorted, const uint32_t* cost, int n_iter, int batch,
                            int k_pad, const hydref_scheme* schemes, const uint8_t* cand,
                            const uint8_t* cand_np, const int32_t* pair_c, const int32_t* pair_t,
                            int n_pairs, int trials, uint64_t seed, uint8_t* pipe, uint64_t* lb,
                            uint16_t* mb, uint16_t* v, uint64_t* ptime, uint64_t* makespan,
                            int32_t* best_trial, uint32_t* status, int n_threads);

/* ------------------------------------------------------------------ NEXT-3 (dpref.c)
 * Strategy-proposal DP.  pre [K][J+1]: pre[k][j] = sum of T(x, P_k) over dataset
 * lengths x (truncated to J step) with x <= j step.  t_num/t_den/choice [(N scale + 1)][J + 1]:
 * t[nu][j] = t_num/t_den for n = nu/scale GPUs and l = j step (den 0 = infinity); choice = -1
 * (carry t[nu-1][j]), -2 (base), else k << 24 | mu << 12 | j' (d = mu/scale pipelines of P_k on
 * the interval (l - j' step, l]). */
void hydref_dp_prefix(const uint32_t* lengths, int n_seq, const hydref_scheme* schemes, int K,
                      int step, int J, uint64_t* pre, uint32_t* status);
int hydref_dp_solve(const uint64_t* pre, const hydref_scheme* schemes, int K, int step, int J,
                    int n_gpus, int scale, uint64_t* t_num, uint64_t* t_den, int32_t* choice);
int hydref_dp_strategy(const int32_t* choice, const uint64_t* t_den, const hydref_scheme* schemes,
                       int K, int J, int n_gpus, int scale, int j, uint32_t* counts,
                       uint32_t* top_k);

/* ------------------------------------------------------------------ NEXT-4 (bbref.c)
 * Exact Eq. 3 optimum by plain depth-first enumeration (pruned by the incumbent only).
 * Returns 1 if proved optimal within node_limit. */
int hydref_eq3_exact(const uint32_t* sorted, const uint32_t* cost, int batch, int k_pad,
                     const hydref_scheme* schemes, const uint8_t* cand_row, int np,
                     uint64_t node_limit, uint8_t* pipe, uint64_t* value, uint64_t* nodes);
/* Exact Eq. 1 for one pipeline's items (ell/tau in sorted order): min over App. D's V range
 * (extended upward while none is feasible) and every capacity-feasible split of
 * max-bin-time (PP-1+V), ties to the smaller V.  Returns 1 if proved within node_limit. */
int hydref_eq1_exact(const uint32_t* ell, const uint32_t* tau, int u, const hydref_scheme* sch,
                     uint64_t node_limit, uint32_t* v_out, uint64_t* obj_out, uint64_t* nodes);

#ifdef __cplusplus
}
#endif
#endif
