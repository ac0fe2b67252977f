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

/* Step 5 -- stage 2 pack of one pipeline (Eq. 1, V enumeration P:616,
 * App. D range P:1097).  ell/tau: the pipeline's items in increasing sorted position.
 * Writes V*, ptime = obj(V*) and the micro-batch id of each item. */
void hydref_pack_pipeline(const uint32_t* ell, const uint32_t* tau, int u, const hydref_scheme* s,
                          uint16_t* v_out, uint64_t* ptime_out, uint16_t* mb_q, uint32_t* status);

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

#ifdef __cplusplus
}
#endif
#endif
