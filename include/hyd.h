/* include/hyd.h -- C ABI of libhyd.so: the Hydraulis two-stage data assignment on B200.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, cited P:<line>):
 *   For every iteration t (a mini-batch of B variable-length sequences) and
 *   every candidate heterogeneous strategy c = P_1 + ... + P_D, the two-stage
 *   sequence assignment of §6: stage 1 dispatches the sequences across the D
 *   pipelines (Eq. 2/3 P:634-650, Alg. 1), stage 2 packs each pipeline's
 *   sequences into micro-batches (Eq. 1, App. D); the estimated
 *   propagation latency of (c,t) is the max over pipelines of the Eq. 1 objective, and the
 *   best candidate per iteration is selected (step ④).  The ILP solves are
 *   replaced by the deterministic heuristic HYD-H1.
 *
 * Conventions (all entry points):
 *   - Pointers are DEVICE pointers unless the name ends in _host.  Every call is
 *     stream-ordered and asynchronous on `stream` (a cudaStream_t passed as void*).
 *   - The caller owns every buffer.  The library allocates no device memory; scratch memory is
 *     a caller-provided device workspace.  Its only global state is diagnostic: a launch
 *     counter (hyd_kernel_launches, atomic) and the text of the last CUDA error seen by the
 *     calling thread (hyd_last_cuda_error, thread-local); neither affects any result.
 *   - Host-side argument validation returns a negative HYD_E_* code synchronously and
 *     launches nothing.  Data-dependent faults set HYD_F_* bits in the device word
 *     `status` (OR-ed, never cleared by the library); the caller reads it after syncing.
 *   - Infeasibility is a result, not an error: if the longest sequence of iteration t
 *     exceeds MaxLen of every pipeline of candidate c, then for (c,t):
 *     pipe row = 0xFF, mb row = 0xFFFF, v = ptime = 0, lb = makespan = UINT64_MAX.
 *   - Sequence-indexed outputs are indexed by SORTED position i (length descending,
 *     original index ascending); perm[t][i] is the original index of position i.
 *   - Limits: 0 <= n_iter <= HYD_MAX_ITER (iterations map to a grid dimension);
 *     1 <= batch <= HYD_MAX_BATCH; 1 <= n_schemes <= HYD_MAX_SCHEMES;
 *     k_pad % 4 == 0 and k_pad >= n_schemes; 1 <= cand_np[c] <= max_np <= 32;
 *     1 <= pp <= HYD_MAX_PP; max_len >= 1; n_cand + cand_offset <= 2^20 - 1 (global candidate
 *     index <= 2^20 - 2, so no key equals the INT64_MAX "none" sentinel).
 *     Lengths must lie in [1, 2^24] (else HYD_F_BAD_LENGTH).
 */
#ifndef HYD_H
#define HYD_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HYD_MAX_ITER 65535
#define HYD_MAX_BATCH 16384
#define HYD_SMALL_MAX_BATCH 128 /* hyd_dispatch_pack: largest batch */
#define HYD_MAX_SCHEMES 64
#define HYD_MAX_PIPES 32
#define HYD_MAX_PP 1024
#define HYD_KEY_SHIFT 20 /* key = makespan << 20 | candidate (global index) */

/* One parallel scheme P = <TP,PP,CP> with its profiled cost models (48 bytes).
 *   T(l,P) = floor((a_q32 l^2 + b_q32 l + c_q32) / 2^32) ticks  (App. C.2; Q32 reading)
 *   max_len  = MaxLen(P): token cap of one micro-batch (App. C.1; Eq. 1)
 *   util_len = UtilLen(P) (App. D); 0 disables the upper bound on V. */
typedef struct {
  uint32_t tp, pp, cp; /* pp enters the arithmetic (Eq. 1/2); tp, cp informational */
  uint32_t max_len;
  uint32_t util_len;
  uint32_t _pad;
  uint64_t a_q32, b_q32, c_q32;
} hyd_scheme;

/* return codes */
enum {
  HYD_OK = 0,
  HYD_E_INVALID = -1,       /* null pointer, size or limit violated */
  HYD_E_NOT_CANONICAL = -2, /* a candidate is not (MaxLen desc, scheme index asc) ordered */
  HYD_E_OVERFLOW = -3,
  HYD_E_ZERO_COST = -4,
  HYD_E_CUDA = -5,      /* a CUDA launch/copy failed (see hyd_last_cuda_error) */
  HYD_E_WORKSPACE = -6, /* workspace null or smaller than the *_workspace() size */
  HYD_E_REDUCE = -7     /* the caller's allreduce callback returned non-zero */
};

/* device status bits */
enum {
  HYD_F_OVERFLOW = 1u,      /* a cost exceeded 2^32-1 */
  HYD_F_ZERO_COST = 2u,     /* a cost evaluated to 0 */
  HYD_F_BAD_LENGTH = 4u,    /* a length was 0 or > 2^24 */
  HYD_F_KEY_RANGE = 8u,     /* a feasible makespan >= 2^43 (excluded from selection) */
  HYD_F_NOT_CANONICAL = 16u, /* device-side candidate check failed (treated infeasible) */
  HYD_F_BAD_PIPE = 32u       /* hyd_pipe_index: a pipe row is not an assignment (treated infeasible) */
};

/* ---- a1+a2: per-iteration stable sort + cost table ------------------------------------
 * len [n_iter][batch] u32 -> sorted_len [n_iter][batch] (length descending, ties by
 * original index ascending), perm [n_iter][batch] (original index of each sorted position),
 * cost [n_iter][batch][k_pad] u32: cost[t][i][k] = T(sorted_len[t][i], schemes[k]) for
 * k < n_schemes, 0 for padding.  An on-device LSD radix sort (one CTA per iteration).
 * Status: HYD_F_BAD_LENGTH (cost = 0xFFFFFFFF), HYD_F_OVERFLOW (cost = 0xFFFFFFFF),
 * HYD_F_ZERO_COST (cost = 0).  No workspace. */
int hyd_cost_table(const uint32_t* len, int n_iter, int batch, const hyd_scheme* schemes,
                   int n_schemes, int k_pad, uint32_t* sorted_len, uint32_t* perm, uint32_t* cost,
                   uint32_t* status, void* stream);

/* Per-pipeline statistics of a dispatch, consumed by hyd_pack (24 bytes):
 *   u = U_j (sequences dispatched to pipeline j), tau_max = T(longest of them, P_j)
 *   (its first one in sorted order), s = S_j (their token sum), sum_t = sum of their T(l, P_j).
 * Layout [n_iter][n_cand][max_np] (iteration-major, so one iteration's candidates are
 * contiguous); for an infeasible (c,t) only stats[t][c][0].u is defined, = 0xFFFFFFFF. */
typedef struct {
  uint32_t u;
  uint32_t tau_max;
  uint64_t s;
  uint64_t sum_t;
} hyd_pipe_stats;

/* ---- a3: stage 1 dispatch (Eq. 2/3, Alg. 1) ---------------------------------------------
 * cand [n_cand][32] u8 scheme indices (pipelines j = 0..cand_np[c]-1 in canonical order,
 * i.e. MaxLen non-increasing, scheme index ascending on ties), cand_np [n_cand] u8.
 * For each (c,t), sequences in sorted order go to the feasible pipeline (MaxLen_j >= l)
 * minimising (C_j + tau + e_j, j) where tau = T(l,P_j) and e_j = tau (PP_j - 1) for an empty
 * pipeline, else the pipeline's extra term E_j (Alg. 1 lines 8-14 with LPT order).
 * Outputs pipe [n_cand][n_iter][batch] u8 (pipeline of each sorted position),
 * lb [n_cand][n_iter] u64 = max_j (C_j + E_j) (the Eq. 3 objective),
 * stats [n_iter][n_cand][max_np] (hyd_pipe_stats, for hyd_pack) and
 * members [n_iter][n_cand][ceil(batch/32)][max_np] u32 (word-major): bit (i mod 32) of word
 * [t][c][i/32][j] is set iff sorted position i was dispatched to pipeline j (the m_ij matrix
 * of Eq. 3, as bitmaps; for hyd_pack).  Rows of infeasible (c,t) are undefined.
 * max_np = max over c of cand_np[c] (host-known; selects the kernel width).
 * ws: hyd_dispatch_workspace(n_iter) bytes of device scratch (per-iteration load bounds that
 * pick the kernels' integer width); HYD_E_WORKSPACE if smaller. */
size_t hyd_dispatch_workspace(int n_iter);
int hyd_dispatch(const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch,
                 int k_pad, const hyd_scheme* schemes, int n_schemes, const uint8_t* cand,
                 const uint8_t* cand_np, int n_cand, int max_np, uint8_t* pipe, uint64_t* lb,
                 hyd_pipe_stats* stats, uint32_t* members, uint32_t* status, void* ws,
                 size_t ws_bytes, void* stream);

/* ---- a3 -> a4 interface from an arbitrary stage-1 result ---------------------------------
 * hyd_pipe_index: builds the (stats, members) that hyd_pack consumes from ANY stage-1
 * assignment pipe [n_cand][n_iter][batch] u8 (the m_ij matrix of Eq. 3) -- e.g. a
 * host-side Alg. 1 or the caller's own dispatcher -- and lb [n_cand][n_iter] u64 =
 * Eq. 2's max_j (sum T(l, P_j) + T(longest on j, P_j)(PP_j - 1)) (lb may be NULL).  A row is an
 * assignment iff every entry j satisfies j < cand_np[c] and MaxLen_j >= l_i (J_i), or,
 * for a pair with l_0 > MaxLen_0 (infeasible), every entry is 0xFF.  Any other row sets
 * HYD_F_BAD_PIPE and the pair is marked infeasible (hyd_pack then writes its infeasible rows).
 * Layouts, sizes and the ragged form as hyd_dispatch / hyd_dispatch_ragged.  No workspace. */
int hyd_pipe_index(const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch, int k_pad,
                   const hyd_scheme* schemes, int n_schemes, const uint8_t* cand, const uint8_t* cand_np,
                   int n_cand, int max_np, const uint8_t* pipe, uint64_t* lb, hyd_pipe_stats* stats,
                   uint32_t* members, uint32_t* status, void* stream);

/* ---- a4: stage 2 packing (Eq. 1 + App. D) -------------------------------------------
 * The stage-1 result enters as `pipe` together with its index (stats, members): both come
 * from hyd_dispatch / hyd_dispatch_alg1 (which emit them while deciding) or, for a pipe made
 * anywhere else, from hyd_pipe_index (same n_cand/n_iter/max_np).  The kernels read the
 * index; `pipe` is the assignment it describes (a stats/members pair that does not describe
 * `pipe` is a caller error: the outputs are then those of the assignment the index describes).
 * For each (c,t,j): the pipeline's sequences Q (sorted order), U = |Q|, S = sum l:
 * V in [max(ceil(S/MaxLen),1), min(floor(S/UtilLen),U)] (clamped up to the lower end);
 * LPT(V): each sequence to the least-time micro-batch that stays within MaxLen (smallest
 * index on ties); objective (max micro-batch time)(PP-1+V); V* = argmin (objective, V);
 * if no V in range is feasible, the smallest feasible V above it.  The search over V is
 * pruned with exact lower bounds (never changes the result).
 * Outputs mb [n_cand][n_iter][batch] u16 (micro-batch of each sorted position),
 * v [n_cand][n_iter][32] u16 (V* per pipeline, 0 for empty/unused),
 * ptime [n_cand][n_iter][32] u64 (objective of V*), makespan [n_iter][n_cand] u64
 * (max_j ptime; UINT64_MAX if infeasible).  ws: hyd_pack_workspace() bytes; after the
 * call completes, the u64 at ws byte offset 16 holds the number of (sequence, micro-batch)
 * evaluations the LPT runs performed (diagnostic work counter for the roofline) and bytes
 * [24, 152) sixteen u64 diagnostic counters (pipelines handed between the internal passes and
 * why, per-phase SM cycles of the lane pass, its phase-2 units and tasks; assign.py names them). */
size_t hyd_pack_workspace(int n_iter, int batch, int n_cand, int max_np);
int hyd_pack(const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch, int k_pad,
             const hyd_scheme* schemes, int n_schemes, const uint8_t* cand, const uint8_t* cand_np,
             int n_cand, int max_np, const uint8_t* pipe, const hyd_pipe_stats* stats,
             const uint32_t* members, uint16_t* mb, uint16_t* v,
             uint64_t* ptime, uint64_t* makespan, uint32_t* status, void* ws, size_t ws_bytes,
             void* stream);

/* ---- a3 + a4 fused for small batches ------------------------------------------------------
 * hyd_dispatch_pack: the same results as hyd_dispatch followed by hyd_pack -- pipe, lb, mb, v,
 * ptime, makespan, bit for bit -- in one kernel for batch <= HYD_SMALL_MAX_BATCH sequences and
 * max_np <= 16 pipelines (the paper's token-budget iterations), without the
 * stats / members index (not written).  ws: hyd_dispatch_pack_workspace() bytes; the u64 at ws
 * byte 0 counts the (sequence, micro-batch) evaluations performed (diagnostic).  Larger batches
 * or candidates return HYD_E_INVALID (use hyd_dispatch + hyd_pack). */
size_t hyd_dispatch_pack_workspace(void);
int hyd_dispatch_pack(const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch, int k_pad,
                      const hyd_scheme* schemes, int n_schemes, const uint8_t* cand, const uint8_t* cand_np,
                      int n_cand, int max_np, uint8_t* pipe, uint64_t* lb, uint16_t* mb, uint16_t* v,
                      uint64_t* ptime, uint64_t* makespan, uint32_t* status, void* ws, size_t ws_bytes,
                      void* stream);

/* ---- a5: selection ---------------------------------------------------------------------
 * key[t] = min over c of (makespan[t][c] << 20 | (c + cand_offset)) among feasible
 * candidates with makespan < 2^43 (others: HYD_F_KEY_RANGE); INT64_MAX if none.  The
 * minimum key is the argmin of (makespan, c).  Across ranks, an allreduce(MIN) of key
 * (a6, done by the caller over NCCL) yields the global winner. */
int hyd_select_best(const uint64_t* makespan, int n_iter, int n_cand, int cand_offset,
                    int64_t* key, uint32_t* status, void* stream);

/* ---- winner extraction ---------------------------------------------------------------
 * For every t whose winning candidate (key[t] & (2^20-1)) - cand_offset lies in
 * [0, n_cand): win_pipe[t][perm[t][i]] = pipe[c][t][i], win_mb[t][perm[t][i]] = mb[c][t][i]
 * (ORIGINAL sequence order), win_v[t][:] = v[c][t][:], win_ptime[t][:] = ptime[c][t][:].
 * Rows of other iterations are left untouched.  Returns nothing per t; see key. */
int hyd_gather_winners(const int64_t* key, const uint32_t* perm, const uint8_t* pipe,
                       const uint16_t* mb, const uint16_t* v, const uint64_t* ptime, int n_iter,
                       int batch, int n_cand, int cand_offset, uint8_t* win_pipe, uint16_t* win_mb,
                       uint16_t* win_v, uint64_t* win_ptime, void* stream);

/* ---- end-to-end call on HOST buffers -----------------------------------------------------
 * Copies len_host [n_iter][batch] (and the scheme/candidate tables) to the device, runs
 * a1-a5, and returns the selected plan of every iteration (step 4, "select the optimal one",
 * P:446-448): key_host [n_iter], win_pipe_host [n_iter][batch], win_mb_host
 * [n_iter][batch] (ORIGINAL sequence order), win_v_host / win_ptime_host [n_iter][32] and
 * *status_host; then synchronises `stream`.  Pinned host memory gives asynchronous copies.
 * Rows of an all-infeasible iteration (key INT64_MAX) are zero.
 * Multi-GPU (one process per GPU, this rank holding candidates [cand_offset, cand_offset +
 * n_cand)): pass a collective callback `coll`.  The library calls it twice, in stream order:
 *   1. coll(key_dev, n_iter, HYD_COLL_MIN_I64, user, stream): allreduce-MIN of the int64 keys
 *      over the caller's process group (a6) -- afterwards key holds the global winners;
 *   2. coll(rows_dev, n_words, HYD_COLL_SUM_I32, user, stream): allreduce-SUM of int32 words
 *      over the winner-row block (win_pipe | win_mb | win_v | win_ptime, zero-filled, each rank
 *      writing only the rows of iterations its candidates won), so every rank ends with every
 *      iteration's plan (exactly one rank contributes a non-zero row per iteration).
 * The callback must enqueue its work on `stream` (or order it after `stream`'s prior work and
 * before its later work) and return 0; non-zero aborts with HYD_E_REDUCE.  coll = NULL: a
 * single rank (no exchange).  ws: hyd_assign_workspace() bytes of device memory. */
enum { HYD_COLL_MIN_I64 = 0, HYD_COLL_SUM_I32 = 1 };
typedef int (*hyd_collective_fn)(void* buf_dev, size_t count, int op, void* user, void* stream);
size_t hyd_assign_workspace(int n_iter, int batch, int n_schemes, int k_pad, int n_cand, int max_np);
/* byte offset of the device key buffer [n_iter] i64 inside the assign workspace */
size_t hyd_assign_key_offset(int n_iter, int batch, int n_schemes, int k_pad, int n_cand, int max_np);
int hyd_assign_host(const uint32_t* len_host, int n_iter, int batch, const hyd_scheme* schemes_host,
                    int n_schemes, int k_pad, const uint8_t* cand_host, const uint8_t* cand_np_host,
                    int n_cand, int cand_offset, int64_t* key_host, uint8_t* win_pipe_host,
                    uint16_t* win_mb_host, uint16_t* win_v_host, uint64_t* win_ptime_host,
                    uint32_t* status_host, hyd_collective_fn coll, void* coll_user, void* ws,
                    size_t ws_bytes, void* stream);

/* ---- NEXT-1: Alg. 1 as stage 1 (T random trials) ----------------------
 * hyd_alg1_permutations: the trial orders, order [n_iter][trials][batch] u16 (a permutation of
 * the sorted positions 0..batch-1 per (t, trial)): Fisher-Yates (Durstenfeld); for k = batch-1
 * down to 1: r = Philox4x32-10(counter = (k / 4, t, trial, 0), key = (seed mod 2^32,
 * seed / 2^32)) word k % 4, j = (r (k + 1)) >> 32, swap(order[k], order[j]).  One order per
 * (t, trial), shared by every candidate.  1 <= trials <= HYD_MAX_TRIALS.
 *
 * hyd_dispatch_alg1: same inputs and outputs as hyd_dispatch (pipe, lb, stats, members; the
 * pack stage is unchanged), but each (c,t) runs `trials` greedy trials: the sequences arrive
 * in order[t][trial] and each goes to the feasible pipeline j minimising
 * O_max = max(C_j' + E_j', C_k + E_k for k != j), C_j' = C_j + T(l,P_j),
 * E_j' = T(max length on j incl. l, P_j)(PP_j - 1), the first j on ties (Alg. 1 lines 5-14);
 * the trial with the smallest (O_trial = max_j C_j + E_j, trial) is kept and lb = its O.
 * best [n_cand][n_iter] u64 (caller-owned) receives O_best << 8 | trial (UINT64_MAX for an
 * infeasible pair).  ws: hyd_alg1_workspace(n_iter) bytes of device scratch. */
#define HYD_MAX_TRIALS 256
size_t hyd_alg1_workspace(int n_iter);
int hyd_alg1_permutations(uint64_t seed, int n_iter, int batch, int trials, uint16_t* order,
                          void* stream);
int hyd_dispatch_alg1(const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch,
                      int k_pad, const hyd_scheme* schemes, int n_schemes, const uint8_t* cand,
                      const uint8_t* cand_np, int n_cand, int max_np, int trials,
                      const uint16_t* order, uint64_t* best, uint8_t* pipe, uint64_t* lb,
                      hyd_pipe_stats* stats, uint32_t* members, uint32_t* status, void* ws,
                      size_t ws_bytes, void* stream);

/* ---- NEXT-2: token-budget (ragged) batches ------------------------------
 * Iteration t holds B_t sequences (1 <= B_t <= batch_max <= HYD_MAX_BATCH): offsets [n_iter+1]
 * u32 CSR on the DEVICE (offsets[0] = 0, offsets[t+1] - offsets[t] = B_t, offsets[n_iter] =
 * n_total), lengths len [n_total] concatenated by iteration.  Every iteration-indexed array
 * keeps its meaning with the row of (t, i) at offsets[t] + i: sorted_len, perm (index within
 * the iteration) [n_total], cost [n_total][k_pad], pipe [n_cand][n_total] u8,
 * mb [n_cand][n_total] u16, win_pipe / win_mb [n_total]; members rows have the stride of
 * batch_max: [n_iter][n_cand][ceil(batch_max/32)][max_np]; lb, stats, v, ptime, makespan and
 * key are unchanged.  Results are those of the uniform entry points applied to each iteration
 * separately.  Device faults: an iteration with B_t outside [1, batch_max] sets
 * HYD_F_BAD_LENGTH (hyd_cost_table_ragged) and its rows are undefined.
 * Workspaces: hyd_dispatch_workspace(n_iter), hyd_pack_workspace(n_iter, batch_max, n_cand,
 * max_np); the e2e call takes HOST offsets and checks them synchronously (HYD_E_INVALID). */
int hyd_cost_table_ragged(const uint32_t* len, int n_iter, const uint32_t* offsets, int n_total,
                          int batch_max, const hyd_scheme* schemes, int n_schemes, int k_pad,
                          uint32_t* sorted_len, uint32_t* perm, uint32_t* cost, uint32_t* status,
                          void* stream);
int hyd_dispatch_ragged(const uint32_t* sorted_len, const uint32_t* cost, int n_iter,
                        const uint32_t* offsets, int n_total, int batch_max, int k_pad,
                        const hyd_scheme* schemes, int n_schemes, const uint8_t* cand,
                        const uint8_t* cand_np, int n_cand, int max_np, uint8_t* pipe, uint64_t* lb,
                        hyd_pipe_stats* stats, uint32_t* members, uint32_t* status, void* ws,
                        size_t ws_bytes, void* stream);
int hyd_pack_ragged(const uint32_t* sorted_len, const uint32_t* cost, int n_iter,
                    const uint32_t* offsets, int n_total, int batch_max, int k_pad,
                    const hyd_scheme* schemes, int n_schemes, const uint8_t* cand,
                    const uint8_t* cand_np, int n_cand, int max_np, const uint8_t* pipe,
                    const hyd_pipe_stats* stats, const uint32_t* members, uint16_t* mb, uint16_t* v,
                    uint64_t* ptime, uint64_t* makespan, uint32_t* status, void* ws,
                    size_t ws_bytes, void* stream);
int hyd_pipe_index_ragged(const uint32_t* sorted_len, const uint32_t* cost, int n_iter,
                          const uint32_t* offsets, int n_total, int batch_max, int k_pad,
                          const hyd_scheme* schemes, int n_schemes, const uint8_t* cand,
                          const uint8_t* cand_np, int n_cand, int max_np, const uint8_t* pipe,
                          uint64_t* lb, hyd_pipe_stats* stats, uint32_t* members, uint32_t* status,
                          void* stream);
int hyd_dispatch_pack_ragged(const uint32_t* sorted_len, const uint32_t* cost, int n_iter,
                             const uint32_t* offsets, int n_total, int batch_max, int k_pad,
                             const hyd_scheme* schemes, int n_schemes, const uint8_t* cand,
                             const uint8_t* cand_np, int n_cand, int max_np, uint8_t* pipe, uint64_t* lb,
                             uint16_t* mb, uint16_t* v, uint64_t* ptime, uint64_t* makespan,
                             uint32_t* status, void* ws, size_t ws_bytes, void* stream);
int hyd_gather_winners_ragged(const int64_t* key, const uint32_t* perm, const uint8_t* pipe,
                              const uint16_t* mb, const uint16_t* v, const uint64_t* ptime,
                              int n_iter, const uint32_t* offsets, int n_total, int batch_max,
                              int n_cand, int cand_offset, uint8_t* win_pipe, uint16_t* win_mb,
                              uint16_t* win_v, uint64_t* win_ptime, void* stream);
size_t hyd_assign_workspace_ragged(int n_iter, int n_total, int batch_max, int n_schemes, int k_pad,
                                   int n_cand, int max_np);
size_t hyd_assign_key_offset_ragged(int n_iter, int n_total, int batch_max, int n_schemes,
                                    int k_pad, int n_cand, int max_np);
int hyd_assign_host_ragged(const uint32_t* len_host, int n_iter, const uint32_t* offsets_host,
                           int batch_max, const hyd_scheme* schemes_host, int n_schemes, int k_pad,
                           const uint8_t* cand_host, const uint8_t* cand_np_host, int n_cand,
                           int cand_offset, int64_t* key_host, uint8_t* win_pipe_host,
                           uint16_t* win_mb_host, uint16_t* win_v_host, uint64_t* win_ptime_host,
                           uint32_t* status_host, hyd_collective_fn coll, void* coll_user, void* ws,
                           size_t ws_bytes, void* stream);

/* ---- NEXT-3: strategy-proposal dynamic programme (§5) -------------------------
 * lengths [n_seq] u32 (device): a sample of the dataset's sequence lengths, truncated to the
 * context J * step.  Length grid l = j * step (j = 0..J), GPU grid n = nu / scale
 * (nu = 0..n_gpus * scale; scale 1 = the integer DP, 10 = the 0.1-step continuous relaxation).
 *   t[n][l] = min(t[n-1][l], min over (k, d, l') of max(t[n - d N(P_k)][l - l'],
 *             (1/d) sum_{x in (l - l', l]} T(x, P_k))),  MaxLen(P_k) >= l, d N(P_k) <= n,
 *   t[n][0] = 0, t[0][l > 0] = infinity; N(P_k) = tp * pp * cp.
 * Outputs (caller-owned device buffers):
 *   t_num, t_den [(n_gpus*scale + 1)][J + 1] u64: t = t_num / t_den exactly (t_den 0 = infinity;
 *     t_num = scale * (sum of T) of the binding interval, t_den = scale * d);
 *   choice [(n_gpus*scale + 1)][J + 1] i32: -1 = t[n-1][l] (carry), -2 = base state, else
 *     k << 24 | (d * scale) << 12 | l'/step (ties: carry, then k, d, l' ascending);
 *   counts [J + 1][n_schemes] u16: S[N][l]'s pipelines per scheme in units of 1/scale;
 *   rows [J + 1][HYD_DP_MAX_ROUND][n_schemes] u8, valid [J + 1][HYD_DP_MAX_ROUND] u8: the integer
 *     candidates near S[N][l] (every non-integer d_k rounded down or up; combination m takes the
 *     ceiling for the q-th non-integer scheme, ascending k, iff bit q of m is set; valid iff
 *     within n_gpus GPUs and the scheme of the longest interval keeps a pipeline);
 *   keep [J + 1][HYD_DP_MAX_ROUND] u8: 1 for the first occurrence of each valid candidate in
 *     (l, m) order -- the proposed subset is the rows with keep = 1.
 * Limits: 1 <= n_schemes <= HYD_MAX_SCHEMES, 1 <= J, n_gpus * scale <= 4095, step >= 1,
 * J * step <= HYD_LEN_LIMIT.  More than log2(HYD_DP_MAX_ROUND) non-integer d_k set HYD_F_OVERFLOW
 * (that l proposes nothing).  ws: hyd_dp_workspace(n_schemes, J) bytes. */
#define HYD_DP_MAX_ROUND 64
size_t hyd_dp_workspace(int n_schemes, int J);
int hyd_dp_propose(const uint32_t* lengths, int n_seq, const hyd_scheme* schemes, int n_schemes,
                   int step, int J, int n_gpus, int scale, uint64_t* t_num, uint64_t* t_den,
                   int32_t* choice, uint16_t* counts, uint8_t* rows, uint8_t* valid, uint8_t* keep,
                   uint32_t* status, void* ws, size_t ws_bytes, void* stream);

/* hyd_dp_candidates: the proposed subset of a hyd_dp_propose result (rows / keep) as the
 * candidate tables hyd_dispatch takes, in first-occurrence (l, m) order: cand [M][32] u8 with
 * the pipelines in canonical order (MaxLen non-increasing, scheme index ascending),
 * each scheme repeated by its pipeline count, padded with 0xFF; cand_np [M] u8 (0 for a row
 * with more than HYD_MAX_PIPES pipelines); *n_out (device i32) = M.  Capacity: (J + 1) *
 * HYD_DP_MAX_ROUND rows.  schemes: the table passed to hyd_dp_propose. */
int hyd_dp_candidates(const uint8_t* rows, const uint8_t* keep, int J, const hyd_scheme* schemes,
                      int n_schemes, uint8_t* cand, uint8_t* cand_np, int32_t* n_out, void* stream);

/* ---- NEXT-4: exact Eq. 3 optimum for small batches (gap study P:654) --------------
 * For each listed (pair_c[p], pair_t[p]): the minimum over every dispatch (each sequence on a
 * pipeline with MaxLen >= l) of max_j LB_j, LB_j = sum T(l, P_j) + T(max l, P_j)(PP_j - 1)
 * (Eq. 2), by branch-and-bound (exact pruning only), started from the HYD-H1 greedy dispatch.
 * Inputs as hyd_dispatch (uniform batches, sorted_len / cost from hyd_cost_table).
 * Outputs: value [n_pairs] u64 (the optimum; UINT64_MAX for an infeasible pair), pipe
 * [n_pairs][batch] u8 (an optimal assignment by sorted position; ties between optima are not
 * specified), nodes [n_pairs] u64 (search nodes), proved [n_pairs] u8 (0: the node budget
 * ran out; value / pipe are then the best found).
 * Limits: batch <= HYD_BB_MAX_BATCH, max_np <= 8. */
#define HYD_BB_MAX_BATCH 64
int hyd_eq3_exact(const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch, int k_pad,
                  const hyd_scheme* schemes, int n_schemes, const uint8_t* cand,
                  const uint8_t* cand_np, int n_cand, const int32_t* pair_c, const int32_t* pair_t,
                  int n_pairs, uint64_t node_limit, uint64_t* value, uint8_t* pipe, uint64_t* nodes,
                  uint8_t* proved, uint32_t* status, void* stream);

/* Exact Eq. 1 per listed pipeline (pair_c, pair_t, pair_j) of a dispatched batch
 * (members / sorted_len / cost from hyd_dispatch and hyd_cost_table): min over V in App. D's
 * range (extended upward while none is feasible) and every split of the pipeline's sequences
 * into V non-empty micro-batches within MaxLen of (max micro-batch time)(PP - 1 + V), ties to
 * the smaller V, by branch-and-bound from the LPT(V) incumbent.  Outputs v [n] u32 (0 if the
 * pipeline is empty or nothing was proved), obj [n] u64, nodes [n] u64, proved [n] u8.
 * Limits: at most 32 sequences per pipeline (larger ones report proved = 0). */
int hyd_eq1_exact(const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch, int k_pad,
                  const hyd_scheme* schemes, int n_schemes, const uint8_t* cand, int n_cand,
                  int max_np, const uint32_t* members, const int32_t* pair_c, const int32_t* pair_t,
                  const int32_t* pair_j, int n_pairs, uint64_t node_limit, uint32_t* v,
                  uint64_t* obj, uint64_t* nodes, uint8_t* proved, uint32_t* status, void* stream);

/* ---- host utilities --------------------------------------------------------------------
 * hyd_check_candidates: HOST tables; HYD_OK, HYD_E_INVALID or HYD_E_NOT_CANONICAL; writes
 * max over c of cand_np to *max_np_out (if non-null). */
int hyd_check_candidates(const uint8_t* cand_host, const uint8_t* cand_np_host, int n_cand,
                         const hyd_scheme* schemes_host, int n_schemes, int* max_np_out);
const char* hyd_status_string(int code); /* static string for a HYD_E_* code */
const char* hyd_last_cuda_error(void);   /* static string of the last CUDA error seen */
int hyd_kernel_launches(void);           /* kernel launches issued by this library so far */

#ifdef __cplusplus
}
#endif
#endif
