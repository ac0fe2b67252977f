// pack.cu -- a4: stage 2 sequence packing within each pipeline (§6.1, App. D).
//
// For every (c, t, j): the pipeline's sequences Q in sorted (longest-first) order,
// U = |Q|, S = sum l, sumT = sum tau, tau_max = tau of Q[0] (T non-decreasing in l).
//   V range (App. D): [max(ceil(S/MaxLen),1), min(floor(S/UtilLen),U)], clamped up.
//   LPT(V): each item to the least-time bin whose tokens stay <= MaxLen (Eq. 1 constraint,
//   P:606-607), smallest bin on ties; objective (max bin time)(PP-1+V) (Eq. 1).
//   V* = argmin (objective, V); if no V in range is feasible, the smallest feasible V above.
//
// Exact pruned V search (never changes the result; SURVEY §8(c) "freedom"):
//   obj(V) >= LB(V) = max(sumT (PP-1+V)/V, tau_max (PP-1+V))   (average and largest item)
//   1. evaluate V_a first: V_lo if PP = 1 (LB flat, smaller V wins ties), else the integer
//      nearest sumT/tau_max (the real minimiser of LB), clamped to the range;
//   2. scan V ascending; stop when tau_max(PP-1+V) > best (or >= best with V > V_best):
//      that term only grows with V; skip V when sumT(PP-1+V) > best V (or >= with V > V_best);
//   3. inside LPT(V), abort as soon as the running max bin time exceeds
//      floor(best/(PP-1+V)) (or floor((best-1)/(PP-1+V)) when V > V_best) -- bins only grow.
//   A completed run therefore always improves (obj, V); its bin ids (kept in shared memory)
//   are then copied to mb.
//
// Three kernels (all stream-ordered after hyd_dispatch, which supplies U, S, sumT, tau_max):
//   (the VMAX-16 pass also writes every (c,t) row of v / ptime / makespan and the mb rows of
//    infeasible pairs, so no separate initialisation kernel runs)
//   k_pack_lanes: one LANE per pipeline task, persistent inside a CTA that owns one iteration
//     (its lengths + cost rows staged in smem) and ~2048 (c,j) tasks sorted into VMAX classes
//     8 / 16 by V_a.  Each loop iteration advances one sequence of the lane's current LPT run
//     (or sets up its next task), so lanes never wait for each other's runs or tasks.  Members
//     are found in sorted order by 16-byte SIMD byte compares on the pipe row; bins are packed
//     u32 keys time<<5|b with a sign-bit capacity mask (3 ops per bin for the argmin, 3 to
//     place).  The first run (V_a, never aborted) writes mb directly; if a later V wins, a final
//     run rewrites it.  Tasks needing V > 16, sumT >= 2^26 or a ragged batch are queued.
//   k_pack_big: persistent warps pop queued (c,t,j) tasks; the WARP owns one pipeline, lanes own
//     bins b = lane + 32 r (r < R <= 8 in registers, or global scratch beyond 256 bins); per
//     item a redux.sync min over times, then over bin ids, picks the bin.
//   makespan[t][c] = max_j ptime via atomicMax from the tasks.
#include <type_traits>

#include "hyd_internal.cuh"
#include "search.cuh"

namespace hyd {

constexpr int kLaneThreads = 256;
// flagged VMAX-32 tasks in all (counted by k_flag_list) up to which the warp queue takes them
constexpr unsigned long long kFlaggedToQueue = 16384;
constexpr size_t kLaneSmem16 = 74 * 1024;   // VMAX 16 pass: 3 CTAs per SM
constexpr size_t kLaneSmem32 = 110 * 1024;  // VMAX 32 pass: 2 CTAs per SM
constexpr int kLaneEpoch = 24;     // sequences per lane between bookkeeping phases
constexpr int kChunk32 = 400;      // flagged tasks per staged VMAX-32 CTA (measured: 2048 / 512 / 400 / 256)
constexpr int kBigRMax = 8;       // k_pack_big: register bins per lane (V <= 256)
constexpr int kBigWarps = 3584;   // persistent warps of k_pack_big (scratch slots): 148 SMs x 24
// A short warp queue (at most kSplitTasks pipelines) runs split: every task's reference run, then
// its surviving V as independent units spread over all warps, then the winners' re-runs -- so the
// queue's duration is a few runs, not its longest sequential search.
#ifndef HYD_SPLIT_TASKS  // the debug build sets 0: its queue always runs the sequential search
#define HYD_SPLIT_TASKS (1 << 21)
#endif
constexpr int kSplitTasks = HYD_SPLIT_TASKS;
constexpr int kSplitUnits = 1 << 24;

struct PackArgs {
  const uint32_t* sorted_len;
  const uint32_t* cost;
  int n_iter, batch, k_pad;  // batch: the largest batch (row stride of members, scratch)
  uint32_t kp4;              // 4 k_pad: the staged cost row stride in bytes
  const uint32_t* off;       // ragged CSR offsets [n_iter + 1] or nullptr (uniform)
  size_t n_total;            // rows of iteration-indexed arrays (n_iter * batch if uniform)
  const hyd_scheme* schemes;
  int n_schemes;
  const uint8_t* cand;
  const uint8_t* cand_np;
  int n_cand;
  const uint8_t* pipe;
  const hyd_pipe_stats* stats;
  const uint32_t* members;  // [It][C][nwords][mnp] membership words from hyd_dispatch
  int mnp, nwords;
  uint16_t* mb;
  uint16_t* v;
  uint64_t* ptime;
  uint64_t* makespan;
  uint32_t* status;
  // q_count points at a 256-byte counter block (ws bytes [0, 256), zeroed per call): [0] queued
  // tasks, [1] queue head, [2] evaluations, [3..18] diagnostic counters, [19] split units
  // reserved, [20] split unit head, [21] flagged VMAX-32 tasks in all
  unsigned long long* q_count;
  unsigned long long* q_head;
  unsigned long long* evals;  // (item, bin) evaluations performed (ws bytes [16, 24))
  unsigned long long* why;    // diagnostic counters (ws bytes [24, 152)): hand-offs, phase cycles
  unsigned long long* queue;
  unsigned long long q_cap;
  uint32_t* flags;  // [It*C*mnp bits] tasks handed from the VMAX-16 to the VMAX-32 lane pass
  unsigned long long* sp_key;  // [kSplitTasks] split warp queue: best (obj << 16 | V) per queued task
  uint32_t* sp_wv;             // [kSplitTasks] the V whose mb the reference run wrote (0: task done in A)
  unsigned long long* units;   // [kSplitUnits] (task << 16 | V) candidate runs of the split queue
  uint32_t* list32;   // [It][C*mnp] the flagged tasks of each iteration, compacted (c*mnp + j)
  uint32_t* count32;  // [It] their number
  uint64_t* scr_time;  // [kBigWarps][B]
  uint32_t* scr_tok;   // [kBigWarps][B]
};

// ------------------------------------------------------------------ pair-level init
// makespan = 0 (feasible) or UINT64_MAX (infeasible); v/ptime rows zeroed; infeasible
// pairs get mb = 0xFFFF.  Tasks then write their v/ptime slot and atomicMax the makespan.
// ------------------------------------------------------------------ persistent lanes (V <= 32)
// bins as packed u32 keys: key_b = time_b << SH | b, and rem_b = MaxLen - tokens of bin b.
// SH = 4 for VMAX 16 (sumT < 2^27), 5 for VMAX 32 (sumT < 2^26).  masked_b = key_b |
// ((rem_b - l) & 2^31) is >= 2^31 iff tok_b + l > MaxLen, so the minimum masked key is the
// least-time fitting bin with the smallest index; the chosen bin's new rem is rem_b - l, the
// difference the mask already formed.
template <int VM>
struct LaneCfg {
  static constexpr int SH = VM <= 16 ? 4 : 5;
  static constexpr uint64_t SUMT_LIMIT = 1ull << (31 - SH);
};

constexpr int pow2_ceil(int n) { return n <= 1 ? 1 : 2 * pow2_ceil((n + 1) / 2); }

template <int N, int VM>
__device__ __forceinline__ uint32_t argmin_keys(const uint32_t (&keys)[VM],
                                                const uint32_t (&rem)[VM], uint32_t l) {
  uint32_t m[N];
#pragma unroll
  for (int b = 0; b < N; ++b) m[b] = keys[b] | ((rem[b] - l) & 0x80000000u);
  return min_tree3<N>(m);
}

// place the item in the bin whose key is mk (no bin when mk = 0xFFFFFFFF): one compare and two
// predicated updates per bin (the C++ form compiles to compare + 2 SEL + 2 IADD)
template <int N, int VM>
__device__ __forceinline__ void place_key(uint32_t (&keys)[VM], uint32_t (&rem)[VM], uint32_t mk,
                                          uint32_t tau_sh, uint32_t l) {
#pragma unroll
  for (int b = 0; b < N; ++b)
    asm("{\n\t.reg .pred p;\n\t"
        "setp.eq.u32 p, %0, %2;\n\t"
        "@p add.u32 %0, %0, %3;\n\t"
        "@p sub.u32 %1, %1, %4;\n\t}"
        : "+r"(keys[b]), "+r"(rem[b])
        : "r"(mk), "r"(tau_sh), "r"(l));
}

// Capacity-free runs (an exact shortcut): with alpha = min_i tau_i / l_i over
// the iteration's sequences that scheme k can hold, every bin satisfies alpha * tokens <= time.
// A run whose abort threshold thr satisfies thr <= cap_k = floor(alpha MaxLen_k) can never place
// a sequence into a bin it overflows without that bin's time exceeding thr (which aborts the run
// under either rule, and the capacity rule would pick a bin of no smaller time), so LPT with and
// without the capacity mask agree step for step.  Such runs skip the mask and the token updates;
// a warp whose units are all capacity-free takes this path (bin tokens of those units go stale,
// which can only let a later masked step see a bin as fitting -- and every bin fits for them).
template <int N, int VM>
__device__ __forceinline__ uint32_t min_keys(const uint32_t (&keys)[VM]) {
  uint32_t m[N];
#pragma unroll
  for (int b = 0; b < N; ++b) m[b] = keys[b];
  return min_tree3<N>(m);
}

template <int N, int VM>
__device__ __forceinline__ void add_key(uint32_t (&keys)[VM], uint32_t mk, uint32_t nk) {
#pragma unroll
  for (int b = 0; b < N; ++b)
    asm("{\n\t.reg .pred p;\n\t"
        "setp.eq.u32 p, %0, %1;\n\t"
        "@p mov.u32 %0, %2;\n\t}"
        : "+r"(keys[b])
        : "r"(mk), "r"(nk));
}

// per-CTA task records (compacted slots), built in parallel before the lane phases
struct TaskRecs {
  unsigned long long* key;  // best (obj << 16 | V) found so far
  uint32_t* sum_t;
  uint32_t* tau_max;
  uint32_t* eid;    // tile-local task id: (candidate - c0) * mnp + j
  uint32_t* list2;  // phase-2 units: slot << 16 | V (class 16 from the front, class 8 from the middle)
  uint16_t* u;
  uint16_t* vlo;
  uint16_t* vhi;
  uint16_t* va;
  uint16_t* perm;   // phase-1 order of slots (longest-processing-time first)
  uint16_t* ncand;  // phase-2 candidate count
  uint8_t* k;
  uint8_t* state;   // 0 active, 1 handed to another pass
  uint8_t* cbucket; // phase-2 bucket
};

// one bulk L2 prefetch of a contiguous block (TMA engine), clipped to 16-byte granules
__device__ __forceinline__ void prefetch_l2_block(const void* base, size_t off, size_t bytes, size_t total) {
  size_t lo = off & ~(size_t)15, hi = (off + bytes + 15) & ~(size_t)15;
  if (hi > (total & ~(size_t)15)) hi = total & ~(size_t)15;
  if (hi <= lo) return;
  const char* p = static_cast<const char*>(base) + lo;
  size_t n = hi - lo;
  while (n) {
    const uint32_t chunk = n > (1u << 20) ? (1u << 20) : (uint32_t)n;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(chunk) : "memory");
    p += chunk;
    n -= chunk;
  }
}

// One LPT run as a lane's unit of work (state carried across loop iterations).
template <int VM>
struct LaneUnit {
  uint32_t keys[VM], rem[VM];  // rem_b = MaxLen - tokens of bin b
  const uint32_t* mw;
  uint16_t* mrow;
  uint32_t qw, cur, wbase, nxtw;
  uint32_t V, thr, mx, k, M;
  uint32_t tb;  // STAGED: shared-window address of the cost column k (row 0)
  uint32_t pi, pl, pt;  // !STAGED: the next member's index, length and cost, loaded a step early
#ifdef HYD_DEBUG_CHECKS
  uint32_t bt;  // the iteration's sequences (member indices must stay below)
#endif
  int e;
  bool write;
  bool F;  // capacity-free: no placement of this run can exceed MaxLen before it completes or aborts
};

template <int VM>
__device__ __forceinline__ void unit_start(LaneUnit<VM>& u, uint32_t V, uint32_t thr) {
  u.V = V;
  u.thr = thr;
  u.mx = 0;
#pragma unroll
  for (int b = 0; b < VM; ++b) {
    u.keys[b] = (uint32_t)b < V ? (uint32_t)b : 0xFFFFFFFEu;  // unused: never fits, never 'mk'
    u.rem[b] = u.M;
  }
  u.qw = 0;
  u.cur = 0;
  u.nxtw = __ldg(u.mw);  // word w of the pipeline at mw[w * mnp]
  u.pi = 0xFFFFFFFFu;
}

// Advance the unit by one sequence.  Returns 0 while running, 1 when the run completed,
// 2 when it failed (no micro-batch fits: LPT(V) infeasible, or it cannot beat u.thr).
// Straight-line apart from the membership-word refill: a lane whose current word is used up
// takes the next one (an all-zero word costs it one idle step), and the step's placement is
// predicated on having a member, so the warp never splits inside the bin arithmetic.
// STAGED: lengths at sm[0, B), costs at sm[B + i * kp + k] (shared window, 32-bit addressing).
__device__ __forceinline__ uint32_t ld_shared_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// PH: the lane phase the run belongs to -- 1: V_a runs (write mb, no threshold), 2: candidate runs
// (threshold, no mb), 3: winner re-runs (write mb; neither the threshold nor the maximum is needed)
template <int N, int VM, bool STAGED, bool FREE, int PH>
__device__ __forceinline__ int unit_step(LaneUnit<VM>& u, uint32_t nwords, uint32_t mnp, uint32_t sbase,
                                         const uint32_t* __restrict__ slen,
                                         const uint32_t* __restrict__ cst, int kp, uint32_t kp4, uint32_t& ev) {
  constexpr int SH = LaneCfg<VM>::SH;
  if (u.cur == 0 && u.qw < nwords) {
    u.cur = u.nxtw;
    u.wbase = u.qw * 32u;
    ++u.qw;
    u.nxtw = u.qw < nwords ? __ldg(u.mw + u.qw * mnp) : 0u;
  }
  const bool valid = u.cur != 0u;
  const uint32_t i = valid ? u.wbase + (uint32_t)(__ffs(u.cur) - 1) : 0u;
  u.cur &= u.cur - 1u;
  // STAGED: 32-bit shared-window addresses (sbase: lengths; u.tb + 4 kp i: the cost of row i)
  HYD_CHECK(!valid || i < u.bt);
  uint32_t tau, l;
  if constexpr (STAGED) {
    tau = ld_shared_u32(u.tb + i * kp4);
    l = FREE ? 0u : ld_shared_u32(sbase + i * 4u);
  } else {  // L2 reads: this member's were issued a step early; issue the next member's now
    const bool pre = u.pi == i;
    tau = pre ? u.pt : cst[(size_t)i * kp + u.k];
    l = FREE ? 0u : (pre ? u.pl : slen[i]);
    const uint32_t i2 = u.cur ? u.wbase + (uint32_t)(__ffs(u.cur) - 1)
                              : (u.qw < nwords && u.nxtw ? u.qw * 32u + (uint32_t)(__ffs(u.nxtw) - 1) : 0xFFFFFFFFu);
    u.pi = i2;
    if (i2 != 0xFFFFFFFFu) {  // (the length too in capacity-free steps: the warp's next epoch may be masked)
      u.pt = cst[(size_t)i2 * kp + u.k];
      u.pl = slen[i2];
    }
  }
  uint32_t m0;
  if constexpr (FREE) {  // capacity cannot bind: plain least-time bin, bin tokens not tracked
    m0 = min_keys<N, VM>(u.keys);
  } else {
    m0 = argmin_keys<N, VM>(u.keys, u.rem, l);
  }
  const bool ok = valid && (m0 >> 31) == 0u;
  const uint32_t mk = ok ? m0 : 0xFFFFFFFFu;  // matches no bin key: placement is a no-op
  if constexpr (FREE) {
    add_key<N, VM>(u.keys, mk, mk + (tau << SH));  // the chosen key's new value, computed once
  } else {
    place_key<N, VM>(u.keys, u.rem, mk, tau << SH, l);
  }
  if (PH != 3) u.mx = ok ? max(u.mx, (mk >> SH) + tau) : u.mx;
  if (PH != 2 && ok) u.mrow[i] = (uint16_t)(mk & ((1u << SH) - 1u));
  ev += valid ? u.V : 0u;
  if (!valid) return u.qw >= nwords ? 1 : 0;  // every member placed / empty word
  return (!ok || (PH == 2 && u.mx > u.thr)) ? 2 : 0;
}

// VM = 16: every (c,t,j) of the tile, classes 8 / 16; a task needing some V > 16 is flagged
//          for the VM = 32 pass.  VM = 32: flagged tasks only (tiles of up to 2048 candidates, records
//          compacted).  Tasks the lanes cannot hold (V > VM in the last pass, sumT over the key
//          limit, no feasible LPT(V) for V_a <= V <= min(V_hi, VM)) go to the warp queue, which runs the sequential
//          exact search.
template <bool STAGED, int VM>
__global__ void __launch_bounds__(kLaneThreads, VM == 16 ? 3 : 2) k_pack_lanes(PackArgs a, int tc, int mnp, int ncap) {
  constexpr int NB = 128;  // LPT-order buckets: (class, mode, U) descending (phase 1: 64 used)
  constexpr unsigned long long kBottom = ~0ull;
  extern __shared__ __align__(16) uint32_t sm[];
  __shared__ int s_next, s_nrec, s_n2a, s_n2b;
  __shared__ int s_hist[NB];
  __shared__ uint32_t s_ml[HYD_MAX_SCHEMES], s_pp[HYD_MAX_SCHEMES], s_ul[HYD_MAX_SCHEMES];
  __shared__ uint32_t s_cap[HYD_MAX_SCHEMES];  // floor(alpha_k MaxLen_k), see min_keys
  const int kp = a.k_pad;
  // VMAX 16: CTA = (candidate tile, iteration); VMAX 32: CTA = (chunk of <= ncap of the
  // iteration's flagged tasks from the compacted list, iteration), task ids c * mnp + j (c0 = 0)
  const int t = blockIdx.y, c0 = VM == 16 ? blockIdx.x * tc : 0;
  const int chunk0 = VM == 32 ? blockIdx.x * ncap : 0;
  const int nchunk = VM == 32 ? min(ncap, (int)a.count32[t] - chunk0) : 0;
  if (VM == 32 && nchunk <= 0) return;
  if (VM == 32 && a.q_count[21] <= kFlaggedToQueue) {
    // few flagged tasks in all (configs 2 and 3: ~1 and ~40 per iteration): a CTA per iteration
    // would mostly stage and wait, so they go to the warp queue, which runs the same exact
    // search from scratch (same V*, ptime and mb) right after this pass
    const size_t lbase = (size_t)blockIdx.y * ((size_t)a.n_cand * mnp) + chunk0;
    for (int q = threadIdx.x; q < nchunk; q += kLaneThreads) {
      const int e = (int)a.list32[lbase + q];
      const unsigned long long slot = atomicAdd(a.q_count, 1ull);
      if (slot < a.q_cap)
        a.queue[slot] = ((unsigned long long)(e / mnp) << 37) | ((unsigned long long)blockIdx.y << 5) | (unsigned)(e % mnp);
    }
    return;
  }
  const int B = geo_bt(a.off, a.batch, t);  // this iteration's sequences
  const size_t tbase = geo_base(a.off, a.batch, t);
  const int tid = threadIdx.x, lane = tid & 31;
  const int ncl = VM == 16 ? min(tc, a.n_cand - c0) : a.n_cand;
  const int ntile = ncl * mnp;  // task ids of the tile
  const uint32_t nwords = (uint32_t)a.nwords;           // member row stride (largest batch)
  const uint32_t nwords_t = (uint32_t)((B + 31) >> 5);  // words of this iteration
  const size_t fbase = ((size_t)t * a.n_cand + c0) * mnp;  // first task bit / stats row of the tile
  if (tid == 0 && VM == 16) {  // this CTA's stats and membership rows are contiguous: pull them into L2
    const size_t total_rows = (size_t)a.n_iter * a.n_cand * mnp;
    prefetch_l2_block(a.members, fbase * nwords * 4, (size_t)ntile * nwords * 4, total_rows * nwords * 4);
    prefetch_l2_block(a.stats, fbase * sizeof(hyd_pipe_stats), (size_t)ntile * sizeof(hyd_pipe_stats),
                      total_rows * sizeof(hyd_pipe_stats));
  }
  // dynamic smem: [stage B*(1+kp) u32] [key u64] [sum_t, tau_max, eid, list2 u32]
  //               [u, vlo, vhi, va, perm, ncand u16] [k, state, cbucket u8]   (ncap slots each)
  uint32_t* recbase = sm + (STAGED ? (((size_t)a.batch * (1 + kp) + 3) & ~(size_t)3) : 0);  // 16 B
  TaskRecs R;
  R.key = reinterpret_cast<unsigned long long*>(recbase);
  R.sum_t = reinterpret_cast<uint32_t*>(R.key + ncap);
  R.tau_max = R.sum_t + ncap;
  R.eid = R.tau_max + ncap;
  R.list2 = R.eid + ncap;
  R.u = reinterpret_cast<uint16_t*>(R.list2 + ncap);
  R.vlo = R.u + ncap;
  R.vhi = R.vlo + ncap;
  R.va = R.vhi + ncap;
  R.perm = R.va + ncap;
  R.ncand = R.perm + ncap;
  R.k = reinterpret_cast<uint8_t*>(R.ncand + ncap);
  R.state = R.k + ncap;
  R.cbucket = R.state + ncap;
  if (tid == 0) {
    s_next = 0;
    s_nrec = 0;
    s_n2a = 0;
    s_n2b = 0;
  }
  for (int b = tid; b < NB; b += kLaneThreads) s_hist[b] = 0;
  for (int k = tid; k < a.n_schemes; k += kLaneThreads) {
    s_ml[k] = a.schemes[k].max_len;
    s_pp[k] = a.schemes[k].pp;
    s_ul[k] = a.schemes[k].util_len;
  }
  __syncthreads();

  auto to_queue = [&](int c, int j) {
    const unsigned long long slot = atomicAdd(a.q_count, 1ull);
    if (slot < a.q_cap)
      a.queue[slot] = ((unsigned long long)c << 37) | ((unsigned long long)t << 5) | (unsigned)j;
  };
  auto hand_off_e = [&](int e) {  // the task leaves this pass
    const int c = c0 + e / mnp, j = e % mnp;
    if (VM == 16) {
      const size_t bit = fbase + e;
      atomicOr(a.flags + (bit >> 5), 1u << (bit & 31));
    } else {
      to_queue(c, j);
    }
  };

  long long t_mark = clock64();
  auto phase_clock = [&](int slot) {  // diagnostic: per-phase SM cycles (thread 0, VM = 16)
    if (VM == 16 && tid == 0) {
      const long long now = clock64();
      atomicAdd(a.why + 8 + slot, (unsigned long long)(now - t_mark));
      t_mark = now;
    }
  };
  // ---- task records (parallel, compacted), bucketed by (class, U) for LPT-order processing
  for (int q = tid; q < (VM == 16 ? ntile : nchunk); q += kLaneThreads) {
    const int e = VM == 16 ? q : (int)a.list32[(size_t)t * ((size_t)a.n_cand * mnp) + chunk0 + q];
    const int c = c0 + e / mnp, j = e % mnp;
    if (j >= (int)a.cand_np[c]) continue;
    const hyd_pipe_stats* sp = a.stats + (fbase + e - j);
    if (VM == 16 && sp[0].u == 0xFFFFFFFFu) continue;  // infeasible pair: rows written below
    const hyd_pipe_stats st = sp[j];
    if (st.u == 0) continue;  // empty pipeline: V = ptime = 0 (row writes)
    const uint32_t k = a.cand[(size_t)c * HYD_MAX_PIPES + j];
    Search s;
    s.M = s_ml[k];
    s.P = s_pp[k];
    s.UL = s_ul[k];
    s.U = st.u;
    s.S = st.s;
    s.sumT = st.sum_t;
    s.tau_max = st.tau_max;
    search_init(s);
    if (s.sumT >= LaneCfg<VM>::SUMT_LIMIT || s.M >= 0x80000000u || (VM == 32 && s.va > 32u)) {
      atomicAdd(a.why + (VM == 16 ? 0 : 4), 1ull);
      to_queue(c, j);
      continue;
    }
    if (VM == 16 && s.va > 16u) {
      atomicAdd(a.why + 1, 1ull);
      hand_off_e(e);
      continue;
    }
    const int r = atomicAdd(&s_nrec, 1);
    if (r >= ncap) {  // record space full (cannot happen: tiles / chunks hold at most ncap tasks)
      atomicAdd(a.why + 7, 1ull);
      to_queue(c, j);
      continue;
    }
    R.eid[r] = (uint32_t)e;
    R.sum_t[r] = (uint32_t)s.sumT;
    R.tau_max[r] = s.tau_max;
    R.u[r] = (uint16_t)s.U;
    R.vlo[r] = (uint16_t)s.vlo;
    R.vhi[r] = (uint16_t)s.vhi;
    R.va[r] = (uint16_t)s.va;
    R.k[r] = (uint8_t)k;
    R.state[r] = 0;
    const int ub = min(31, (int)(s.U >> 3));
    const int bk = (VM == 16 && s.va <= 8) ? ub : 32 + ub;  // heavier class first, then larger U
    R.perm[r] = (uint16_t)bk;  // bucket, replaced by the order below
    HYD_CHECK(bk >= 0 && bk < NB && r < ncap);
    atomicAdd(&s_hist[bk], 1);
  }
  __syncthreads();
  const int nrec = min(s_nrec, ncap);
  // VMAX-16 pass: this CTA owns the (c, t) rows of its tile and writes them whole -- v and ptime
  // (32 slots: its tasks' results, 0 elsewhere; tasks handed to later passes overwrite their
  // slot), makespan (max over its tasks; later passes atomicMax into it) and, for an infeasible
  // pair, UINT64_MAX and a 0xFFFF mb row -- one warp per candidate, full-sector row stores.
  auto write_rows = [&](int nr) {
    uint16_t* map = R.perm;  // free after phase 1: tile task id -> record slot
    for (int e = tid; e < ntile; e += kLaneThreads) map[e] = 0xFFFFu;
    __syncthreads();
    for (int r = tid; r < nr; r += kLaneThreads)
      if (R.state[r] != 1) map[R.eid[r]] = (uint16_t)r;
    __syncthreads();
    const int warp = tid >> 5;
    for (int cc = warp; cc < ncl; cc += kLaneThreads / 32) {
      const int c = c0 + cc;
      const size_t row = (size_t)c * a.n_iter + t;
      const bool feasible = a.stats[(fbase + (size_t)cc * mnp)].u != 0xFFFFFFFFu;
      auto slot_key = [&](int j) -> unsigned long long {
        if (j >= mnp || !feasible) return 0ull;
        const uint16_t r = map[cc * mnp + j];
        return r == 0xFFFFu ? 0ull : R.key[r];
      };
      unsigned long long mx = 0ull;
      if (lane < 4) {  // v: 8 slots per 16-byte chunk
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          w[q] = (uint32_t)(slot_key(8 * lane + 2 * q) & 0xFFFFu) |
                 ((uint32_t)(slot_key(8 * lane + 2 * q + 1) & 0xFFFFu) << 16);
        reinterpret_cast<uint4*>(a.v + row * HYD_MAX_PIPES)[lane] = make_uint4(w[0], w[1], w[2], w[3]);
      } else if (lane < 20) {  // ptime: 2 slots per 16-byte chunk
        const int j = 2 * (lane - 4);
        const unsigned long long p0 = slot_key(j) >> 16, p1 = slot_key(j + 1) >> 16;
        mx = max(p0, p1);
        reinterpret_cast<ulonglong2*>(a.ptime + row * HYD_MAX_PIPES)[lane - 4] = make_ulonglong2(p0, p1);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(HYD_FULL, mx, o));
      if (lane == 0) a.makespan[(size_t)t * a.n_cand + c] = feasible ? (uint64_t)mx : ~0ull;
      if (!feasible) {
        uint16_t* mrow = a.mb + (size_t)c * a.n_total + tbase;
        for (int i = lane; i < B; i += 32) mrow[i] = 0xFFFF;
      }
    }
  };
  if (nrec == 0) {
    if (VM == 16) write_rows(0);
    return;
  }
  if (tid == 0) {  // exclusive scan over the 64 buckets in descending order
    int run = 0;
    for (int b = NB - 1; b >= 0; --b) {
      const int h = s_hist[b];
      s_hist[b] = run;
      run += h;
    }
  }
  __syncthreads();
  {
    // bucket -> position (list2 is free until phase 1.5: used as scratch for the order)
    for (int r0 = 0; r0 < nrec; r0 += kLaneThreads) {  // warp-aggregated bucket cursors
      const int r = r0 + tid;
      const int bk = r < nrec ? (int)R.perm[r] : -1 - lane;  // distinct dummies for idle lanes
      const unsigned peers = __match_any_sync(HYD_FULL, bk);
      const int leader = __ffs(peers) - 1;
      int pos = 0;
      if (lane == leader && bk >= 0) pos = atomicAdd(&s_hist[bk], __popc(peers));
      pos = __shfl_sync(HYD_FULL, pos, leader) + __popc(peers & ((1u << lane) - 1u));
      HYD_CHECK(bk < 0 || (pos >= 0 && pos < nrec));
      if (bk >= 0) R.list2[pos] = (uint32_t)r;
    }
    __syncthreads();
    for (int q = tid; q < nrec; q += kLaneThreads) R.perm[q] = (uint16_t)R.list2[q];
  }
  if (STAGED && a.off) {  // ragged rows need not be 16-byte aligned
    for (int e = tid; e < B; e += kLaneThreads) sm[e] = __ldg(a.sorted_len + tbase + e);
    for (int e = tid; e < B * kp; e += kLaneThreads) sm[B + e] = __ldg(a.cost + tbase * kp + e);
  } else if (STAGED) {
    const uint4* gl = reinterpret_cast<const uint4*>(a.sorted_len + tbase);
    uint4* s4 = reinterpret_cast<uint4*>(sm);
    for (int e = tid; e < B / 4; e += kLaneThreads) s4[e] = __ldg(gl + e);
    const uint4* gc = reinterpret_cast<const uint4*>(a.cost + tbase * kp);
    uint4* c4 = reinterpret_cast<uint4*>(sm + B);
    for (int e = tid; e < B * kp / 4; e += kLaneThreads) c4[e] = __ldg(gc + e);
  }
  __syncthreads();
  const uint32_t* slen = STAGED ? sm : a.sorted_len + tbase;
  const uint32_t* cst = STAGED ? sm + B : a.cost + tbase * kp;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);
  // alpha_k = min tau_ik / l_i over the iteration's sequences with l_i <= MaxLen_k (warp per scheme)
  for (int k = tid >> 5; k < a.n_schemes; k += kLaneThreads / 32) {
    const uint32_t ml = s_ml[k];
    uint32_t tn = 1u, td = 0u;  // running minimum tn / td (td = 0: none yet, +infinity)
    for (int i = lane; i < B; i += 32) {
      const uint32_t l = slen[i];
      if (l > ml) continue;
      const uint32_t tau = cst[(size_t)i * kp + k];
      if (td == 0u || (uint64_t)tau * td < (uint64_t)tn * l) {
        tn = tau;
        td = l;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint32_t on = __shfl_xor_sync(HYD_FULL, tn, o), od = __shfl_xor_sync(HYD_FULL, td, o);
      if (od != 0u && (td == 0u || (uint64_t)on * td < (uint64_t)tn * od)) {
        tn = on;
        td = od;
      }
    }
    if (lane == 0) {
      const uint64_t cap = td ? (uint64_t)tn * ml / td : 0xFFFFFFFFull;
      s_cap[k] = cap > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)cap;
    }
  }
  __syncthreads();

  LaneUnit<VM> u;
  uint32_t ev = 0;
  auto load_unit = [&](int r, uint32_t V, uint32_t thr, bool write, bool F) {
    const int e = (int)R.eid[r];
    const int c = c0 + e / mnp;
    u.e = r;
    u.k = R.k[r];
    u.M = s_ml[u.k];
    u.mw = a.members + (fbase + e - e % mnp) * nwords + e % mnp;  // word-major rows of (t, c)
    u.mrow = a.mb + (size_t)c * a.n_total + tbase;
    u.write = write;
    u.F = F;
    u.tb = sbase + ((uint32_t)B + u.k) * 4u;
#ifdef HYD_DEBUG_CHECKS
    u.bt = (uint32_t)B;
    HYD_CHECK(r >= 0 && r < ncap && u.k < (uint32_t)kp);
#endif
    unit_start<VM>(u, V, thr);
  };
  // Lanes pull consecutive units of a list sorted by (class, U) -- so the units a warp holds at
  // any time have the same class and similar U -- and refill as soon as their unit ends.
  // Between epochs of kLaneEpoch sequences, all lanes whose unit ended record it and pull the
  // next one together (converged); the VMAX code path is chosen per epoch for the whole warp.
  auto run_units = [&](auto allow_free, auto phase, int n_units, auto&& pull, auto&& finish) {
    constexpr bool AF = decltype(allow_free)::value;
    constexpr int WR = decltype(phase)::value;
    if (tid == 0) s_next = 0;
    __syncthreads();
    bool have = false, done = false;
    while (true) {
      while (!have && !done) {
        const int q = atomicAdd(&s_next, 1);
        if (q >= n_units) done = true;
        else have = pull(q);
      }
      if (__all_sync(HYD_FULL, !have)) break;
      // bins the warp's widest unit needs: VMAX 16 paths 8 / 16, VMAX 32 paths 24 / 32
      constexpr int N0 = VM == 16 ? 8 : 24;
      const bool narrow = __all_sync(HYD_FULL, !have || u.V <= (uint32_t)N0);
      const bool fr = AF && __all_sync(HYD_FULL, !have || u.F);
      if (have) {
        // one epoch on the chosen path (the path is fixed for the epoch: one loop per path)
        auto epoch = [&](auto n_c, auto f_c) -> int {
          constexpr int NN = decltype(n_c)::value;
          constexpr bool FF = decltype(f_c)::value;
          int st = 0;
#pragma unroll 1
          for (int e = 0; e < kLaneEpoch && st == 0; ++e)
            st = unit_step<NN, VM, STAGED, FF, WR>(u, nwords_t, mnp, sbase, slen, cst, kp, a.kp4, ev);
          return st;
        };
        int st;
        if constexpr (AF) {
          if (fr)
            st = narrow ? epoch(std::integral_constant<int, N0>{}, std::true_type{})
                        : epoch(std::integral_constant<int, VM>{}, std::true_type{});
          else
            st = narrow ? epoch(std::integral_constant<int, N0>{}, std::false_type{})
                        : epoch(std::integral_constant<int, VM>{}, std::false_type{});
        } else {
          st = narrow ? epoch(std::integral_constant<int, N0>{}, std::false_type{})
                      : epoch(std::integral_constant<int, VM>{}, std::false_type{});
        }
        if (st) have = finish(st);  // finish may load a follow-up unit into this lane
      }
    }
    __syncthreads();
  };
  auto obj_key = [&](const LaneUnit<VM>& w) {
    return (((uint64_t)w.mx * (uint64_t)(s_pp[w.k] - 1 + w.V)) << 16) | w.V;
  };
  phase_clock(0);
  // ---- phase 1: the V_a run of every task (writes mb); where LPT(V_a) is infeasible
  //      (capacity), the same lane goes on with V_a + 1, V_a + 2, ... (up to min(V_hi, VM)); the
  //      first feasible one takes V_a's place as the reference run of the exact tests below (any
  //      completed run is a valid reference: the walk re-examines every other V of the range)
  run_units(
      std::false_type{}, std::integral_constant<int, 1>{}, nrec,
      [&](int q) {
        const int r = R.perm[q];
        load_unit(r, R.va[r], 0xFFFFFFFFu, true, false);
        return true;
      },
      [&](int st) -> bool {
        const int r = u.e;
        if (st == 1) {
          R.key[r] = obj_key(u);
          return false;
        }
        R.key[r] = kBottom;
        const uint32_t V = u.V + 1u;
        if (V > (uint32_t)R.vhi[r] || V > (uint32_t)VM) return false;
        R.va[r] = (uint16_t)V;
        load_unit(r, V, 0xFFFFFFFFu, true, false);
        return true;  // keep the lane on this task
      });
  phase_clock(1);
  phase_clock(2);
  // ---- phase 1.5 (thread per task): every V of App. D's range that survives the exact tests
  //      against the reference run, bucket-sorted by (class, U) into list2; tasks that do not
  //      fit are handed off
  auto walk = [&](int r, Search& s) {
    s.P = s_pp[R.k[r]];
    s.U = R.u[r];
    s.sumT = R.sum_t[r];
    s.tau_max = R.tau_max[r];
    s.vlo = R.vlo[r];
    s.vhi = R.vhi[r];
    s.va = R.va[r];
    s.cursor = s.vlo;
    s.phase = 1;
    s.have = false;
    // reference run: best = its objective (search_take's bookkeeping without the division)
    s.best = R.key[r] >> 16;
    s.vbest = s.va;
    s.have = true;
    if (s.P > 1) {
      if (s.best <= s.sumT) {
        s.cursor = s.vhi + 1;
      } else {
        const float est = (float)s.sumT * (float)(s.P - 1) / (float)(s.best - s.sumT);
        const float lo = est - 2.0f;
        if (lo > (float)s.cursor) s.cursor = lo >= (float)s.vhi ? s.vhi + 1 : (uint32_t)lo;
      }
    }
  };
  // thr of a phase-2 unit against best (the run's abort threshold, search_thr_approx clamped)
  auto unit_thr = [&](int r, uint32_t V, uint64_t best) -> uint32_t {
    Search s;
    s.P = s_pp[R.k[r]];
    s.have = true;
    s.best = best;
    const uint64_t th = search_thr_approx(s, V);
    return th > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)th;
  };
  // pass A (thread per task): candidate counts (class <= 8 / > 8), bucket and mode of every task
  // (mode: every candidate's run is capacity-free against the reference, bit 5 of cbucket)
  if (tid == 0) s_n2a = 0;
  __syncthreads();
  for (int r = tid; r < nrec; r += kLaneThreads) {
    R.ncand[r] = 0;
    if (R.key[r] == kBottom) {  // the sequential search (with extension) runs elsewhere
      atomicAdd(a.why + (VM == 16 ? 2 : 5), 1ull);
      const int e = (int)R.eid[r];
      to_queue(c0 + e / mnp, e % mnp);
      R.state[r] = 1;
      continue;
    }
    Search s;
    walk(r, s);
    int n_lo = 0, n_hi = 0;  // candidates with V <= 8 / V > 8 (VM = 32: all counted high)
    uint32_t vmax = 0, V, vmask = 0;
    bool all_free = true;
    const uint32_t cap = s_cap[R.k[r]];
    while ((V = search_next(s)) != 0) {
      vmax = max(vmax, V);
      if (VM == 16 && V <= 8) ++n_lo;
      else ++n_hi;
      if (V <= 32u) vmask |= 1u << (V - 1u);
      all_free = all_free && unit_thr(r, V, R.key[r] >> 16) <= cap;
    }
    R.sum_t[r] = vmask;  // the candidates as a bit set over V (sum_t is not read after this walk)
    if (vmax > (uint32_t)VM) {
      atomicAdd(a.why + (VM == 16 ? 3 : 6), 1ull);
      hand_off_e((int)R.eid[r]);
      R.state[r] = 1;
      continue;
    }
    if (n_lo + n_hi == 0) continue;
    R.ncand[r] = (uint16_t)(n_lo | (n_hi << 8));
    R.cbucket[r] = (uint8_t)(min(31, (int)(R.u[r] >> 3)) | (all_free ? 32 : 0));
    atomicAdd(&s_n2a, n_lo + n_hi);
  }
  __syncthreads();
  phase_clock(3);
  const int total2 = s_n2a;
  if (VM == 16 && tid == 0) atomicAdd(a.why + 14, (unsigned long long)total2);
  // bucket of a unit: (class, mode, U) -- capacity-free units apart from masked ones, so warps
  // pulling consecutive units mostly run one path
  auto bucket_of = [&](bool hi, int cb) { return (hi ? 64 : 0) + ((cb & 32) ? 0 : 32) + (cb & 31); };
  auto scan_hist = [&]() {  // exclusive scan, descending buckets; s_n2b = total
    __syncthreads();
    if (tid == 0) {
      int run = 0;
      for (int b = NB - 1; b >= 0; --b) {
        const int h = s_hist[b];
        s_hist[b] = run;
        run += h;
      }
      s_n2b = run;
    }
    __syncthreads();
  };
  // ---- phase 2 in rounds of whole tasks whose units fit list2 (one round unless the tile
  //      has more than ncap surviving V): the surviving V, each an independent run against
  //      the best so far; argmin by atomicMin on (obj << 16 | V)
  for (int r0 = 0; r0 < nrec;) {
    __syncthreads();
    if (tid < 32) {  // round end r1: longest task range from r0 whose units fit ncap
      int r1 = nrec;
      if (total2 > ncap) {
        int acc = 0;
        r1 = r0;
        for (int q0 = r0; q0 < nrec; q0 += 32) {
          const int q = q0 + lane;
          const int packed = q < nrec ? (int)R.ncand[q] : 0;
          int x = (q < nrec && R.state[q] != 1) ? (packed & 0xFF) + (packed >> 8) : 0;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {  // inclusive warp scan
            const int y = __shfl_up_sync(HYD_FULL, x, o);
            if (lane >= o) x += y;
          }
          const unsigned fit = __ballot_sync(HYD_FULL, q < nrec && acc + x <= ncap);
          const int nfit = __popc(fit);  // prefix property: the fitting lanes are 0..nfit-1
          r1 = q0 + nfit;
          if (nfit < 32) break;
          acc += __shfl_sync(HYD_FULL, x, 31);
        }
        if (r1 == r0) r1 = r0 + 1;  // cannot happen (a task has <= VM <= ncap units)
      }
      if (lane == 0) s_n2b = r1;
    }
    for (int b = tid; b < NB; b += kLaneThreads) s_hist[b] = 0;
    __syncthreads();
    const int r1 = s_n2b;
    for (int r = r0 + tid; r < r1; r += kLaneThreads) {
      const int packed = R.ncand[r];
      if (packed == 0 || R.state[r] == 1) continue;
      const int cb = R.cbucket[r];
      if (packed & 0xFF) atomicAdd(&s_hist[bucket_of(false, cb)], packed & 0xFF);
      if (packed >> 8) atomicAdd(&s_hist[bucket_of(true, cb)], packed >> 8);
    }
    scan_hist();
    // pass B: bucket-sorted units of the round (slot << 16 | V)
    for (int r = r0 + tid; r < r1; r += kLaneThreads) {
      const int packed = R.ncand[r];
      if (packed == 0 || R.state[r] == 1) continue;
      const int n_lo = packed & 0xFF, n_hi = packed >> 8;
      const int cb = R.cbucket[r];
      const int p_lo = n_lo ? atomicAdd(&s_hist[bucket_of(false, cb)], n_lo) : 0;
      const int p_hi = n_hi ? atomicAdd(&s_hist[bucket_of(true, cb)], n_hi) : 0;
      int i_lo = 0, i_hi = 0;
      for (uint32_t m = R.sum_t[r]; m != 0u; m &= m - 1u) {  // pass A's candidates
        const uint32_t V = (uint32_t)__ffs(m);
        const uint32_t w = ((uint32_t)r << 16) | V;
        if (VM == 16 && V <= 8) {
          HYD_CHECK(i_lo >= n_lo || p_lo + i_lo < ncap);
          if (i_lo < n_lo) R.list2[p_lo + i_lo++] = w;
        } else {
          HYD_CHECK(i_hi >= n_hi || p_hi + i_hi < ncap);
          if (i_hi < n_hi) R.list2[p_hi + i_hi++] = w;
        }
      }
    }
    __syncthreads();
    run_units(
        std::true_type{}, std::integral_constant<int, 2>{}, s_n2b,
        [&](int q) {
          HYD_CHECK(q < ncap);
          const uint32_t w = R.list2[q];
          const int r = (int)(w >> 16);
          HYD_CHECK(r < nrec);
          const uint32_t V = w & 0xFFFFu;
          const uint32_t thr = unit_thr(r, V, R.key[r] >> 16);
          load_unit(r, V, thr, false, thr <= s_cap[R.k[r]]);
          return true;
        },
        [&](int st) -> bool {
          if (st == 1) atomicMin(&R.key[u.e], obj_key(u));
          return false;
        });
    r0 = r1;
  }
  // ---- phase 3: the mb row of every task whose winner is not its reference run (whose mb phase
  //      1 wrote): one more run of the winning V, capacity-free when its known maximum bin time
  //      is within cap_k
  for (int b = tid; b < NB; b += kLaneThreads) s_hist[b] = 0;
  __syncthreads();
  auto rewrite_of = [&](int r, uint32_t& V, bool& F) -> bool {
    if (R.state[r] == 1 || R.ncand[r] == 0) return false;
    const unsigned long long key = R.key[r];
    V = (uint32_t)(key & 0xFFFFu);
    if (V == (uint32_t)R.va[r]) return false;
    const uint64_t mx = (key >> 16) / (uint64_t)(s_pp[R.k[r]] - 1u + V);
    F = mx <= (uint64_t)s_cap[R.k[r]];
    return true;
  };
  for (int r = tid; r < nrec; r += kLaneThreads) {
    uint32_t V;
    bool F;
    if (rewrite_of(r, V, F))
      atomicAdd(&s_hist[bucket_of(VM == 32 || V > 8, min(31, (int)(R.u[r] >> 3)) | (F ? 32 : 0))], 1);
  }
  scan_hist();
  for (int r = tid; r < nrec; r += kLaneThreads) {
    uint32_t V;
    bool F;
    if (rewrite_of(r, V, F)) {
      const int pos = atomicAdd(&s_hist[bucket_of(VM == 32 || V > 8, min(31, (int)(R.u[r] >> 3)) | (F ? 32 : 0))], 1);
      R.list2[pos] = ((uint32_t)r << 16) | V | (F ? 0x8000u : 0u);
    }
  }
  __syncthreads();
  run_units(
      std::true_type{}, std::integral_constant<int, 3>{}, s_n2b,
      [&](int q) {
        const uint32_t w = R.list2[q];
        load_unit((int)(w >> 16), w & 0x7FFFu, 0xFFFFFFFFu, true, (w & 0x8000u) != 0u);
        return true;
      },
      [&](int) -> bool { return false; });

  phase_clock(4);
  phase_clock(5);
  if (VM == 16 && tid == 0) atomicAdd(a.why + 15, (unsigned long long)nrec);
  // ---- outputs
  if constexpr (VM == 16) {
    write_rows(nrec);
  } else {
    for (int r = tid; r < nrec; r += kLaneThreads) {  // VMAX-32 pass: its tasks' slots only
      if (R.state[r] == 1) continue;
      const int e = (int)R.eid[r];
      const int c = c0 + e / mnp, j = e % mnp;
      const size_t row = (size_t)c * a.n_iter + t;
      const unsigned long long key = R.key[r];
      a.v[row * HYD_MAX_PIPES + j] = (uint16_t)(key & 0xFFFFu);
      a.ptime[row * HYD_MAX_PIPES + j] = key >> 16;
      atomicMax(reinterpret_cast<unsigned long long*>(a.makespan + (size_t)t * a.n_cand + c), key >> 16);
    }
  }
  if (ev) atomicAdd(a.evals, (unsigned long long)ev);
}

// The tasks the VMAX-16 pass flagged, per iteration, as a compacted list in ascending task id
// (c * mnp + j): one CTA per iteration, block-wide scan of per-thread counts of 32-task groups.
__global__ void __launch_bounds__(256) k_flag_list(const uint32_t* __restrict__ flags, int n_cand, int mnp,
                                                   uint32_t* __restrict__ list32, uint32_t* __restrict__ count32,
                                                   unsigned long long* __restrict__ total) {
  __shared__ int s_w[8];
  __shared__ int s_base;
  const int t = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t n = (size_t)n_cand * mnp, bit0 = (size_t)t * n;
  uint32_t* out = list32 + (size_t)t * n;
  if (tid == 0) s_base = 0;
  __syncthreads();
  for (size_t g0 = 0; g0 < n; g0 += 256 * 32) {
    const size_t e0 = g0 + (size_t)tid * 32;  // this thread's 32 tasks
    uint32_t bits = 0u;
    if (e0 < n) {
      const size_t b = bit0 + e0, w = b >> 5, sh = b & 31;
      const size_t last = bit0 + min(n, e0 + 32) - 1;  // the group's last task bit
      bits = flags[w] >> sh;
      if (sh && (last >> 5) > w) bits |= flags[w + 1] << (32 - sh);
      if (n - e0 < 32) bits &= (1u << (n - e0)) - 1u;
    }
    int x = __popc(bits);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(HYD_FULL, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    int wbase = s_base;
    for (int q = 0; q < warp; ++q) wbase += s_w[q];
    int pos = wbase + x - __popc(bits);
    for (uint32_t m = bits; m; m &= m - 1u) out[pos++] = (uint32_t)(e0 + __ffs(m) - 1);
    __syncthreads();
    if (tid == 255) s_base = wbase + x;
    __syncthreads();
  }
  if (tid == 0) {
    count32[t] = (uint32_t)s_base;
    if (s_base) atomicAdd(total, (unsigned long long)s_base);
  }
}

// ------------------------------------------------------------------ LPT, one warp per pipeline
template <typename TT>
__device__ __forceinline__ TT warp_min(TT x);
template <>
__device__ __forceinline__ uint32_t warp_min<uint32_t>(uint32_t x) {
  return __reduce_min_sync(HYD_FULL, x);
}
template <>
__device__ __forceinline__ uint64_t warp_min<uint64_t>(uint64_t x) {
  const uint32_t hi = __reduce_min_sync(HYD_FULL, (uint32_t)(x >> 32));
  const uint32_t lo = __reduce_min_sync(HYD_FULL, (uint32_t)(x >> 32) == hi ? (uint32_t)x : 0xFFFFFFFFu);
  return ((uint64_t)hi << 32) | lo;
}

// bins b = lane + 32 r; R register slots per lane (R*32 >= V), or scratch when R == 0
// Warp-cooperative member stream of one pipeline: the membership bitmap is decoded 32
// members at a time (word popcounts, warp prefix scan, per-lane rank search), each lane
// gathering its member's (l, tau) so the sequential LPT loop reads them by shuffle.
struct MemberStream {
  const uint32_t* mw;     // word w at mw[w * stride]
  uint32_t nwords, stride, wpos;  // wpos: next word window start
  uint32_t wbits;         // this lane's word of the current window (already consumed bits cleared)
  uint32_t incl;          // inclusive prefix of remaining popcounts in the window
  uint32_t left;          // members left in the window
};

__device__ __forceinline__ void ms_open(MemberStream& m, const uint32_t* mw, uint32_t nwords,
                                        uint32_t stride) {
  m.mw = mw;
  m.nwords = nwords;
  m.stride = stride;
  m.wpos = 0;
  m.left = 0;
  m.wbits = 0;
  m.incl = 0;
}

// Fill (idx, l, tau) for up to 32 next members; returns how many (0 at the end).
__device__ __forceinline__ uint32_t ms_next32(MemberStream& m, const uint32_t* __restrict__ sl,
                                              const uint32_t* __restrict__ cs, int kp, uint32_t k,
                                              uint32_t& idx, uint32_t& l, uint32_t& tau) {
  const int lane = threadIdx.x & 31;
  while (m.left == 0) {
    if (m.wpos >= m.nwords) return 0;
    const uint32_t w = m.wpos + lane;
    m.wbits = w < m.nwords ? __ldg(m.mw + (size_t)w * m.stride) : 0u;
    uint32_t c = __popc(m.wbits);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(HYD_FULL, c, o);
      if (lane >= o) c += y;
    }
    m.incl = c;
    m.left = __shfl_sync(HYD_FULL, c, 31);
    m.wpos += 32;
  }
  const uint32_t n = min(m.left, 32u);
  // lane r takes the r-th remaining member: the word w with incl[w-1] <= r < incl[w]
  const uint32_t r = (uint32_t)lane;
  uint32_t lo = 0;
#pragma unroll
  for (int step = 16; step > 0; step >>= 1) {
    const uint32_t probe = __shfl_sync(HYD_FULL, m.incl, lo + step - 1);
    if (probe <= r) lo += step;
  }
  // lo = word index holding rank r (valid when r < n)
  const uint32_t before_raw = __shfl_sync(HYD_FULL, m.incl, lo ? lo - 1 : 0);  // all lanes shuffle
  const uint32_t before = lo ? before_raw : 0u;
  const uint32_t bits = __shfl_sync(HYD_FULL, m.wbits, lo & 31u);
  if (r < n) {
    const uint32_t bit = __fns(bits, 0, (int)(r - before) + 1);
    idx = (m.wpos - 32u + lo) * 32u + bit;
    l = __ldg(sl + idx);
    tau = __ldg(cs + (size_t)idx * kp + k);
  }
  // consume n members: clear the n lowest set bits across the window
  const uint32_t up = __shfl_up_sync(HYD_FULL, m.incl, 1);  // all lanes shuffle
  const uint32_t mine_before = lane ? up : 0u;
  const uint32_t take0 = n > mine_before ? n - mine_before : 0u;
  uint32_t take = min(take0, (uint32_t)__popc(m.wbits));
  while (take--) m.wbits &= m.wbits - 1u;
  m.incl = m.incl > n ? m.incl - n : 0u;
  m.left -= n;
  return n;
}

// LPT(V) over the member stream, bins b = lane + 32 r (R register slots, or scratch when R == 0).
// Writes mb when `write`; returns false if infeasible or the running max exceeds thr.
template <int R, typename TT>
__device__ __forceinline__ bool lpt_warp(const uint32_t* __restrict__ mw, uint32_t nwords,
                                         uint32_t mstride, uint32_t V, uint32_t M, const uint32_t* __restrict__ sl,
                                         const uint32_t* __restrict__ cs, int kp, uint32_t k,
                                         uint64_t thr64, bool write, uint16_t* __restrict__ mrow,
                                         uint64_t& maxbin, uint64_t* scr_t, uint32_t* scr_k,
                                         uint64_t& evals) {
  const int lane = threadIdx.x & 31;
  const TT thr = thr64 > (uint64_t)(TT)(~TT(0)) ? (TT)(~TT(0)) : (TT)thr64;
  constexpr int RR = R > 0 ? R : 1;
  TT tm[RR];
  uint32_t tk[RR];
  const uint32_t rn = (V + 31) >> 5;  // slots in use (generic path)
  if (R > 0) {
#pragma unroll
    for (int r = 0; r < RR; ++r) {
      tm[r] = 0;
      tk[r] = (uint32_t)(lane + 32 * r) < V ? 0u : 0xFFFFFFFFu;
    }
  } else {
    for (uint32_t r = 0; r < rn; ++r) {
      scr_t[32 * r + lane] = 0ull;
      scr_k[32 * r + lane] = (32 * r + lane) < V ? 0u : 0xFFFFFFFFu;
    }
  }
  MemberStream ms;
  ms_open(ms, mw, nwords, mstride);
  TT mx = 0;
  uint32_t cidx = 0, cl = 0, ctau = 0, n;
  while ((n = ms_next32(ms, sl, cs, kp, k, cidx, cl, ctau)) != 0) {
    for (uint32_t q = 0; q < n; ++q) {
      const uint32_t l = __shfl_sync(HYD_FULL, cl, q);
      const TT tau = (TT)__shfl_sync(HYD_FULL, ctau, q);
      const uint32_t iq = __shfl_sync(HYD_FULL, cidx, q);
      const uint32_t cap = M - l;
      TT lt = ~TT(0);
      uint32_t lr = 0xFFFFu;
      if (R > 0) {
#pragma unroll
        for (int r = 0; r < RR; ++r)
          if (tk[r] <= cap && tm[r] < lt) {
            lt = tm[r];
            lr = (uint32_t)r;
          }
      } else {
        for (uint32_t r = 0; r < rn; ++r) {
          const uint32_t tkr = scr_k[32 * r + lane];
          const TT tmr = (TT)scr_t[32 * r + lane];
          if (tkr <= cap && tmr < lt) {
            lt = tmr;
            lr = r;
          }
        }
      }
      const TT m = warp_min<TT>(lt);
      evals += V;
      if (m == ~TT(0)) return false;  // no bin fits: LPT(V) = bottom (warp-uniform)
      const uint32_t bstar = __reduce_min_sync(HYD_FULL, lt == m ? (uint32_t)lane + 32u * lr : 0xFFFFFFFFu);
      if ((bstar & 31u) == (uint32_t)lane) {
        const uint32_t rs = bstar >> 5;
        if (R > 0) {
#pragma unroll
          for (int r = 0; r < RR; ++r) {  // branch-free (a switch compiles to a jump table)
            const bool h = (uint32_t)r == rs;
            tm[r] += h ? tau : (TT)0;
            tk[r] += h ? l : 0u;
          }
        } else {
          HYD_CHECK(bstar < V);
          scr_t[bstar] += (uint64_t)tau;
          scr_k[bstar] += l;
        }
        if (write) mrow[iq] = (uint16_t)bstar;
      }
      const TT nt = m + tau;
      mx = nt > mx ? nt : mx;
      if (mx > thr) return false;
    }
  }
  maxbin = (uint64_t)mx;
  return true;
}

// LPT(V <= 32) with packed keys, lane b = bin b: key = time << 5 | b (sumT < 2^26), a sign-bit
// capacity mask as in the lanes, so one redux.sync min per sequence picks the least-time fitting
// bin with the smallest index (same rule and result as lpt_warp).
__device__ __forceinline__ bool lpt_warp_packed(const uint32_t* __restrict__ mw, uint32_t nwords,
                                                uint32_t mstride, uint32_t V, uint32_t M,
                                                const uint32_t* __restrict__ sl,
                                                const uint32_t* __restrict__ cs, int kp, uint32_t k,
                                                uint64_t thr64, bool write, uint16_t* __restrict__ mrow,
                                                uint64_t& maxbin, uint64_t& evals) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t thr = thr64 > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)thr64;
  uint32_t key = lane < V ? lane : 0xFFFFFFFFu;  // unused lanes never fit
  uint32_t rem = M;                               // MaxLen - tokens of bin `lane`
  uint32_t mx = 0;
  MemberStream ms;
  ms_open(ms, mw, nwords, mstride);
  uint32_t cidx = 0, cl = 0, ctau = 0, n;
  while ((n = ms_next32(ms, sl, cs, kp, k, cidx, cl, ctau)) != 0) {
    for (uint32_t q = 0; q < n; ++q) {
      const uint32_t l = __shfl_sync(HYD_FULL, cl, q);
      const uint32_t tau = __shfl_sync(HYD_FULL, ctau, q);
      const uint32_t iq = __shfl_sync(HYD_FULL, cidx, q);
      const uint32_t d = rem - l;
      const uint32_t mk = key | (d & 0x80000000u);
      const uint32_t m = __reduce_min_sync(HYD_FULL, mk);
      evals += V;
      if (m >> 31) return false;  // no bin fits
      if (mk == m) {
        key += tau << 5;
        rem = d;
        if (write) mrow[iq] = (uint16_t)lane;
      }
      mx = max(mx, (m >> 5) + tau);
      if (mx > thr) return false;
    }
  }
  maxbin = mx;
  return true;
}

// LPT(V <= 32 R) with packed keys over R bins per lane (b = lane + 32 r): key = time << S | b,
// S = 5 + log2 R, bins that cannot take the sequence masked to 0xFFFFFFFF by a select (so keys
// use all 32 bits: sum T < 2^(32 - S) - 1); per sequence one lane-local min, ONE redux.sync and a
// compare-and-add per bin -- the same rule and result as lpt_warp (least-time fitting bin,
// smallest index), with one warp reduction in the dependent chain instead of two.
template <int R>
__device__ __forceinline__ bool lpt_warp_packed_r(const uint32_t* __restrict__ mw, uint32_t nwords, uint32_t mstride,
                                                  uint32_t V, uint32_t M, const uint32_t* __restrict__ sl,
                                                  const uint32_t* __restrict__ cs, int kp, uint32_t k, uint64_t thr64,
                                                  bool write, uint16_t* __restrict__ mrow, uint64_t& maxbin,
                                                  uint64_t& evals) {
  constexpr int S = R == 1 ? 5 : R == 2 ? 6 : 7;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t thr = thr64 > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)thr64;
  uint32_t key[R], rem[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const uint32_t b = lane + 32u * r;
    key[r] = b < V ? b : 0xFFFFFFFFu;  // unused bins are always masked
    rem[r] = M;                        // MaxLen - tokens of bin b
  }
  uint32_t mx = 0;
  MemberStream ms;
  ms_open(ms, mw, nwords, mstride);
  uint32_t cidx = 0, cl = 0, ctau = 0, n;
  while ((n = ms_next32(ms, sl, cs, kp, k, cidx, cl, ctau)) != 0) {
    for (uint32_t q = 0; q < n; ++q) {
      const uint32_t l = __shfl_sync(HYD_FULL, cl, q);
      const uint32_t tau = __shfl_sync(HYD_FULL, ctau, q);
      const uint32_t iq = __shfl_sync(HYD_FULL, cidx, q);
      uint32_t mk = 0xFFFFFFFFu;
#pragma unroll
      for (int r = 0; r < R; ++r) mk = min(mk, rem[r] >= l ? key[r] : 0xFFFFFFFFu);
      const uint32_t m = __reduce_min_sync(HYD_FULL, mk);
      evals += V;
      if (m == 0xFFFFFFFFu) return false;  // no bin fits
      const uint32_t add = tau << S;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const bool h = key[r] == m;
        key[r] = h ? key[r] + add : key[r];
        rem[r] = h ? rem[r] - l : rem[r];
      }
      if (write && (m & 31u) == lane) mrow[iq] = (uint16_t)(m & ((1u << S) - 1u));
      mx = max(mx, (m >> S) + tau);
      if (mx > thr) return false;
    }
  }
  maxbin = mx;
  return true;
}

template <typename TT>
__device__ __forceinline__ bool lpt_warp_dispatch(const uint32_t* mw, uint32_t nwords, uint32_t mstride, uint32_t V,
                                                  uint32_t M, const uint32_t* sl, const uint32_t* cs,
                                                  int kp, uint32_t k, uint64_t thr, bool write,
                                                  uint16_t* mrow, uint64_t& maxbin, uint64_t* st,
                                                  uint32_t* sk, uint64_t& ev) {
  if (V <= 32) return lpt_warp<1, TT>(mw, nwords, mstride, V, M, sl, cs, kp, k, thr, write, mrow, maxbin, st, sk, ev);
  if (V <= 64) return lpt_warp<2, TT>(mw, nwords, mstride, V, M, sl, cs, kp, k, thr, write, mrow, maxbin, st, sk, ev);
  if (V <= 128) return lpt_warp<4, TT>(mw, nwords, mstride, V, M, sl, cs, kp, k, thr, write, mrow, maxbin, st, sk, ev);
  if (V <= 32 * kBigRMax) return lpt_warp<kBigRMax, TT>(mw, nwords, mstride, V, M, sl, cs, kp, k, thr, write, mrow, maxbin, st, sk, ev);
  return lpt_warp<0, TT>(mw, nwords, mstride, V, M, sl, cs, kp, k, thr, write, mrow, maxbin, st, sk, ev);
}

// One queued task's geometry and search inputs (k_pack_big and its split phases).
struct BigTask {
  int c, t, j;
  size_t row, srow, tbase;
  uint32_t nwords_t, k;
  const uint32_t *sl, *cs, *mw;
  uint16_t* mrow;
  Search s;
  bool narrow, packed, packed2, packed4;
};

__device__ __forceinline__ void big_task(const PackArgs& a, unsigned long long e, BigTask& b) {
  b.c = (int)(e >> 37);
  b.t = (int)((e >> 5) & 0xFFFFFFFFull);
  b.j = (int)(e & 31);
  b.row = (size_t)b.c * a.n_iter + b.t;
  b.srow = ((size_t)b.t * a.n_cand + b.c) * a.mnp + b.j;
  b.tbase = geo_base(a.off, a.batch, b.t);
  b.nwords_t = (uint32_t)((geo_bt(a.off, a.batch, b.t) + 31) >> 5);
  b.sl = a.sorted_len + b.tbase;
  b.cs = a.cost + b.tbase * a.k_pad;
  b.mw = a.members + (b.srow - b.j) * a.nwords + b.j;  // word-major rows of (t, c)
  b.k = a.cand[(size_t)b.c * HYD_MAX_PIPES + b.j];
  const hyd_pipe_stats st = a.stats[b.srow];
  Search& s = b.s;
  s.M = a.schemes[b.k].max_len;
  s.P = a.schemes[b.k].pp;
  s.UL = a.schemes[b.k].util_len;
  s.U = st.u;
  s.S = st.s;
  s.sumT = st.sum_t;
  s.tau_max = st.tau_max;
  b.mrow = a.mb + (size_t)b.c * a.n_total + b.tbase;
  b.narrow = s.sumT < 0xFFFFFFFFull;
  b.packed = s.sumT < (1ull << 26) && s.M < 0x80000000u;  // lpt_warp_packed's keys
  // the select-masked packed keys of lpt_warp_packed_r: V <= 64 with sum T < 2^26 - 1, V <= 128
  // with sum T < 2^25 - 1
  b.packed2 = s.sumT < (1ull << 26) - 1ull;
  b.packed4 = s.sumT < (1ull << 25) - 1ull;
}

// LPT(V) of the task on the fastest warp path that holds it
__device__ __forceinline__ bool big_run(const PackArgs& a, const BigTask& b, uint32_t V, uint64_t thr, bool write,
                                        uint64_t& mx, uint64_t* scr_t, uint32_t* scr_k, uint64_t& ev) {
  const uint32_t mnp = (uint32_t)a.mnp, M = b.s.M;
  const int kp = a.k_pad;
  if (b.packed && V <= 32u)
    return lpt_warp_packed(b.mw, b.nwords_t, mnp, V, M, b.sl, b.cs, kp, b.k, thr, write, b.mrow, mx, ev);
  if (b.packed2 && V <= 64u)
    return lpt_warp_packed_r<2>(b.mw, b.nwords_t, mnp, V, M, b.sl, b.cs, kp, b.k, thr, write, b.mrow, mx, ev);
  if (b.packed4 && V <= 128u)
    return lpt_warp_packed_r<4>(b.mw, b.nwords_t, mnp, V, M, b.sl, b.cs, kp, b.k, thr, write, b.mrow, mx, ev);
  if (b.narrow)
    return lpt_warp_dispatch<uint32_t>(b.mw, b.nwords_t, mnp, V, M, b.sl, b.cs, kp, b.k, thr, write, b.mrow, mx,
                                       scr_t, scr_k, ev);
  return lpt_warp_dispatch<uint64_t>(b.mw, b.nwords_t, mnp, V, M, b.sl, b.cs, kp, b.k, thr, write, b.mrow, mx, scr_t,
                                     scr_k, ev);
}

__device__ __forceinline__ void big_outputs(const PackArgs& a, const BigTask& b, uint32_t vbest, uint64_t best) {
  if ((threadIdx.x & 31) == 0) {
    a.v[b.row * HYD_MAX_PIPES + b.j] = (uint16_t)vbest;
    a.ptime[b.row * HYD_MAX_PIPES + b.j] = best;
    atomicMax(reinterpret_cast<unsigned long long*>(a.makespan + (size_t)b.t * a.n_cand + b.c),
              (unsigned long long)best);
  }
}

// Persistent warps over the queue: one pipeline per warp, the sequential exact search
// (V_a, ascending scan with the exact pruning, extension above the range).  SPLIT (a short queue,
// k_pack_big_ref): only the reference run V_a and the enqueueing of the V that survive its exact
// tests (k_pack_big_units runs them, k_pack_big_finish re-runs the winners); a task whose V_a is
// infeasible, or whose units do not fit the unit queue, finishes sequentially here.  Both kernels
// are launched; each leaves the queue to the other unless its mode applies.
template <bool SPLIT>
__device__ __forceinline__ void big_queue(const PackArgs& a) {
  const int B = a.batch;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + warp;  // scratch slot
  uint64_t* scr_t = a.scr_time + (size_t)gw * B;
  uint32_t* scr_k = a.scr_tok + (size_t)gw * B;
  const unsigned long long total = min(*a.q_count, a.q_cap);
  if ((total <= (unsigned long long)kSplitTasks) != SPLIT) return;
  unsigned long long* ucount = a.q_count + 19;
  uint64_t ev = 0;
  while (true) {
    unsigned long long task = 0;
    if (lane == 0) task = atomicAdd(a.q_head, 1ull);
    task = __shfl_sync(HYD_FULL, task, 0);
    if (task >= total) break;
    BigTask b;
    big_task(a, a.queue[task], b);
    Search& s = b.s;
    if (!s.U) {
      if (SPLIT && lane == 0) a.sp_wv[task] = 0u;
      big_outputs(a, b, 0u, 0ull);
      continue;
    }
    search_init(s);
    uint32_t V, wV = 0;
    bool first = true;
    if constexpr (SPLIT) {  // the reference run, then the surviving V as units (if they fit)
      V = search_next(s);  // V_a
      uint64_t mx = 0;
      const bool ok = big_run(a, b, V, ~0ull, true, mx, scr_t, scr_k, ev);
      first = false;
      if (ok) {
        wV = V;
        search_take(s, V, mx);
        Search q = s;  // count the units the exact tests keep
        uint32_t n = 0;
        while (search_next(q) != 0) ++n;
        unsigned long long at = 0;
        if (lane == 0) at = n ? atomicAdd(ucount, (unsigned long long)n) : 0ull;
        at = __shfl_sync(HYD_FULL, at, 0);
        if (at + n <= (unsigned long long)kSplitUnits) {
          uint32_t q2 = 0, V2;
          while ((V2 = search_next(s)) != 0) {
            if (lane == 0) a.units[at + q2] = (task << 16) | V2;
            ++q2;
          }
          if (lane == 0) {
            a.sp_key[task] = (s.best << 16) | s.vbest;
            a.sp_wv[task] = wV;
          }
          continue;  // k_pack_big_units / k_pack_big_finish complete this task
        }
        // the unit queue is full: mark the reserved slots that exist as empty, finish this task
        // sequentially (below)
        if (lane == 0)
          for (unsigned long long q3 = at; q3 < at + n && q3 < (unsigned long long)kSplitUnits; ++q3)
            a.units[q3] = ~0ull;
      }
    }
    while ((V = search_next(s)) != 0) {
      const uint64_t thr = first ? ~0ull : search_thr_approx(s, V);
      uint64_t mx = 0;
      const bool ok = big_run(a, b, V, thr, first, mx, scr_t, scr_k, ev);
      if (ok && first) wV = V;
      first = false;
      if (ok && search_improves(s, V, mx)) search_take(s, V, mx);
    }
    if (s.have && s.vbest != wV) {  // the winner's mb was not written by the first run
      uint64_t mx = 0;
      big_run(a, b, s.vbest, ~0ull, true, mx, scr_t, scr_k, ev);
    }
    if (SPLIT && lane == 0) a.sp_wv[task] = 0u;  // done here
    big_outputs(a, b, s.vbest, s.best);
  }
  if (lane == 0 && ev) atomicAdd(a.evals, (unsigned long long)ev);
}

__global__ void __launch_bounds__(256, 3) k_pack_big(PackArgs a) { big_queue<false>(a); }
__global__ void __launch_bounds__(256) k_pack_big_ref(PackArgs a) { big_queue<true>(a); }

// Split queue, step 2: every enqueued (task, V) as an independent LPT(V) run against the task's
// best so far (abort threshold as in the lanes' phase 2); atomicMin of (obj << 16 | V).
__global__ void __launch_bounds__(256) k_pack_big_units(PackArgs a) {
  const unsigned long long total = min(*a.q_count, a.q_cap);
  if (total > (unsigned long long)kSplitTasks) return;
  const unsigned long long nunits = min(a.q_count[19], (unsigned long long)kSplitUnits);
  const int B = a.batch;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + warp;
  uint64_t* scr_t = a.scr_time + (size_t)gw * B;
  uint32_t* scr_k = a.scr_tok + (size_t)gw * B;
  uint64_t ev = 0;
  while (true) {
    unsigned long long u = 0;
    if (lane == 0) u = atomicAdd(a.q_count + 20, 1ull);
    u = __shfl_sync(HYD_FULL, u, 0);
    if (u >= nunits) break;
    const unsigned long long w = a.units[u];
    if (w == ~0ull) continue;  // a slot of a task that finished sequentially
    const unsigned long long task = w >> 16;
    const uint32_t V = (uint32_t)(w & 0xFFFFu);
    BigTask b;
    big_task(a, a.queue[task], b);
    Search& s = b.s;
    unsigned long long cur = 0;
    if (lane == 0) cur = *reinterpret_cast<volatile unsigned long long*>(a.sp_key + task);
    cur = __shfl_sync(HYD_FULL, cur, 0);
    s.have = true;
    s.best = cur >> 16;
    s.vbest = (uint32_t)(cur & 0xFFFFu);
    // exact LB test against the current best (the best can only have improved since enqueueing)
    const uint64_t m = (uint64_t)(s.P - 1 + V);
    uint64_t ah, al, bh, bl;
    mul128(s.sumT, m, ah, al);
    mul128(s.best, (uint64_t)V, bh, bl);
    if (gt128(ah, al, bh, bl) || (!gt128(bh, bl, ah, al) && V > s.vbest)) continue;
    uint64_t mx = 0;
    const bool ok = big_run(a, b, V, search_thr_approx(s, V), false, mx, scr_t, scr_k, ev);
    if (ok && lane == 0) atomicMin(a.sp_key + task, ((mx * m) << 16) | V);
  }
  if (lane == 0 && ev) atomicAdd(a.evals, (unsigned long long)ev);
}

// Split queue, step 3: per task, the winner's re-run when it is not the reference run (whose mb is
// written), and the v / ptime / makespan outputs.
__global__ void __launch_bounds__(256) k_pack_big_finish(PackArgs a) {
  const unsigned long long total = min(*a.q_count, a.q_cap);
  if (total > (unsigned long long)kSplitTasks) return;
  const int B = a.batch;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + warp;
  uint64_t* scr_t = a.scr_time + (size_t)gw * B;
  uint32_t* scr_k = a.scr_tok + (size_t)gw * B;
  uint64_t ev = 0;
  for (unsigned long long task = gw; task < total; task += (unsigned long long)gridDim.x * (blockDim.x >> 5)) {
    const uint32_t wv = a.sp_wv[task];
    if (wv == 0u) continue;  // finished in k_pack_big
    BigTask b;
    big_task(a, a.queue[task], b);
    const unsigned long long key = a.sp_key[task];
    const uint32_t vbest = (uint32_t)(key & 0xFFFFu);
    if (vbest != wv) {
      uint64_t mx = 0;
      big_run(a, b, vbest, ~0ull, true, mx, scr_t, scr_k, ev);
    }
    big_outputs(a, b, vbest, key >> 16);
  }
  if (lane == 0 && ev) atomicAdd(a.evals, (unsigned long long)ev);
}

// ------------------------------------------------------------------ host side
static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static int dp_of(int max_np) {
  return max_np <= 2 ? 2 : max_np <= 4 ? 4 : max_np <= 8 ? 8 : max_np <= 16 ? 16 : 32;
}

static size_t flag_bytes(int n_iter, int n_cand, int max_np) {
  return ((size_t)n_iter * n_cand * max_np + 31) / 32 * 4;
}

size_t pack_workspace(int n_iter, int batch, int n_cand, int max_np) {
  const size_t cap = (size_t)n_iter * n_cand * dp_of(max_np);
  return align256(256) + align256(cap * 8) + align256((size_t)kBigWarps * batch * 8) +
         align256((size_t)kBigWarps * batch * 4) + align256(flag_bytes(n_iter, n_cand, max_np)) +
         align256((size_t)n_iter * n_cand * max_np * 4) + align256((size_t)n_iter * 4) +
         align256((size_t)kSplitTasks * 8) + align256((size_t)kSplitTasks * 4) + align256((size_t)kSplitUnits * 8);
}

template <bool STAGED, int VM>
static cudaError_t launch_lanes(dim3 grid, size_t smem, cudaStream_t s, const PackArgs& a, int tc,
                                int mnp, int ncap) {
  cudaError_t e = cudaFuncSetAttribute(k_pack_lanes<STAGED, VM>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_pack_lanes<STAGED, VM><<<grid, kLaneThreads, smem, s>>>(a, tc, mnp, ncap);
  return cudaGetLastError();
}

int launch_pack(const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch,
                const uint32_t* off, size_t n_total, int k_pad,
                const hyd_scheme* schemes, int n_schemes, const uint8_t* cand,
                const uint8_t* cand_np, int n_cand, int max_np, const uint8_t* pipe,
                const hyd_pipe_stats* stats, const uint32_t* members, uint16_t* mb, uint16_t* v,
                uint64_t* ptime,
                uint64_t* makespan, uint32_t* status, void* ws, size_t ws_bytes, cudaStream_t s) {
  (void)ws_bytes;
  if (n_iter == 0 || n_cand == 0) return HYD_OK;
  const int dp = dp_of(max_np);
  PackArgs a;
  a.sorted_len = sorted_len;
  a.cost = cost;
  a.n_iter = n_iter;
  a.batch = batch;
  a.off = off;
  a.n_total = n_total;
  a.k_pad = k_pad;
  a.kp4 = 4u * (uint32_t)k_pad;
  a.schemes = schemes;
  a.n_schemes = n_schemes;
  a.cand = cand;
  a.cand_np = cand_np;
  a.n_cand = n_cand;
  a.pipe = pipe;
  a.stats = stats;
  a.members = members;
  a.mnp = max_np;
  a.nwords = (batch + 31) / 32;
  a.mb = mb;
  a.v = v;
  a.ptime = ptime;
  a.makespan = makespan;
  a.status = status;
  char* w = static_cast<char*>(ws);
  a.q_count = reinterpret_cast<unsigned long long*>(w);
  a.q_head = a.q_count + 1;
  a.evals = a.q_count + 2;
  a.why = a.q_count + 3;
  w += align256(256);
  a.q_cap = (unsigned long long)n_iter * n_cand * dp;
  a.queue = reinterpret_cast<unsigned long long*>(w);
  w += align256(a.q_cap * 8);
  a.scr_time = reinterpret_cast<uint64_t*>(w);
  w += align256((size_t)kBigWarps * batch * 8);
  a.scr_tok = reinterpret_cast<uint32_t*>(w);
  w += align256((size_t)kBigWarps * batch * 4);
  a.flags = reinterpret_cast<uint32_t*>(w);
  w += align256(flag_bytes(n_iter, n_cand, max_np));
  a.list32 = reinterpret_cast<uint32_t*>(w);
  w += align256((size_t)n_iter * n_cand * max_np * 4);
  a.count32 = reinterpret_cast<uint32_t*>(w);
  w += align256((size_t)n_iter * 4);
  a.sp_key = reinterpret_cast<unsigned long long*>(w);
  w += align256((size_t)kSplitTasks * 8);
  a.sp_wv = reinterpret_cast<uint32_t*>(w);
  w += align256((size_t)kSplitTasks * 4);
  a.units = reinterpret_cast<unsigned long long*>(w);

  cudaError_t e = cudaMemsetAsync(a.q_count, 0, 256, s);
  if (e != cudaSuccess) return record_cuda_error(e);
  e = cudaMemsetAsync(a.flags, 0, flag_bytes(n_iter, n_cand, max_np), s);
  if (e != cudaSuccess) return record_cuda_error(e);
  // (v / ptime / makespan rows and infeasible mb rows are written whole by the VMAX-16 pass)

  // persistent lanes: pass 1 (VMAX 16) CTA = one iteration x tc candidates (~2048 tasks);
  // pass 2 (VMAX 32, flagged tasks, compacted records) CTA = one iteration x up to 2048 candidates
  // two CTAs per SM: ~110 KB of dynamic smem each for the staged iteration + task records
  const size_t stage = ((size_t)batch * 4 * (1 + (size_t)k_pad) + 15) & ~(size_t)15;
  auto plan = [&](size_t budget, bool& staged, int& ncap, size_t& smem) {
    staged = (off || (batch % 4) == 0) && stage + 512 * 39 <= budget;
    ncap = (int)(((staged ? budget - stage : budget) / 39) & ~(size_t)31);
    ncap = ncap > 2048 ? 2048 : ncap;
    smem = (size_t)ncap * 39 + (staged ? stage : 0);  // task records + staged iteration
  };
  bool st1, st2;
  int ncap1, ncap2;
  size_t smem1, smem2;
  plan(kLaneSmem16, st1, ncap1, smem1);  // three CTAs per SM
  plan(kLaneSmem32, st2, ncap2, smem2);  // two CTAs per SM
  const int tc1 = max(1, min(n_cand, ncap1 / max_np));
  dim3 grid1((n_cand + tc1 - 1) / tc1, n_iter);
  e = st1 ? launch_lanes<true, 16>(grid1, smem1, s, a, tc1, max_np, ncap1)
          : launch_lanes<false, 16>(grid1, smem1, s, a, tc1, max_np, ncap1);
  note_launch();
  if (e != cudaSuccess) return record_cuda_error(e);
  // the flagged tasks of each iteration, compacted; VMAX-32 CTAs take chunks of <= ncap2 of them
  // (CTAs past an iteration's count exit at once)
  k_flag_list<<<n_iter, 256, 0, s>>>(a.flags, n_cand, max_np, a.list32, a.count32, a.q_count + 21);
  note_launch();
  const int tc2 = 0;
  // staged passes take chunks of at most kChunk32 flagged tasks: config 4's ~790 per iteration
  // then fill two CTAs each, and the pass runs ~7 waves instead of ~3.5 (a shorter tail)
  const int chunk2 = st2 ? min(ncap2, kChunk32) : ncap2;
  dim3 grid2((unsigned)(((size_t)n_cand * max_np + chunk2 - 1) / chunk2), n_iter);
  e = st2 ? launch_lanes<true, 32>(grid2, smem2, s, a, tc2, max_np, chunk2)
          : launch_lanes<false, 32>(grid2, smem2, s, a, tc2, max_np, chunk2);
  note_launch();
  if (e != cudaSuccess) return record_cuda_error(e);

  // warp per pipeline for the queue (V > 32, wide sums, infeasible V_a): persistent, no smem;
  // a short queue runs split (reference runs, then every surviving V as a unit, then re-runs)
  k_pack_big<<<kBigWarps / 8, 256, 0, s>>>(a);
  note_launch();
  k_pack_big_ref<<<kBigWarps / 8, 256, 0, s>>>(a);
  note_launch();
  k_pack_big_units<<<kBigWarps / 8, 256, 0, s>>>(a);
  note_launch();
  k_pack_big_finish<<<kBigWarps / 8, 256, 0, s>>>(a);
  note_launch();
  e = cudaGetLastError();
  return e == cudaSuccess ? HYD_OK : record_cuda_error(e);
}

}  // namespace hyd
