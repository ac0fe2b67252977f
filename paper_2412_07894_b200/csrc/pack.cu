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
//   k_pack_init: per (c,t) makespan = 0 / UINT64_MAX, v/ptime rows zeroed, infeasible mb rows.
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
#include "hyd_internal.cuh"

namespace hyd {

constexpr int kLaneVMax = 16;     // largest V handled by k_pack_lanes
constexpr int kLaneThreads = 256;
constexpr int kBigRMax = 8;       // k_pack_big: register bins per lane (V <= 256)
constexpr int kBigWarps = 2048;   // persistent warps of k_pack_big (scratch slots)

struct PackArgs {
  const uint32_t* sorted_len;
  const uint32_t* cost;
  int n_iter, batch, k_pad;
  const hyd_scheme* schemes;
  int n_schemes;
  const uint8_t* cand;
  const uint8_t* cand_np;
  int n_cand;
  const uint8_t* pipe;
  const hyd_pipe_stats* stats;
  uint16_t* mb;
  uint16_t* v;
  uint64_t* ptime;
  uint64_t* makespan;
  uint32_t* status;
  unsigned long long* q_count;
  unsigned long long* q_head;
  unsigned long long* evals;  // (item, bin) evaluations performed (ws bytes [16, 24))
  unsigned long long* queue;
  unsigned long long q_cap;
  uint64_t* scr_time;  // [kBigWarps][B]
  uint32_t* scr_tok;   // [kBigWarps][B]
};

// ------------------------------------------------------------------ exact V search state
struct Search {
  uint64_t S, sumT, best;
  uint32_t U, M, P, UL, tau_max, vlo, vhi, va, cursor, vbest;
  int phase;
  bool have;
};

__device__ __forceinline__ void search_init(Search& s) {
  const uint64_t vlo = max((s.S + s.M - 1) / s.M, (uint64_t)1);
  uint64_t vhi = s.UL ? min(s.S / s.UL, (uint64_t)s.U) : (uint64_t)s.U;
  if (vhi < vlo) vhi = vlo;
  s.vlo = (uint32_t)vlo;
  s.vhi = (uint32_t)vhi;
  uint32_t va = s.vlo;
  if (s.P > 1 && s.tau_max > 0) {
    const float vc = (float)s.sumT / (float)s.tau_max;
    const float vcl = fminf(fmaxf(vc + 0.5f, (float)s.vlo), (float)s.vhi);
    va = (uint32_t)vcl;
    va = min(max(va, s.vlo), s.vhi);
  }
  s.va = va;
  s.cursor = s.vlo;
  s.phase = 0;
  s.have = false;
  s.best = 0;
  s.vbest = 0;
}

// next V to evaluate, 0 when the search is complete
__device__ __forceinline__ uint32_t search_next(Search& s) {
  if (s.phase == 0) {
    s.phase = 1;
    return s.va;
  }
  if (s.phase == 1) {
    while (s.cursor <= s.vhi) {
      const uint32_t V = s.cursor++;
      if (V == s.va) continue;
      if (s.have) {
        const uint64_t m = (uint64_t)(s.P - 1 + V);
        const uint64_t tb = (uint64_t)s.tau_max * m;
        if (tb > s.best || (tb >= s.best && V > s.vbest)) {
          s.cursor = s.vhi + 1;  // tau_max (PP-1+V) grows with V: no later V can win
          break;
        }
        uint64_t ah, al, bh, bl;
        mul128(s.sumT, m, ah, al);
        mul128(s.best, (uint64_t)V, bh, bl);
        if (gt128(ah, al, bh, bl)) continue;                          // LB(V) > best
        if (!gt128(bh, bl, ah, al) && V > s.vbest) continue;          // LB(V) >= best, larger V
      }
      return V;
    }
    s.phase = 2;
    s.cursor = s.vhi + 1;
  }
  if (s.phase == 2) {
    if (!s.have && s.cursor <= s.U) return s.cursor++;  // extension above the range (reading 5)
    s.phase = 3;
  }
  return 0;
}

// largest max-bin time that can still improve (obj, V)
__device__ __forceinline__ uint64_t search_thr(const Search& s, uint32_t V) {
  if (!s.have) return ~0ull;
  const uint64_t m = (uint64_t)(s.P - 1 + V);
  if (V < s.vbest) return s.best / m;
  return s.best == 0 ? 0ull : (s.best - 1) / m;
}

__device__ __forceinline__ void search_take(Search& s, uint32_t V, uint64_t maxbin) {
  s.best = maxbin * (uint64_t)(s.P - 1 + V);
  s.vbest = V;
  s.have = true;
}

// ------------------------------------------------------------------ pair-level init
// makespan = 0 (feasible) or UINT64_MAX (infeasible); v/ptime rows zeroed; infeasible
// pairs get mb = 0xFFFF.  Tasks then write their v/ptime slot and atomicMax the makespan.
__global__ void __launch_bounds__(256) k_pack_init(const uint8_t* __restrict__ pipe, int n_iter,
                                                   int batch, int n_cand, uint16_t* __restrict__ mb,
                                                   uint16_t* __restrict__ v,
                                                   uint64_t* __restrict__ ptime,
                                                   uint64_t* __restrict__ makespan) {
  const size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (e >= (size_t)n_iter * n_cand) return;
  const int t = (int)(e / n_cand), c = (int)(e - (size_t)t * n_cand);
  const size_t row = (size_t)c * n_iter + t;
  const bool feasible = pipe[row * batch] != 0xFF;
  makespan[(size_t)t * n_cand + c] = feasible ? 0ull : ~0ull;
  uint4* v4 = reinterpret_cast<uint4*>(v + row * HYD_MAX_PIPES);
  uint4* p4 = reinterpret_cast<uint4*>(ptime + row * HYD_MAX_PIPES);
  const uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
  for (int q = 0; q < 4; ++q) v4[q] = z;
#pragma unroll
  for (int q = 0; q < 16; ++q) p4[q] = z;
  if (!feasible) {
    uint16_t* mrow = mb + row * batch;
    if ((batch & 7) == 0) {
      const uint4 f = make_uint4(~0u, ~0u, ~0u, ~0u);
      for (int q = 0; q < batch / 8; ++q) reinterpret_cast<uint4*>(mrow)[q] = f;
    } else {
      for (int i = 0; i < batch; ++i) mrow[i] = 0xFFFF;
    }
  }
}

// ------------------------------------------------------------------ persistent lanes (V <= 16)
// bins as packed u32 keys: key_b = time_b << 5 | b (needs sumT < 2^26), tokens tok_b.
// masked_b = key_b | ((cap - tok_b) & 2^31) is >= 2^31 iff tok_b + l > MaxLen, so the
// minimum masked key is the least-time fitting bin with the smallest index.
template <int N>
__device__ __forceinline__ uint32_t argmin_keys(const uint32_t (&keys)[kLaneVMax],
                                                const uint32_t (&toks)[kLaneVMax], uint32_t cap) {
  uint32_t m[N];
#pragma unroll
  for (int b = 0; b < N; ++b) m[b] = keys[b] | ((cap - toks[b]) & 0x80000000u);
#pragma unroll
  for (int w = N / 2; w > 0; w >>= 1)
#pragma unroll
    for (int b = 0; b < w; ++b) m[b] = min(m[b], m[b + w]);
  return m[0];
}

template <int N>
__device__ __forceinline__ void place_key(uint32_t (&keys)[kLaneVMax], uint32_t (&toks)[kLaneVMax],
                                          uint32_t mk, uint32_t tau5, uint32_t l) {
#pragma unroll
  for (int b = 0; b < N; ++b) {
    const bool hit = keys[b] == mk;
    keys[b] += hit ? tau5 : 0u;
    toks[b] += hit ? l : 0u;
  }
}

struct LaneRun {
  uint32_t V, thr, mx, wV;
  bool writing, final_run;
};

template <bool STAGED>
__global__ void __launch_bounds__(kLaneThreads, 2) k_pack_lanes(PackArgs a, int tc, int mnp) {
  extern __shared__ __align__(16) uint32_t sm[];
  __shared__ int s_n8, s_n16, s_next;
  const int B = a.batch, kp = a.k_pad;
  const int t = blockIdx.y, c0 = blockIdx.x * tc;
  const int tid = threadIdx.x;
  const int ntask_max = tc * mnp;
  uint16_t* list = reinterpret_cast<uint16_t*>(sm + (STAGED ? (size_t)B * (1 + kp) : 0));
  if (tid == 0) {
    s_n8 = 0;
    s_n16 = 0;
    s_next = 0;
  }
  if (STAGED) {
    const uint4* gl = reinterpret_cast<const uint4*>(a.sorted_len + (size_t)t * B);
    uint4* s4 = reinterpret_cast<uint4*>(sm);
    for (int e = tid; e < B / 4; e += kLaneThreads) s4[e] = __ldg(gl + e);
    const uint4* gc = reinterpret_cast<const uint4*>(a.cost + (size_t)t * B * kp);
    uint4* c4 = reinterpret_cast<uint4*>(sm + B);
    for (int e = tid; e < B * kp / 4; e += kLaneThreads) c4[e] = __ldg(gc + e);
  }
  __syncthreads();
  const uint32_t* slen = STAGED ? sm : a.sorted_len + (size_t)t * B;
  const uint32_t* cst = STAGED ? sm + B : a.cost + (size_t)t * B * kp;
  const bool vec_ok = (B & 15) == 0;

  // ---- task list of this CTA, split into VMAX classes 8 (front) and 16 (back)
  for (int e = tid; e < ntask_max; e += kLaneThreads) {
    const int c = c0 + e / mnp, j = e % mnp;
    if (c >= a.n_cand || j >= (int)a.cand_np[c]) continue;
    const size_t row = (size_t)c * a.n_iter + t;
    if (a.pipe[row * B] == 0xFF) continue;  // infeasible pair: k_pack_init wrote it
    const hyd_pipe_stats st = a.stats[row * mnp + j];
    if (st.u == 0) continue;  // empty pipeline: V = ptime = 0 (k_pack_init)
    const uint32_t k = a.cand[(size_t)c * HYD_MAX_PIPES + j];
    Search s;
    s.M = a.schemes[k].max_len;
    s.P = a.schemes[k].pp;
    s.UL = a.schemes[k].util_len;
    s.U = st.u;
    s.S = st.s;
    s.sumT = st.sum_t;
    s.tau_max = st.tau_max;
    search_init(s);
    if (!vec_ok || s.sumT >= (1ull << 26) || s.M >= 0x80000000u || s.va > (uint32_t)kLaneVMax) {
      const unsigned long long slot = atomicAdd(a.q_count, 1ull);
      if (slot < a.q_cap)
        a.queue[slot] = ((unsigned long long)c << 37) | ((unsigned long long)t << 5) | (unsigned)j;
    } else if (s.va <= 8) {
      list[atomicAdd(&s_n8, 1)] = (uint16_t)e;
    } else {
      list[ntask_max - 1 - atomicAdd(&s_n16, 1)] = (uint16_t)e;
    }
  }
  __syncthreads();
  const int n8 = s_n8, ntask = s_n8 + s_n16;

  // ---- persistent lane state machine: one sequence (or one task set-up) per iteration
  bool have = false;
  int c = 0, j = 0;
  uint32_t k = 0, jjjj = 0;
  size_t row = 0;
  const uint8_t* prow = nullptr;
  uint16_t* mrow = nullptr;
  Search s;
  LaneRun r;
  r.V = r.thr = r.mx = r.wV = 0;
  r.writing = r.final_run = false;
  uint32_t keys[kLaneVMax], toks[kLaneVMax];
  uint32_t qc = 0, m16 = 0, cbase = 0;
  const uint32_t nchunks = (uint32_t)B / 16;
  uint64_t ev = 0;

  auto start_run = [&](uint32_t V, bool write, bool fin) {
    r.V = V;
    r.writing = write;
    r.final_run = fin;
    const uint64_t th = (write || fin) ? ~0ull : search_thr(s, V);
    r.thr = th > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)th;
    r.mx = 0;
#pragma unroll
    for (int b = 0; b < kLaneVMax; ++b) {
      keys[b] = (uint32_t)b < V ? (uint32_t)b : 0xFFFFFFFFu;
      toks[b] = 0u;
    }
    qc = 0;
    m16 = 0;
  };
  auto finalize = [&]() {
    a.v[row * HYD_MAX_PIPES + j] = (uint16_t)s.vbest;
    a.ptime[row * HYD_MAX_PIPES + j] = s.best;
    atomicMax(reinterpret_cast<unsigned long long*>(a.makespan + (size_t)t * a.n_cand + c),
              (unsigned long long)s.best);
    have = false;
  };
  auto defer = [&]() {
    const unsigned long long slot = atomicAdd(a.q_count, 1ull);
    if (slot < a.q_cap)
      a.queue[slot] = ((unsigned long long)c << 37) | ((unsigned long long)t << 5) | (unsigned)j;
    have = false;
  };
  auto run_end = [&](bool ok) {
    if (ok) {
      search_take(s, r.V, r.mx);
      if (r.writing) r.wV = r.V;
    }
    if (r.final_run) {
      finalize();
      return;
    }
    const uint32_t nv = search_next(s);
    if (nv == 0) {
      if (!s.have) defer();  // cannot happen (V = U is always feasible); safety net
      else if (s.vbest != r.wV) start_run(s.vbest, true, true);  // write the winner's mb
      else finalize();
    } else if (nv > (uint32_t)kLaneVMax) {
      defer();
    } else {
      start_run(nv, false, false);
    }
  };

  while (true) {
    if (!have) {
      const int e = atomicAdd(&s_next, 1);
      if (e >= ntask) break;
      const int le = e < n8 ? list[e] : list[ntask_max - (ntask - e)];
      c = c0 + le / mnp;
      j = le % mnp;
      row = (size_t)c * a.n_iter + t;
      prow = a.pipe + row * B;
      mrow = a.mb + row * B;
      k = a.cand[(size_t)c * HYD_MAX_PIPES + j];
      jjjj = 0x01010101u * (uint32_t)j;
      const hyd_pipe_stats st = a.stats[row * mnp + j];
      s.M = a.schemes[k].max_len;
      s.P = a.schemes[k].pp;
      s.UL = a.schemes[k].util_len;
      s.U = st.u;
      s.S = st.s;
      s.sumT = st.sum_t;
      s.tau_max = st.tau_max;
      search_init(s);
      r.wV = 0;
      start_run(s.va, true, false);  // the first run always completes or is infeasible
      have = true;
    }
    // next member of pipeline j in sorted order: 16 pipe bytes -> 16-bit match mask
    while (m16 == 0 && qc < nchunks) {
      const uint4 w4 = __ldg(reinterpret_cast<const uint4*>(prow) + qc);
      const uint32_t x0 = __vcmpeq4(w4.x, jjjj) & 0x01010101u, x1 = __vcmpeq4(w4.y, jjjj) & 0x01010101u;
      const uint32_t x2 = __vcmpeq4(w4.z, jjjj) & 0x01010101u, x3 = __vcmpeq4(w4.w, jjjj) & 0x01010101u;
      m16 = ((x0 * 0x204081u) >> 21 & 0xFu) | (((x1 * 0x204081u) >> 21 & 0xFu) << 4) |
            (((x2 * 0x204081u) >> 21 & 0xFu) << 8) | (((x3 * 0x204081u) >> 21 & 0xFu) << 12);
      cbase = qc * 16u;
      ++qc;
    }
    if (m16 == 0) {  // every member placed: run complete
      run_end(true);
      continue;
    }
    const uint32_t i = cbase + (uint32_t)(__ffs(m16) - 1);
    m16 &= m16 - 1u;
    const uint32_t l = slen[i];
    const uint32_t tau = cst[(size_t)i * kp + k];
    const uint32_t cap = s.M - l;
    ev += r.V;
    uint32_t mk;
    if (r.V <= 8) {
      mk = argmin_keys<8>(keys, toks, cap);
    } else {
      mk = argmin_keys<16>(keys, toks, cap);
    }
    if (mk >> 31) {  // no micro-batch can take the sequence: LPT(V) infeasible
      run_end(false);
      continue;
    }
    const uint32_t nt = (mk >> 5) + tau;
    if (r.V <= 8) {
      place_key<8>(keys, toks, mk, tau << 5, l);
    } else {
      place_key<16>(keys, toks, mk, tau << 5, l);
    }
    r.mx = max(r.mx, nt);
    if (r.writing) mrow[i] = (uint16_t)(mk & 31u);
    if (r.mx > r.thr) run_end(false);  // cannot improve (obj, V): abort this V
  }
  ev = __reduce_add_sync(__activemask(), (uint32_t)min(ev, (uint64_t)0xFFFFFFFFull));
  if ((tid & 31) == 0 && ev) atomicAdd(a.evals, (unsigned long long)ev);
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
template <int R, typename TT>
__device__ __forceinline__ bool lpt_warp(const uint16_t* __restrict__ lst, uint16_t* __restrict__ mbr,
                                         uint32_t U, uint32_t V, uint32_t M,
                                         const uint32_t* __restrict__ sl,
                                         const uint32_t* __restrict__ cs, int kp, uint32_t k,
                                         uint64_t thr64, uint64_t& maxbin, uint64_t* scr_t,
                                         uint32_t* scr_k, uint64_t& evals) {
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
  TT mx = 0;
  for (uint32_t q = 0; q < U; ++q) {
    const uint32_t idx = lst[q];
    const uint32_t l = __ldg(sl + idx);
    const TT tau = (TT)__ldg(cs + (size_t)idx * kp + k);
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
        for (int r = 0; r < RR; ++r)
          if ((uint32_t)r == rs) {
            tm[r] += tau;
            tk[r] += l;
          }
      } else {
        scr_t[bstar] += (uint64_t)tau;
        scr_k[bstar] += l;
      }
    }
    const TT nt = m + tau;
    mx = nt > mx ? nt : mx;
    if (mx > thr) return false;
    if (lane == 0) mbr[q] = (uint16_t)bstar;
  }
  maxbin = (uint64_t)mx;
  return true;
}

template <typename TT>
__device__ __forceinline__ bool lpt_warp_dispatch(const uint16_t* lst, uint16_t* mbr, uint32_t U,
                                                  uint32_t V, uint32_t M, const uint32_t* sl,
                                                  const uint32_t* cs, int kp, uint32_t k,
                                                  uint64_t thr, uint64_t& maxbin, uint64_t* st,
                                                  uint32_t* sk, uint64_t& ev) {
  if (V <= 32) return lpt_warp<1, TT>(lst, mbr, U, V, M, sl, cs, kp, k, thr, maxbin, st, sk, ev);
  if (V <= 64) return lpt_warp<2, TT>(lst, mbr, U, V, M, sl, cs, kp, k, thr, maxbin, st, sk, ev);
  if (V <= 128) return lpt_warp<4, TT>(lst, mbr, U, V, M, sl, cs, kp, k, thr, maxbin, st, sk, ev);
  if (V <= 32 * kBigRMax) return lpt_warp<kBigRMax, TT>(lst, mbr, U, V, M, sl, cs, kp, k, thr, maxbin, st, sk, ev);
  return lpt_warp<0, TT>(lst, mbr, U, V, M, sl, cs, kp, k, thr, maxbin, st, sk, ev);
}

__global__ void __launch_bounds__(256) k_pack_big(PackArgs a) {
  extern __shared__ __align__(16) uint32_t sm[];
  const int B = a.batch, kp = a.k_pad;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + warp;  // scratch slot
  uint16_t* lst = reinterpret_cast<uint16_t*>(sm) + (size_t)warp * 2 * B;
  uint16_t* mbr = lst + B;
  uint64_t* scr_t = a.scr_time + (size_t)gw * B;
  uint32_t* scr_k = a.scr_tok + (size_t)gw * B;
  const unsigned long long total = min(*a.q_count, a.q_cap);
  uint64_t ev = 0;
  while (true) {
    unsigned long long task = 0;
    if (lane == 0) task = atomicAdd(a.q_head, 1ull);
    task = __shfl_sync(HYD_FULL, task, 0);
    if (task >= total) break;
    const unsigned long long e = a.queue[task];
    const int c = (int)(e >> 37), t = (int)((e >> 5) & 0xFFFFFFFFull), j = (int)(e & 31);
    const size_t row = (size_t)c * a.n_iter + t;
    const uint8_t* prow = a.pipe + row * B;
    const uint32_t* sl = a.sorted_len + (size_t)t * B;
    const uint32_t* cs = a.cost + (size_t)t * B * kp;
    const uint32_t k = a.cand[(size_t)c * HYD_MAX_PIPES + j];
    Search s;
    s.M = a.schemes[k].max_len;
    s.P = a.schemes[k].pp;
    s.UL = a.schemes[k].util_len;
    // member list: 16 pipe bytes per lane per round, warp-wide exclusive scan of counts
    uint32_t n = 0;
    uint64_t S = 0, sumT = 0;
    for (int base = 0; base < B; base += 512) {
      const int i0 = base + 16 * lane;
      uint32_t m16 = 0;
      for (int b = 0; b < 16; ++b)
        if (i0 + b < B && prow[i0 + b] == (uint8_t)j) m16 |= 1u << b;
      const uint32_t cnt = __popc(m16);
      uint32_t incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(HYD_FULL, incl, o);
        if (lane >= o) incl += y;
      }
      uint32_t pos = n + incl - cnt;
      while (m16) {
        const int b = __ffs(m16) - 1;
        m16 &= m16 - 1;
        const uint32_t idx = (uint32_t)(i0 + b);
        lst[pos++] = (uint16_t)idx;
        S += __ldg(sl + idx);
        sumT += __ldg(cs + (size_t)idx * kp + k);
      }
      n += __shfl_sync(HYD_FULL, incl, 31);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      S += __shfl_xor_sync(HYD_FULL, S, o);
      sumT += __shfl_xor_sync(HYD_FULL, sumT, o);
    }
    __syncwarp();
    s.U = n;
    s.S = S;
    s.sumT = sumT;
    s.tau_max = n ? __ldg(cs + (size_t)lst[0] * kp + k) : 0u;
    uint16_t* mrow = a.mb + row * B;
    if (n) {
      search_init(s);
      const bool narrow = s.sumT < 0xFFFFFFFFull;
      uint32_t V;
      while ((V = search_next(s)) != 0) {
        const uint64_t thr = search_thr(s, V);
        uint64_t mx = 0;
        const bool ok = narrow ? lpt_warp_dispatch<uint32_t>(lst, mbr, s.U, V, s.M, sl, cs, kp, k, thr, mx, scr_t, scr_k, ev)
                               : lpt_warp_dispatch<uint64_t>(lst, mbr, s.U, V, s.M, sl, cs, kp, k, thr, mx, scr_t, scr_k, ev);
        __syncwarp();
        if (ok) {
          search_take(s, V, mx);
          for (uint32_t q = lane; q < s.U; q += 32) mrow[lst[q]] = mbr[q];
        }
        __syncwarp();
      }
    } else {
      s.best = 0;
      s.vbest = 0;
    }
    if (lane == 0) {
      a.v[row * HYD_MAX_PIPES + j] = (uint16_t)s.vbest;
      a.ptime[row * HYD_MAX_PIPES + j] = s.best;
      atomicMax(reinterpret_cast<unsigned long long*>(a.makespan + (size_t)t * a.n_cand + c),
                (unsigned long long)s.best);
    }
    __syncwarp();
  }
  if (lane == 0 && ev) atomicAdd(a.evals, (unsigned long long)ev);
}

// ------------------------------------------------------------------ host side
static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static int dp_of(int max_np) {
  return max_np <= 2 ? 2 : max_np <= 4 ? 4 : max_np <= 8 ? 8 : max_np <= 16 ? 16 : 32;
}

size_t pack_workspace(int n_iter, int batch, int n_cand, int max_np) {
  const size_t cap = (size_t)n_iter * n_cand * dp_of(max_np);
  return align256(32) + align256(cap * 8) + align256((size_t)kBigWarps * batch * 8) +
         align256((size_t)kBigWarps * batch * 4);
}

template <bool STAGED>
static cudaError_t launch_lanes(dim3 grid, size_t smem, cudaStream_t s, const PackArgs& a, int tc,
                                int mnp) {
  cudaError_t e = cudaFuncSetAttribute(k_pack_lanes<STAGED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  k_pack_lanes<STAGED><<<grid, kLaneThreads, smem, s>>>(a, tc, mnp);
  return cudaGetLastError();
}

int launch_pack(const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch, int k_pad,
                const hyd_scheme* schemes, int n_schemes, const uint8_t* cand,
                const uint8_t* cand_np, int n_cand, int max_np, const uint8_t* pipe,
                const hyd_pipe_stats* stats, uint16_t* mb, uint16_t* v, uint64_t* ptime,
                uint64_t* makespan, uint32_t* status, void* ws, size_t ws_bytes, cudaStream_t s) {
  (void)ws_bytes;
  if (n_iter == 0 || n_cand == 0) return HYD_OK;
  const int dp = dp_of(max_np);
  PackArgs a;
  a.sorted_len = sorted_len;
  a.cost = cost;
  a.n_iter = n_iter;
  a.batch = batch;
  a.k_pad = k_pad;
  a.schemes = schemes;
  a.n_schemes = n_schemes;
  a.cand = cand;
  a.cand_np = cand_np;
  a.n_cand = n_cand;
  a.pipe = pipe;
  a.stats = stats;
  a.mb = mb;
  a.v = v;
  a.ptime = ptime;
  a.makespan = makespan;
  a.status = status;
  char* w = static_cast<char*>(ws);
  a.q_count = reinterpret_cast<unsigned long long*>(w);
  a.q_head = a.q_count + 1;
  a.evals = a.q_count + 2;
  w += align256(32);
  a.q_cap = (unsigned long long)n_iter * n_cand * dp;
  a.queue = reinterpret_cast<unsigned long long*>(w);
  w += align256(a.q_cap * 8);
  a.scr_time = reinterpret_cast<uint64_t*>(w);
  w += align256((size_t)kBigWarps * batch * 8);
  a.scr_tok = reinterpret_cast<uint32_t*>(w);

  cudaError_t e = cudaMemsetAsync(a.q_count, 0, 24, s);
  if (e != cudaSuccess) return record_cuda_error(e);
  const size_t pairs = (size_t)n_iter * n_cand;
  k_pack_init<<<(unsigned)((pairs + 255) / 256), 256, 0, s>>>(pipe, n_iter, batch, n_cand, mb, v, ptime,
                                                              makespan);
  note_launch();
  e = cudaGetLastError();
  if (e != cudaSuccess) return record_cuda_error(e);

  // persistent lanes: a CTA = one iteration x tc candidates (~2048 pipeline tasks)
  const int tc = n_cand < 2048 / max_np ? n_cand : (2048 / max_np > 0 ? 2048 / max_np : 1);
  const size_t stage = (size_t)batch * 4 * (1 + (size_t)k_pad);
  const size_t list = (((size_t)tc * max_np * 2) + 15) & ~(size_t)15;
  const bool staged = (batch % 4) == 0 && stage + list <= 100 * 1024;
  dim3 grid((n_cand + tc - 1) / tc, n_iter);
  e = staged ? launch_lanes<true>(grid, stage + list, s, a, tc, max_np)
             : launch_lanes<false>(grid, list, s, a, tc, max_np);
  note_launch();
  if (e != cudaSuccess) return record_cuda_error(e);

  // warp per pipeline for the queue (V > 16, wide sums, ragged batches)
  int wpb = 8;
  while (wpb > 1 && (size_t)wpb * batch * 4 > 96 * 1024) wpb >>= 1;
  const size_t bsm = (size_t)wpb * batch * 4;
  e = cudaFuncSetAttribute(k_pack_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm);
  if (e != cudaSuccess) return record_cuda_error(e);
  k_pack_big<<<kBigWarps / wpb, wpb * 32, bsm, s>>>(a);
  note_launch();
  e = cudaGetLastError();
  return e == cudaSuccess ? HYD_OK : record_cuda_error(e);
}

}  // namespace hyd
