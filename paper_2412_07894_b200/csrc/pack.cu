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
// Two kernels:
//   k_pack_small: one LANE per pipeline (DP = next_pow2(max_np) lanes per (c,t), 32/DP
//     pairs per warp), member lists built in shared memory from the pipe row with SIMD byte
//     compares, bins in registers for V <= 32 (unrolled to a warp-uniform VMAX of 4/8/16/32),
//     u32 bin times when the pipeline's sumT < 2^32-1.  A lane whose search needs V > 32 is
//     pushed to a work queue instead.
//   k_pack_big: persistent warps pop (c,t,j) tasks; the WARP owns one pipeline, lanes own
//     bins b = lane + 32 r (r < R <= 8 in registers, or global scratch beyond 256 bins);
//     per item a redux.sync min over times, then over bin ids, picks the bin.
//   makespan[t][c] = max_j ptime: written by k_pack_small over its lanes, completed with
//   atomicMax by k_pack_big for queued pipelines.
#include "hyd_internal.cuh"

namespace hyd {

constexpr int kVReg = 32;       // largest V handled by k_pack_small
constexpr int kBigRMax = 8;     // k_pack_big: register bins per lane (V <= 256)
constexpr int kBigWarps = 2048; // persistent warps of k_pack_big (scratch slots)

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

// ------------------------------------------------------------------ LPT, one lane per pipeline
template <int VMAX, typename TT>
__device__ __forceinline__ bool lpt_lane(const uint16_t* __restrict__ lst, uint16_t* __restrict__ mbr,
                                         uint32_t U, uint32_t V, uint32_t M,
                                         const uint32_t* __restrict__ sl,
                                         const uint32_t* __restrict__ cs, int kp, uint32_t k,
                                         uint64_t thr64, uint64_t& maxbin, uint64_t& evals) {
  const TT thr = thr64 > (uint64_t)(TT)(~TT(0)) ? (TT)(~TT(0)) : (TT)thr64;
  TT tm[VMAX];
  uint32_t tk[VMAX];
#pragma unroll
  for (int b = 0; b < VMAX; ++b) {
    tm[b] = 0;
    tk[b] = (uint32_t)b < V ? 0u : 0xFFFFFFFFu;  // sentinel: never fits
  }
  TT mx = 0;
  for (uint32_t q = 0; q < U; ++q) {
    const uint32_t idx = lst[q];
    const uint32_t l = sl[idx];
    const TT tau = (TT)cs[(size_t)idx * kp + k];
    const uint32_t cap = M - l;
    TT bt = ~TT(0);
    uint32_t bb = VMAX;
#pragma unroll
    for (int b = 0; b < VMAX; ++b)
      if (tk[b] <= cap && tm[b] < bt) {
        bt = tm[b];
        bb = (uint32_t)b;
      }
    evals += V;
    if (bb == VMAX) return false;  // LPT(V) = bottom
    const TT nt = bt + tau;
#pragma unroll
    for (int b = 0; b < VMAX; ++b)
      if ((uint32_t)b == bb) {
        tm[b] = nt;
        tk[b] += l;
      }
    mx = nt > mx ? nt : mx;
    if (mx > thr) return false;  // cannot improve (obj, V)
    mbr[q] = (uint16_t)bb;
  }
  maxbin = (uint64_t)mx;
  return true;
}

template <typename TT>
__device__ __forceinline__ bool lpt_lane_dispatch(uint32_t vmax, const uint16_t* lst, uint16_t* mbr,
                                                  uint32_t U, uint32_t V, uint32_t M,
                                                  const uint32_t* sl, const uint32_t* cs, int kp,
                                                  uint32_t k, uint64_t thr, uint64_t& maxbin,
                                                  uint64_t& ev) {
  if (vmax <= 4) return lpt_lane<4, TT>(lst, mbr, U, V, M, sl, cs, kp, k, thr, maxbin, ev);
  if (vmax <= 8) return lpt_lane<8, TT>(lst, mbr, U, V, M, sl, cs, kp, k, thr, maxbin, ev);
  if (vmax <= 16) return lpt_lane<16, TT>(lst, mbr, U, V, M, sl, cs, kp, k, thr, maxbin, ev);
  return lpt_lane<32, TT>(lst, mbr, U, V, M, sl, cs, kp, k, thr, maxbin, ev);
}

// bytes of w equal to j (0xFF per matching byte)
__device__ __forceinline__ uint32_t match4(uint32_t w, uint32_t jjjj) { return __vcmpeq4(w, jjjj); }

template <int DP, bool STAGED>
__global__ void __launch_bounds__(128) k_pack_small(PackArgs a, int nw, int ct, int tt) {
  extern __shared__ __align__(16) uint32_t sm[];
  constexpr int G = 32 / DP;
  const int B = a.batch, kp = a.k_pad;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pslot = warp * G + lane / DP;
  const int j = lane % DP;
  const int c0 = blockIdx.x * ct, t0 = blockIdx.y * tt;
  const int npairs = nw * G;
  if (STAGED) {
    const int ntt = min(tt, a.n_iter - t0);
    const uint4* gl = reinterpret_cast<const uint4*>(a.sorted_len + (size_t)t0 * B);
    uint4* sl4 = reinterpret_cast<uint4*>(sm);
    for (int e = threadIdx.x; e < ntt * B / 4; e += blockDim.x) sl4[e] = __ldg(gl + e);
    const uint4* gc = reinterpret_cast<const uint4*>(a.cost + (size_t)t0 * B * kp);
    uint4* sc4 = reinterpret_cast<uint4*>(sm + (size_t)tt * B);
    for (int e = threadIdx.x; e < ntt * B * kp / 4; e += blockDim.x) sc4[e] = __ldg(gc + e);
    __syncthreads();
  }
  uint16_t* lists = reinterpret_cast<uint16_t*>(sm + (STAGED ? (size_t)tt * B * (1 + kp) : 0));
  uint16_t* lst = lists + (size_t)pslot * B;
  uint16_t* mbr = lists + (size_t)npairs * B + (size_t)pslot * B;

  const int lt = pslot / ct, lc = pslot - lt * ct;
  const int c = c0 + lc, t = t0 + lt;
  const bool pair_ok = lt < tt && c < a.n_cand && t < a.n_iter;
  const uint32_t* sl = STAGED ? sm + (size_t)lt * B : a.sorted_len + (size_t)t * B;
  const uint32_t* cs = STAGED ? sm + (size_t)tt * B + (size_t)lt * B * kp
                              : a.cost + (size_t)t * B * kp;
  const size_t row = (size_t)c * a.n_iter + t;
  const uint8_t* prow = a.pipe + row * B;
  uint16_t* mrow = a.mb + row * B;

  const int np = pair_ok ? (int)a.cand_np[c] : 0;
  bool infeasible = pair_ok && prow[0] == 0xFF;
  bool on = pair_ok && !infeasible && j < np;
  uint32_t k = on ? a.cand[(size_t)c * HYD_MAX_PIPES + j] : 0u;
  Search s;
  s.M = on ? a.schemes[k].max_len : 1u;
  s.P = on ? a.schemes[k].pp : 1u;
  s.UL = on ? a.schemes[k].util_len : 0u;

  if (infeasible) {  // whole row: mb 0xFFFF, v = ptime = 0, makespan = UINT64_MAX
    for (int i = j; i < B; i += DP) mrow[i] = 0xFFFF;
    for (int e = j; e < HYD_MAX_PIPES; e += DP) {
      a.v[row * HYD_MAX_PIPES + e] = 0;
      a.ptime[row * HYD_MAX_PIPES + e] = 0ull;
    }
    if (j == 0) a.makespan[(size_t)t * a.n_cand + c] = ~0ull;
  }

  // ---- member list of pipeline j: count, segmented exclusive scan, fill
  const uint32_t jjjj = 0x01010101u * (uint32_t)j;
  const bool vec = (B & 15) == 0;
  uint32_t cnt = 0;
  if (on) {
    if (vec) {
      const uint4* p4 = reinterpret_cast<const uint4*>(prow);
      for (int q = 0; q < B / 16; ++q) {
        const uint4 w = __ldg(p4 + q);
        cnt += (__popc(match4(w.x, jjjj)) + __popc(match4(w.y, jjjj)) + __popc(match4(w.z, jjjj)) +
                __popc(match4(w.w, jjjj))) >> 3;
      }
    } else {
      for (int i = 0; i < B; ++i) cnt += prow[i] == (uint8_t)j;
    }
  }
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < DP; o <<= 1) {
    const uint32_t y = __shfl_up_sync(HYD_FULL, incl, o, DP);
    if (j >= o) incl += y;
  }
  const uint32_t off = incl - cnt;
  lst += off;
  mbr += off;
  s.U = cnt;
  s.S = 0;
  s.sumT = 0;
  s.tau_max = 0;
  if (on && cnt) {
    uint32_t n = 0;
    auto take = [&](uint32_t idx) {
      lst[n] = (uint16_t)idx;
      const uint32_t tau = cs[(size_t)idx * kp + k];
      if (n == 0) s.tau_max = tau;
      s.S += sl[idx];
      s.sumT += tau;
      ++n;
    };
    if (vec) {
      const uint4* p4 = reinterpret_cast<const uint4*>(prow);
      for (int q = 0; q < B / 16 && n < cnt; ++q) {
        const uint4 w4 = __ldg(p4 + q);
        const uint32_t ws[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          uint32_t m = match4(ws[h], jjjj);
          while (m) {
            const int byte = (__ffs(m) - 1) >> 3;
            take((uint32_t)(16 * q + 4 * h + byte));
            m &= ~(0xFFu << (8 * byte));
          }
        }
      }
    } else {
      for (int i = 0; i < B; ++i)
        if (prow[i] == (uint8_t)j) take((uint32_t)i);
    }
  }

  // ---- exact pruned V search, lanes in lock-step rounds with a warp-uniform VMAX
  bool searching = on && s.U > 0;
  bool deferred = false;
  if (searching) search_init(s);
  const bool narrow = __all_sync(HYD_FULL, !searching || s.sumT < 0xFFFFFFFFull);
  uint64_t ev = 0;
  while (true) {
    uint32_t V = searching ? search_next(s) : 0u;
    if (searching && V == 0) searching = false;
    if (V > (uint32_t)kVReg) {
      deferred = true;
      searching = false;
      V = 0;
    }
    const uint32_t vmax = __reduce_max_sync(HYD_FULL, V);
    if (vmax == 0) break;
    if (V) {
      const uint64_t thr = search_thr(s, V);
      uint64_t mx = 0;
      const bool ok = narrow ? lpt_lane_dispatch<uint32_t>(vmax, lst, mbr, s.U, V, s.M, sl, cs, kp, k, thr, mx, ev)
                             : lpt_lane_dispatch<uint64_t>(vmax, lst, mbr, s.U, V, s.M, sl, cs, kp, k, thr, mx, ev);
      if (ok) {
        search_take(s, V, mx);
        for (uint32_t q = 0; q < s.U; ++q) mrow[lst[q]] = mbr[q];
      }
    }
  }

  // ---- outputs
  if (pair_ok && !infeasible) {
    if (!deferred) {
      for (int e = j; e < HYD_MAX_PIPES; e += DP) {
        const bool mine = e == j && on;
        a.v[row * HYD_MAX_PIPES + e] = mine ? (uint16_t)s.vbest : (uint16_t)0;
        a.ptime[row * HYD_MAX_PIPES + e] = mine ? s.best : 0ull;
      }
    } else {
      for (int e = j + DP; e < HYD_MAX_PIPES; e += DP) {
        a.v[row * HYD_MAX_PIPES + e] = 0;
        a.ptime[row * HYD_MAX_PIPES + e] = 0ull;
      }
      const unsigned long long slot = atomicAdd(a.q_count, 1ull);
      if (slot < a.q_cap)
        a.queue[slot] = ((unsigned long long)c << 37) | ((unsigned long long)t << 5) | (unsigned)j;
    }
  }
  ev = __reduce_add_sync(HYD_FULL, (uint32_t)min(ev, (uint64_t)0xFFFFFFFFull)) ;
  if (lane == 0 && ev) atomicAdd(a.evals, (unsigned long long)ev);
  uint64_t pm = (on && !deferred) ? s.best : 0ull;
#pragma unroll
  for (int o = DP / 2; o > 0; o >>= 1) pm = max(pm, __shfl_xor_sync(HYD_FULL, pm, o, DP));
  if (pair_ok && !infeasible && j == 0) a.makespan[(size_t)t * a.n_cand + c] = pm;
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

template <int DP>
static cudaError_t launch_small(bool staged, dim3 grid, int threads, size_t smem, cudaStream_t s,
                                const PackArgs& a, int nw, int ct, int tt) {
  cudaError_t e;
  if (staged) {
    e = cudaFuncSetAttribute(k_pack_small<DP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_pack_small<DP, true><<<grid, threads, smem, s>>>(a, nw, ct, tt);
  } else {
    e = cudaFuncSetAttribute(k_pack_small<DP, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_pack_small<DP, false><<<grid, threads, smem, s>>>(a, nw, ct, tt);
  }
  return cudaGetLastError();
}

int launch_pack(const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch, int k_pad,
                const hyd_scheme* schemes, int n_schemes, const uint8_t* cand,
                const uint8_t* cand_np, int n_cand, int max_np, const uint8_t* pipe, uint16_t* mb,
                uint16_t* v, uint64_t* ptime, uint64_t* makespan, uint32_t* status, void* ws,
                size_t ws_bytes, cudaStream_t s) {
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

  // small kernel geometry: nw warps x (32/dp) pairs; shrink nw until lists fit
  const int G = 32 / dp;
  int nw = 4;
  while (nw > 1 && (size_t)nw * G * batch * 4 > 96 * 1024) nw >>= 1;
  const int npairs = nw * G;
  const int ct = n_cand < npairs ? n_cand : npairs;
  const int tt = npairs / ct;
  const size_t lists = (size_t)npairs * batch * 4;
  const size_t stage = (size_t)tt * batch * 4 * (1 + (size_t)k_pad);
  const bool staged = (batch % 4) == 0 && stage + lists <= 112 * 1024;
  const size_t smem = lists + (staged ? stage : 0);
  dim3 grid((n_cand + ct - 1) / ct, (n_iter + tt - 1) / tt);
  switch (dp) {
    case 2: e = launch_small<2>(staged, grid, nw * 32, smem, s, a, nw, ct, tt); break;
    case 4: e = launch_small<4>(staged, grid, nw * 32, smem, s, a, nw, ct, tt); break;
    case 8: e = launch_small<8>(staged, grid, nw * 32, smem, s, a, nw, ct, tt); break;
    case 16: e = launch_small<16>(staged, grid, nw * 32, smem, s, a, nw, ct, tt); break;
    default: e = launch_small<32>(staged, grid, nw * 32, smem, s, a, nw, ct, tt); break;
  }
  note_launch();
  if (e != cudaSuccess) return record_cuda_error(e);

  // big kernel: persistent warps over the queue
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
