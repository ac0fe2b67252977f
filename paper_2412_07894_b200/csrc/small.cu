// small.cu -- a3 + a4 fused for small batches: the paper's own workload shape (token-budget
// iterations of 100K tokens with a 32K context hold ~51 sequences).
//
// For B_t <= HYD_SMALL_MAX_BATCH (128) and at most 16 pipelines per candidate, one THREAD per
// (c, t) runs stage 1 and stage 2 back to back with everything in registers and shared memory:
//   * the CTA (128 candidates of one iteration; 32 when there are at most 32) stages the sorted lengths and cost
//     rows once;
//   * dispatch (HYD-H1; Eq. 2/3 P:634-650, Alg. 1's rule P:1131-1144):
//     base_j = C_j + E_j and mult_j = PP_j while pipeline j is empty, 1 after, so a candidate
//     load is one multiply-add, new_j = base_j + tau mult_j; j* = argmin (new_j, j) over
//     MaxLen_j >= l (J_i); u32 arithmetic when a per-CTA bound on every load allows;
//     decisions go straight to the pipe row and to per-pipeline membership words in shared
//     memory, token sums S_j and base_j to a per-thread shared record;
//   * pack (Eq. 1 P:604-607 over App. D's range P:1097): per pipeline the exact pruned V search
//     of search.cuh (V_a first writing mb, then the surviving V with an abort threshold, then a
//     re-run of the winner if it was not V_a -- exactly k_pack_big's sequence), bins in
//     registers as packed keys time << 4 | b (u32, or u64 when a bin time can reach 2^27) with the
//     sign-bit capacity mask (pack.cu) for V <= 16, the warp choosing 4 / 8 / 16 bins from its
//     widest run; wider V uses a generic loop with 64-bit bins in local memory;
//   * the mb row is staged in shared memory and leaves whole, with v / ptime rows (16-byte
//     stores), lb and makespan.
// There is no stats / members round trip through HBM and no task records.
#include "hyd_internal.cuh"
#include "search.cuh"

namespace hyd {

constexpr int kSmallThreads = 128;
constexpr int kSmallWords = HYD_SMALL_MAX_BATCH / 32;  // membership words per pipeline

struct SmallArgs {
  const uint32_t* sorted_len;
  const uint32_t* cost;
  int n_iter, batch, k_pad;
  const uint32_t* off;
  size_t n_total;
  const hyd_scheme* schemes;
  int n_schemes;
  const uint8_t* cand;
  const uint8_t* cand_np;
  int n_cand;
  uint8_t* pipe;
  uint64_t* lb;
  uint16_t* mb;
  uint16_t* v;
  uint64_t* ptime;
  uint64_t* makespan;
  uint32_t* status;
  unsigned long long* evals;
};

// per-thread shared records of the pipelines (structure of arrays, stride T = CTA threads so
// lane-consecutive): rs[j] = S_j (tokens), rb[j] = base_j = C_j + E_j; after pipeline j's
// search, rs[j] = V* and rb[j] = its objective (ptime)
template <int T>
struct PipeRec {
  uint32_t* rs;
  unsigned long long* rb;
  __device__ uint32_t& s(int j) const { return rs[j * T]; }
  __device__ unsigned long long& b(int j) const { return rb[j * T]; }
};

// One LPT(V) run over the members of one pipeline (mw: its membership words), V <= N
// <= 16 bins as packed keys time << 4 | b (KT = u32 when every bin time < 2^27, else u64) with
// the sign-bit capacity mask of pack.cu.  Returns false if no micro-batch fits (LPT(V)
// infeasible) or the running maximum exceeds thr.  Writes each member's micro-batch to mbs
// when `write`.
template <int N, typename KT>
__device__ __forceinline__ bool run_keys(const uint32_t* __restrict__ mw, int nw, uint32_t V, uint32_t M,
                                         uint32_t k, uint64_t thr, bool write, uint8_t* __restrict__ mbs,
                                         const uint32_t* __restrict__ sl, const uint32_t* __restrict__ sc,
                                         int kp, uint64_t& mx_out, uint32_t& ev) {
  constexpr int HB = sizeof(KT) * 8 - 1;  // the mask bit
  const KT thr_k = thr > (uint64_t)(KT)~(KT)0 ? (KT)~(KT)0 : (KT)thr;
  KT keys[N];
  uint32_t rem[N];
#pragma unroll
  for (int b = 0; b < N; ++b) {
    keys[b] = (uint32_t)b < V ? (KT)b : (KT)~(KT)1;  // unused bins: never fit, never the minimum
    rem[b] = M;
  }
  KT mx = 0;
  for (int w = 0; w < nw; ++w) {
    uint32_t bits = mw[w];
    while (bits) {
      const uint32_t i = (uint32_t)(w * 32 + __ffs(bits) - 1);
      bits &= bits - 1u;
      const uint32_t l = sl[i];
      const uint32_t tau = sc[i * kp + k];
      // least-time bin whose tokens stay within MaxLen (mask bit set = does not fit), smallest b
      KT m[N];
#pragma unroll
      for (int b = 0; b < N; ++b) m[b] = keys[b] | ((KT)((rem[b] - l) >> 31) << HB);
      KT mk;
      if constexpr (sizeof(KT) == 4) {
        mk = min_tree3<N>(m);
      } else {
#pragma unroll
        for (int wd = N / 2; wd > 0; wd >>= 1)
#pragma unroll
          for (int b = 0; b < wd; ++b) m[b] = min(m[b], m[b + wd]);
        mk = m[0];
      }
      ev += V;
      if (mk >> HB) return false;
      const KT add = (KT)tau << 4;
#pragma unroll
      for (int b = 0; b < N; ++b) {
        const bool h = keys[b] == mk;
        keys[b] = h ? keys[b] + add : keys[b];
        rem[b] = h ? rem[b] - l : rem[b];
      }
      mx = max(mx, (KT)((mk >> 4) + tau));
      if (mx > thr_k) return false;
      HYD_CHECK(i < HYD_SMALL_MAX_BATCH);
      if (write) mbs[i] = (uint8_t)(mk & 15u);
    }
  }
  mx_out = (uint64_t)mx;
  return true;
}

// The same run for any V <= HYD_SMALL_MAX_BATCH with 64-bit bin times (bins in local memory).
__device__ __noinline__ bool run_generic(const uint32_t* __restrict__ mw, int nw, uint32_t V, uint32_t M,
                                         uint32_t k, uint64_t thr, bool write, uint8_t* __restrict__ mbs,
                                         const uint32_t* __restrict__ sl, const uint32_t* __restrict__ sc,
                                         int kp, uint64_t& mx, uint32_t& ev) {
  uint64_t tm[HYD_SMALL_MAX_BATCH];
  uint32_t tok[HYD_SMALL_MAX_BATCH];
  for (uint32_t b = 0; b < V; ++b) {
    tm[b] = 0ull;
    tok[b] = 0u;
  }
  mx = 0ull;
  for (int w = 0; w < nw; ++w) {
    uint32_t bits = mw[w];
    while (bits) {
      const uint32_t i = (uint32_t)(w * 32 + __ffs(bits) - 1);
      bits &= bits - 1u;
      const uint32_t l = sl[i];
      const uint32_t tau = sc[i * kp + k];
      uint64_t best = ~0ull;
      uint32_t bb = 0xFFFFFFFFu;
      for (uint32_t b = 0; b < V; ++b)
        if ((uint64_t)tok[b] + l <= M && tm[b] < best) {
          best = tm[b];
          bb = b;
        }
      ev += V;
      if (bb == 0xFFFFFFFFu) return false;
      HYD_CHECK(bb < V && V <= HYD_SMALL_MAX_BATCH && i < HYD_SMALL_MAX_BATCH);
      tm[bb] += tau;
      tok[bb] += l;
      mx = max(mx, tm[bb]);
      if (mx > thr) return false;
      if (write) mbs[i] = (uint8_t)bb;
    }
  }
  return true;
}

template <int DP, typename TT, int T>
__device__ __forceinline__ void small_dispatch(const uint32_t* __restrict__ sl, const uint32_t* __restrict__ sc,
                                               int B, int kp, int np, const uint32_t (&ml)[DP],
                                               const uint32_t (&pp)[DP], const uint32_t (&kk)[DP],
                                               uint32_t* __restrict__ mem, const PipeRec<T>& rec,
                                               uint8_t* __restrict__ prow, uint64_t& lb_out) {
  TT base[DP];
  uint32_t mult[DP], S[DP];
#pragma unroll
  for (int j = 0; j < DP; ++j) {  // unused slots never win: base = max, mult = 0
    base[j] = j < np ? (TT)0 : (TT)~(TT)0;
    mult[j] = j < np ? pp[j] : 0u;
    S[j] = 0u;
  }
  const bool words = ((size_t)prow & 3) == 0;
  uint32_t word = 0u;
  for (int i = 0; i < B; ++i) {
    const uint32_t l = sl[i];
    const uint32_t* crow = sc + i * kp;
    TT best = (TT)~(TT)0;
    uint32_t bj = 0u;
#pragma unroll
    for (int j = 0; j < DP; ++j) {
      const TT nw = base[j] + (TT)crow[kk[j]] * (TT)mult[j];
      if (l <= ml[j] && nw < best) {
        best = nw;
        bj = (uint32_t)j;
      }
    }
#pragma unroll
    for (int j = 0; j < DP; ++j) {
      const bool hit = (uint32_t)j == bj;
      base[j] = hit ? best : base[j];
      mult[j] = hit ? 1u : mult[j];
      S[j] += hit ? l : 0u;
    }
    HYD_CHECK(bj < (uint32_t)DP && i < HYD_SMALL_MAX_BATCH);
    mem[bj * kSmallWords + (i >> 5)] |= 1u << (i & 31);
    if (words) {
      word |= bj << (8 * (i & 3));
      if ((i & 3) == 3 || i == B - 1) {
        if ((i & 3) == 3) {
          *reinterpret_cast<uint32_t*>(prow + (i & ~3)) = word;
        } else {
          for (int q = i & ~3; q <= i; ++q) prow[q] = (uint8_t)(word >> (8 * (q & 3)));
        }
        word = 0u;
      }
    } else {
      prow[i] = (uint8_t)bj;
    }
  }
  uint64_t m = 0ull;
#pragma unroll
  for (int j = 0; j < DP; ++j)
    if (j < np) {
      m = max(m, (uint64_t)base[j]);
      rec.s(j) = S[j];
      rec.b(j) = (unsigned long long)base[j];
    }
  lb_out = m;
}

// T = CTA threads (candidates of the iteration per CTA): 128, or 32 when there are at most 32
// candidates -- one-warp CTAs then keep four times as many (c, t) latency chains resident.
template <int DP, int T>
__global__ void __launch_bounds__(T) k_assign_small(SmallArgs a) {
  extern __shared__ __align__(16) uint32_t sm[];
  __shared__ uint32_t s_ml[HYD_MAX_SCHEMES], s_pp[HYD_MAX_SCHEMES], s_ul[HYD_MAX_SCHEMES];
  __shared__ unsigned long long s_sum, s_max;
  const int tid = threadIdx.x, lane = tid & 31;
  const int t = blockIdx.y, c = blockIdx.x * T + tid;
  const int B = geo_bt(a.off, a.batch, t);
  const size_t tbase = geo_base(a.off, a.batch, t);
  const int kp = a.k_pad;
  // smem: bases [DP][T] u64 | lengths [Bmax] | costs [Bmax][kp] | members [T][DP][W] |
  //       S [DP][T] u32 | mb [T][Bmax] u8
  unsigned long long* rb_all = reinterpret_cast<unsigned long long*>(sm);
  uint32_t* sl = reinterpret_cast<uint32_t*>(rb_all + T * DP);
  uint32_t* sc = sl + HYD_SMALL_MAX_BATCH;
  uint32_t* mem_all = sc + HYD_SMALL_MAX_BATCH * kp;
  uint32_t* rs_all = mem_all + T * DP * kSmallWords;
  uint8_t* mb_all = reinterpret_cast<uint8_t*>(rs_all + T * DP);
  uint32_t* mem = mem_all + tid * DP * kSmallWords;
  const PipeRec<T> rec{rs_all + tid, rb_all + tid};
  uint8_t* mbs = mb_all + tid * HYD_SMALL_MAX_BATCH;

  if (tid == 0) {
    s_sum = 0ull;
    s_max = 0ull;
  }
  for (int k = tid; k < a.n_schemes; k += T) {
    s_ml[k] = a.schemes[k].max_len;
    s_pp[k] = a.schemes[k].pp;
    s_ul[k] = a.schemes[k].util_len;
  }
  for (int e = tid; e < B; e += T) sl[e] = __ldg(a.sorted_len + tbase + e);
  for (int e = tid; e < B * kp; e += T) sc[e] = __ldg(a.cost + tbase * kp + e);
  for (int e = 0; e < DP * kSmallWords; ++e) mem[e] = 0u;
  __syncthreads();
  // every load of this iteration is below sum_i max_k tau_ik + max tau (PPmax - 1): u32 if < 2^32
  {
    unsigned long long part = 0ull, mxv = 0ull;
    for (int i = tid; i < B; i += T) {
      uint32_t m = 0u;
      for (int k = 0; k < a.n_schemes; ++k) {
        const uint32_t tau = sc[i * kp + k];
        m = max(m, tau);
        mxv = max(mxv, (unsigned long long)tau * (s_pp[k] - 1u));
      }
      part += m;
    }
    atomicAdd(&s_sum, part);
    atomicMax(&s_max, mxv);
  }
  __syncthreads();
  const bool narrow = s_sum + s_max < 0xFFFFFFFFull;

  const bool active = c < a.n_cand;
  int np = 0;
  uint32_t ml[DP], pp[DP], kk[DP];
  bool ok = false;
  if (active) {
    np = a.cand_np[c];
    ok = np >= 1 && np <= DP;
    uint32_t prev_ml = 0xFFFFFFFFu, prev_k = 0u;
#pragma unroll
    for (int j = 0; j < DP; ++j) {
      ml[j] = 0u;
      pp[j] = 1u;
      kk[j] = 0u;
      if (j < np) {
        const uint32_t k = a.cand[(size_t)c * HYD_MAX_PIPES + j];
        if (k < (uint32_t)a.n_schemes) {
          const uint32_t m = s_ml[k], p = s_pp[k];
          ok = ok && (m < prev_ml || (m == prev_ml && k >= prev_k)) && p >= 1u && p <= HYD_MAX_PP && m >= 1u;
          prev_ml = m;
          prev_k = k;
          ml[j] = m;
          pp[j] = p;
          kk[j] = k;
        } else {
          ok = false;
        }
      }
    }
    if (!ok) flag(a.status, HYD_F_NOT_CANONICAL);
  }
  const bool feasible = active && ok && B > 0 && sl[0] <= ml[0];
  const size_t row = (size_t)c * a.n_iter + t;
  uint8_t* prow = a.pipe + (size_t)c * a.n_total + tbase;
  if (feasible) {
    uint64_t lbv;
    if (narrow) small_dispatch<DP, uint32_t, T>(sl, sc, B, kp, np, ml, pp, kk, mem, rec, prow, lbv);
    else small_dispatch<DP, uint64_t, T>(sl, sc, B, kp, np, ml, pp, kk, mem, rec, prow, lbv);
    a.lb[row] = lbv;
  } else if (active) {
    for (int i = 0; i < B; ++i) prow[i] = 0xFF;
    a.lb[row] = ~0ull;
  }

  // ---- stage 2: the exact search of every pipeline, the lanes of a warp in step
  const int nw = (B + 31) >> 5;
  uint32_t ev = 0u;
  int j = 0;
  bool open = false, first = false, rerun = false;
  uint32_t wV = 0u, k = 0u;
  uint64_t msp = 0ull;
  Search s;
  s.have = false;
  while (true) {
    bool pending = false, write = false;
    uint32_t V = 0u;
    uint64_t thr = ~0ull;
    while (feasible && !pending && j < np) {
      if (!open) {  // open pipeline j
        uint32_t u = 0u, first_i = 0xFFFFFFFFu;
        for (int w = 0; w < nw; ++w) {
          const uint32_t bits = mem[j * kSmallWords + w];
          if (bits && first_i == 0xFFFFFFFFu) first_i = (uint32_t)(w * 32 + __ffs(bits) - 1);
          u += __popc(bits);
        }
        if (u == 0u) {  // empty pipeline: V = ptime = 0 (reading 12)
          rec.s(j) = 0u;
          rec.b(j) = 0ull;
          ++j;
          continue;
        }
        k = a.cand[(size_t)c * HYD_MAX_PIPES + j];
        const uint32_t tm = sc[first_i * kp + k];  // T(longest member): it is the first in sorted order
        s.M = s_ml[k];
        s.P = s_pp[k];
        s.UL = s_ul[k];
        s.U = u;
        s.S = rec.s(j);
        s.sumT = rec.b(j) - (unsigned long long)tm * (s.P - 1u);
        s.tau_max = tm;
        search_init(s);
        open = true;
        first = true;
        rerun = false;
        wV = 0u;
      }
      if (!rerun) {
        V = search_next(s);
        if (V) {
          thr = first ? ~0ull : search_thr_approx(s, V);
          write = first;
          pending = true;
        } else if (s.have && s.vbest != wV) {  // the winner's mb was not written by the first run
          rerun = true;
          V = s.vbest;
          write = true;
          pending = true;
        }
      }
      if (!pending) {  // pipeline j done
        rec.s(j) = s.have ? s.vbest : 0u;
        rec.b(j) = s.have ? s.best : 0ull;
        msp = max(msp, (uint64_t)(s.have ? s.best : 0ull));
        open = false;
        rerun = false;
        ++j;
      }
    }
    if (!__any_sync(HYD_FULL, pending)) break;
    const bool fast = pending && V <= 16u && s.M < 0x80000000u;
    const bool wide = __any_sync(HYD_FULL, fast && s.sumT >= (1ull << 27));  // u64 keys for the warp
    const uint32_t nmax = __reduce_max_sync(HYD_FULL, fast ? V : 0u);
    bool okr = false;
    uint64_t mx = 0ull;
    if (fast) {
      const uint32_t* mw = mem + j * kSmallWords;
      if (!wide) {
        if (nmax <= 4u) okr = run_keys<4, uint32_t>(mw, nw, V, s.M, k, thr, write, mbs, sl, sc, kp, mx, ev);
        else if (nmax <= 8u) okr = run_keys<8, uint32_t>(mw, nw, V, s.M, k, thr, write, mbs, sl, sc, kp, mx, ev);
        else okr = run_keys<16, uint32_t>(mw, nw, V, s.M, k, thr, write, mbs, sl, sc, kp, mx, ev);
      } else {
        if (nmax <= 4u) okr = run_keys<4, uint64_t>(mw, nw, V, s.M, k, thr, write, mbs, sl, sc, kp, mx, ev);
        else if (nmax <= 8u) okr = run_keys<8, uint64_t>(mw, nw, V, s.M, k, thr, write, mbs, sl, sc, kp, mx, ev);
        else okr = run_keys<16, uint64_t>(mw, nw, V, s.M, k, thr, write, mbs, sl, sc, kp, mx, ev);
      }
    } else if (pending) {
      okr = run_generic(mem + j * kSmallWords, nw, V, s.M, k, thr, write, mbs, sl, sc, kp, mx, ev);
    }
    if (pending && !rerun) {
      if (okr && first) wV = V;
      first = false;
      if (okr && search_improves(s, V, mx)) search_take(s, V, mx);
    }
  }

  // ---- outputs: mb row (staged), v / ptime rows, makespan
  if (active) {
    uint16_t* mrow = a.mb + (size_t)c * a.n_total + tbase;
    if (feasible) {
      for (int i = 0; i < B; ++i) mrow[i] = mbs[i];
    } else {
      for (int i = 0; i < B; ++i) mrow[i] = 0xFFFF;
    }
    uint32_t vw[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int j0 = 2 * q, j1 = 2 * q + 1;
      const uint32_t v0 = (feasible && j0 < np && j0 < DP) ? rec.s(j0 < DP ? j0 : 0) : 0u;
      const uint32_t v1 = (feasible && j1 < np && j1 < DP) ? rec.s(j1 < DP ? j1 : 0) : 0u;
      vw[q] = (v0 & 0xFFFFu) | (v1 << 16);
    }
    uint4* vrow = reinterpret_cast<uint4*>(a.v + row * HYD_MAX_PIPES);
#pragma unroll
    for (int q = 0; q < 4; ++q) vrow[q] = make_uint4(vw[4 * q], vw[4 * q + 1], vw[4 * q + 2], vw[4 * q + 3]);
    ulonglong2* prow2 = reinterpret_cast<ulonglong2*>(a.ptime + row * HYD_MAX_PIPES);
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int j0 = 2 * q, j1 = 2 * q + 1;
      const unsigned long long p0 = (feasible && j0 < np && j0 < DP) ? rec.b(j0 < DP ? j0 : 0) : 0ull;
      const unsigned long long p1 = (feasible && j1 < np && j1 < DP) ? rec.b(j1 < DP ? j1 : 0) : 0ull;
      prow2[q] = make_ulonglong2(p0, p1);
    }
    a.makespan[(size_t)t * a.n_cand + c] = feasible ? msp : ~0ull;
  }
  if (a.evals) {
    const unsigned long long tot = __reduce_add_sync(HYD_FULL, ev);
    if (lane == 0 && tot) atomicAdd(a.evals, tot);
  }
}

size_t small_smem(int dp, int k_pad, int T) {
  return (size_t)T * dp * 8 + (size_t)HYD_SMALL_MAX_BATCH * 4 * (1 + (size_t)k_pad) +
         (size_t)T * dp * kSmallWords * 4 + (size_t)T * dp * 4 + (size_t)T * HYD_SMALL_MAX_BATCH;
}

template <int DP, int T>
static cudaError_t launch_small_t(int n_cand, int n_iter, cudaStream_t s, const SmallArgs& a) {
  const size_t smem = small_smem(DP, a.k_pad, T);
  cudaError_t e = cudaFuncSetAttribute(k_assign_small<DP, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const dim3 grid((n_cand + T - 1) / T, n_iter);
  k_assign_small<DP, T><<<grid, T, smem, s>>>(a);
  return cudaGetLastError();
}

template <int DP>
static cudaError_t launch_small_dp(int n_cand, int n_iter, cudaStream_t s, const SmallArgs& a) {
  return n_cand <= 32 ? launch_small_t<DP, 32>(n_cand, n_iter, s, a) : launch_small_t<DP, kSmallThreads>(n_cand, n_iter, s, a);
}

int launch_small(const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch, const uint32_t* off,
                 size_t n_total, int k_pad, const hyd_scheme* schemes, int n_schemes, const uint8_t* cand,
                 const uint8_t* cand_np, int n_cand, int max_np, uint8_t* pipe, uint64_t* lb, uint16_t* mb,
                 uint16_t* v, uint64_t* ptime, uint64_t* makespan, uint32_t* status, void* ws, cudaStream_t s) {
  if (n_iter == 0 || n_cand == 0) return HYD_OK;
  SmallArgs a;
  a.sorted_len = sorted_len;
  a.cost = cost;
  a.n_iter = n_iter;
  a.batch = batch;
  a.k_pad = k_pad;
  a.off = off;
  a.n_total = n_total;
  a.schemes = schemes;
  a.n_schemes = n_schemes;
  a.cand = cand;
  a.cand_np = cand_np;
  a.n_cand = n_cand;
  a.pipe = pipe;
  a.lb = lb;
  a.mb = mb;
  a.v = v;
  a.ptime = ptime;
  a.makespan = makespan;
  a.status = status;
  a.evals = reinterpret_cast<unsigned long long*>(ws);
  if (ws) {
    const cudaError_t e = cudaMemsetAsync(ws, 0, 8, s);
    if (e != cudaSuccess) return record_cuda_error(e);
  }
  cudaError_t e;
  if (max_np <= 2) e = launch_small_dp<2>(n_cand, n_iter, s, a);
  else if (max_np <= 4) e = launch_small_dp<4>(n_cand, n_iter, s, a);
  else if (max_np <= 8) e = launch_small_dp<8>(n_cand, n_iter, s, a);
  else e = launch_small_dp<16>(n_cand, n_iter, s, a);
  note_launch();
  return e == cudaSuccess ? HYD_OK : record_cuda_error(e);
}

}  // namespace hyd
