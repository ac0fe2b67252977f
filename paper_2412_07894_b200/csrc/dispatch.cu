// dispatch.cu -- a3: stage 1 sequence dispatching across pipelines (§6.2).
//
// One thread per (candidate c, iteration t).  A CTA covers `ct` candidates x `tt`
// iterations (ct*tt <= 128), so the threads of a warp share the iteration's sorted
// lengths and cost rows; when they fit, those rows are staged in shared memory once per
// CTA (16-byte copies) and each sequence step reads one <= 256 B smem row.
//
// Per pipeline j the register state is base_j = C_j + E_j (Alg. 1's accumulators,
// P:1136-1137) and mult_j = PP_j while the pipeline is empty, 1 afterwards.  Because the
// sequences arrive longest first, the first one a pipeline receives fixes its extra term
// E_j = T(l_max,P_j)(PP_j-1) (Eq. 2), so the candidate load of every feasible j is
//   new_j = base_j + tau * mult_j      (= C_j + tau + e_j of SURVEY §8(c) step 4)
// one IMAD; j* = argmin (new_j, j) over MaxLen_j >= l_i (J_i); base_j* = new_j*.
// Per-pipeline statistics for the packing stage: S_j in a shared-memory column indexed by j*
// (one LDS/STS per sequence); U_j and tau_max,j from the membership bitmap words, which are
// flushed every 32 sequences.
// A per-CTA bound on every load picks the arithmetic: packed u32 keys (packed_run, MODE 0
// kernel) when loads < 2^(31 - log2 DP), else u32 sums (dispatch_run, MODE 1 kernel) when loads
// < 2^32, else u64 sums (MODE 2 kernel) -- three kernels so each carries only its own registers.
// Outputs: pipe[c][t][i] (4 decisions per u32 store), lb[c][t] = max_j base_j, stats.
#include <type_traits>

#include "hyd_internal.cuh"

namespace hyd {

constexpr int kDispatchThreads = 128;

// staged words: [tt][B] lengths + costs (rows [tt][B][k_pad], or transposed [tt][k_pad][B | 1])
__host__ __device__ inline size_t dispatch_stage_words(int tt, int B, int k_pad) {
  return (size_t)tt * B + (size_t)tt * k_pad * (size_t)(B | 1);
}

// One sequence step: candidate loads, argmin (new_j, j), branch-free update of pipeline j*.
// FEAS: test MaxLen_j >= l (only needed while l exceeds the smallest MaxLen of the candidate;
// lengths are sorted descending, so the tail of the batch skips the test).  EMPTY: some
// pipeline of the warp may still be empty (multiplier PP_j); once none is, every used mult_j is
// 1 and stays 1, so the step skips their updates.  The decision j* is shifted into SH bit
// planes (plane_b bit q = bit b of the chunk's q-th decision), expanded into membership words
// once per 32-step chunk (chunk_flush).
template <int DP, typename TT, bool FEAS, bool EMPTY, int SH>
__device__ __forceinline__ uint32_t dispatch_step(uint32_t l, const uint32_t* __restrict__ crow,
                                                  bool staged, const uint32_t (&ml)[DP],
                                                  const uint32_t (&kk)[DP], TT (&base)[DP],
                                                  uint32_t (&mult)[DP], uint32_t (&plane)[SH]) {
  TT best = (TT)~(TT)0;
  uint32_t bj = 0u;
#pragma unroll
  for (int j = 0; j < DP; ++j) {
    const uint32_t tau = staged ? crow[kk[j]] : __ldg(crow + kk[j]);
    const TT nw = base[j] + (TT)tau * (TT)mult[j];
    if ((!FEAS || l <= ml[j]) && nw < best) {
      best = nw;
      bj = (uint32_t)j;
    }
  }
  // branch-free update of pipeline bj (a switch here compiles to a divergent jump table)
#pragma unroll
  for (int j = 0; j < DP; ++j) {
    const bool hit = (uint32_t)j == bj;
    base[j] = hit ? best : base[j];
    if (EMPTY) mult[j] = hit ? 1u : mult[j];
  }
#pragma unroll
  for (int b = 0; b < SH; ++b) plane[b] = __funnelshift_r(plane[b], bj >> b, 1);
  return bj;
}

template <int DP>
struct DispCfg {
  static constexpr int SH = DP <= 2 ? 1 : DP <= 4 ? 2 : DP <= 8 ? 3 : DP <= 16 ? 4 : 5;
};

// true while some used pipeline of some thread of the warp is still empty (mult_j = PP_j > 1)
template <int DP>
__device__ __forceinline__ bool warp_any_empty(const uint32_t (&mult)[DP], int np, unsigned amask) {
  bool e = false;
#pragma unroll
  for (int j = 0; j < DP; ++j) e |= j < np && mult[j] > 1u;
  return __any_sync(amask, e);
}

// End of a chunk of n <= 32 decisions starting at sequence i0: one membership word per pipeline
// (word j = the decisions equal to j, from the bit planes) and cf_j = U_j << 16 | first member + 1.
template <int DP, int SH>
__device__ __forceinline__ void chunk_flush(uint32_t (&plane)[SH], int n, int i0, int np, int mstride,
                                            uint32_t* __restrict__ mbits, uint32_t (&cf)[DP]) {
  if (n < 32) {
#pragma unroll
    for (int b = 0; b < SH; ++b) plane[b] >>= 32 - n;
  }
  const uint32_t valid = n < 32 ? (1u << n) - 1u : 0xFFFFFFFFu;
#pragma unroll
  for (int j = 0; j < DP; ++j) {
    if (j < np) {
      uint32_t wj = valid;
#pragma unroll
      for (int b = 0; b < SH; ++b) wj &= ((j >> b) & 1) ? plane[b] : ~plane[b];
      HYD_CHECK(j < mstride);
      mbits[(size_t)(i0 >> 5) * mstride + j] = wj;
      const uint32_t f = (cf[j] & 0xFFFFu) == 0u && wj != 0u ? (uint32_t)i0 + __ffs(wj) : 0u;
      cf[j] += (__popc(wj) << 16) + f;
    }
  }
#pragma unroll
  for (int b = 0; b < SH; ++b) plane[b] = 0u;
}

// one 32-step chunk of a thread's decisions: steps i0 .. i0 + n - 1 (ls / crow_of read the
// sequence's length and cost row)
template <int DP, typename TT, bool EMPTY, typename LenF, typename RowF>
__device__ __forceinline__ void dispatch_chunk(int i0, int n, bool staged, uint32_t ml_min,
                                               const uint32_t (&ml)[DP], const uint32_t (&kk)[DP],
                                               TT (&base)[DP], uint32_t (&mult)[DP],
                                               uint32_t (&plane)[DispCfg<DP>::SH], LenF&& len_of,
                                               RowF&& row_of, uint8_t* __restrict__ prow, bool words,
                                               unsigned long long* s_sum, uint32_t& pbj, uint32_t& pl) {
  constexpr int SH = DispCfg<DP>::SH;
  uint32_t word = 0u;
  for (int q = 0; q < n; ++q) {
    const int i = i0 + q;
    const unsigned long long sold = s_sum[pbj * kDispatchThreads];
    const uint32_t l = len_of(q);
    const uint32_t* crow = row_of(q);
    const uint32_t bj = l > ml_min ? dispatch_step<DP, TT, true, EMPTY, SH>(l, crow, staged, ml, kk, base, mult, plane)
                                   : dispatch_step<DP, TT, false, EMPTY, SH>(l, crow, staged, ml, kk, base, mult, plane);
    s_sum[pbj * kDispatchThreads] = sold + pl;  // S_j column of this thread, one step late
    pbj = bj;
    pl = l;
    if (words) {
      word |= bj << (8 * (i & 3));
      if ((i & 3) == 3) {
        *reinterpret_cast<uint32_t*>(prow + (i & ~3)) = word;
        word = 0u;
      }
    } else {
      prow[i] = (uint8_t)bj;
    }
  }
}

template <int DP, typename TT>
__device__ __forceinline__ void dispatch_run(const uint32_t* __restrict__ sl,
                                             const uint32_t* __restrict__ cs, bool staged, int B,
                                             int k_pad, const uint32_t (&ml)[DP],
                                             const uint32_t (&pp)[DP], const uint32_t (&kk)[DP],
                                             uint8_t* __restrict__ prow, unsigned long long* s_sum,
                                             uint32_t* __restrict__ mbits, int np, int mstride,
                                             uint64_t& lb_out, TT (&base)[DP],
                                             uint32_t (&cf)[DP]) {
  constexpr int SH = DispCfg<DP>::SH;
  const unsigned amask = __activemask();
  uint32_t mult[DP], plane[SH];
  uint32_t ml_min = 0xFFFFFFFFu;
#pragma unroll
  for (int j = 0; j < DP; ++j) {  // unused slots: base = max, mult = 0 -> never strictly best
    base[j] = j < np ? (TT)0 : (TT)~(TT)0;
    mult[j] = j < np ? pp[j] : 0u;
    cf[j] = 0u;
    if (j < np) ml_min = min(ml_min, ml[j]);
  }
#pragma unroll
  for (int b = 0; b < SH; ++b) plane[b] = 0u;
  const bool words = (B & 3) == 0 && ((size_t)prow & 3) == 0;
  uint32_t pbj = 0u, pl = 0u;  // S_j one step late (as in packed_step)
  for (int i0 = 0; i0 < B; i0 += 32) {
    const int n = min(32, B - i0);
    auto lf = [&](int q) { return sl[i0 + q]; };
    auto rf = [&](int q) { return cs + (size_t)(i0 + q) * k_pad; };
    if (warp_any_empty<DP>(mult, np, amask))
      dispatch_chunk<DP, TT, true>(i0, n, staged, ml_min, ml, kk, base, mult, plane, lf, rf, prow, words, s_sum, pbj, pl);
    else
      dispatch_chunk<DP, TT, false>(i0, n, staged, ml_min, ml, kk, base, mult, plane, lf, rf, prow, words, s_sum, pbj, pl);
    chunk_flush<DP, SH>(plane, n, i0, np, mstride, mbits, cf);
  }
  s_sum[pbj * kDispatchThreads] += pl;  // the last decision's S_j
  uint64_t m = 0ull;
#pragma unroll
  for (int j = 0; j < DP; ++j)
    if (j < np) m = max(m, (uint64_t)base[j]);
  lb_out = m;
}

// dispatch_run for iterations too long to stage whole (config 5: 8192 sequences x 20 schemes):
// the CTA's threads (one iteration, tt = 1) copy windows of kDispatchWin sequences' lengths and
// cost rows into shared memory together, then each live thread runs its steps from there, so
// every cost read is a shared-memory load instead of an L2 round trip.  All threads of the CTA
// take part in the copies and barriers; `live` threads (a feasible candidate) also decide.
constexpr int kDispatchWin = 512;  // a multiple of the 32-step chunk

template <int DP, typename TT>
__device__ __forceinline__ void dispatch_run_win(bool live, const uint32_t* __restrict__ g_sl,
                                                 const uint32_t* __restrict__ g_cs, uint32_t* __restrict__ wsm,
                                                 int B, int k_pad, const uint32_t (&ml)[DP],
                                                 const uint32_t (&pp)[DP], const uint32_t (&kk)[DP],
                                                 uint8_t* __restrict__ prow, unsigned long long* s_sum,
                                                 uint32_t* __restrict__ mbits, int np, int mstride,
                                                 uint64_t& lb_out, TT (&base)[DP], uint32_t (&cf)[DP]) {
  constexpr int SH = DispCfg<DP>::SH;
  const int tid = threadIdx.x;
  const unsigned amask = __ballot_sync(HYD_FULL, live);
  uint32_t mult[DP], plane[SH];
  uint32_t ml_min = 0xFFFFFFFFu;
#pragma unroll
  for (int j = 0; j < DP; ++j) {  // unused slots: base = max, mult = 0 -> never strictly best
    base[j] = j < np ? (TT)0 : (TT)~(TT)0;
    mult[j] = j < np ? pp[j] : 0u;
    cf[j] = 0u;
    if (j < np) ml_min = min(ml_min, ml[j]);
  }
#pragma unroll
  for (int b = 0; b < SH; ++b) plane[b] = 0u;
  const bool words = (B & 3) == 0 && ((size_t)prow & 3) == 0;
  uint32_t pbj = 0u, pl = 0u;  // S_j one step late (as in packed_step)
  uint32_t* wl = wsm;                 // [kDispatchWin] lengths
  uint32_t* wc = wsm + kDispatchWin;  // [kDispatchWin][k_pad] cost rows
  const bool vec = (((size_t)g_cs & 15) == 0) && (k_pad & 3) == 0;
  for (int w0 = 0; w0 < B; w0 += kDispatchWin) {
    const int n = min(kDispatchWin, B - w0);
    __syncthreads();  // the previous window is consumed
    for (int e = tid; e < n; e += kDispatchThreads) wl[e] = __ldg(g_sl + w0 + e);
    if (vec) {
      const uint4* src = reinterpret_cast<const uint4*>(g_cs + (size_t)w0 * k_pad);
      uint4* dst = reinterpret_cast<uint4*>(wc);
      for (int e = tid; e < n * k_pad / 4; e += kDispatchThreads) dst[e] = __ldg(src + e);
    } else {
      for (int e = tid; e < n * k_pad; e += kDispatchThreads) wc[e] = __ldg(g_cs + (size_t)w0 * k_pad + e);
    }
    __syncthreads();
    if (!live) continue;
    for (int q0 = 0; q0 < n; q0 += 32) {
      const int nq = min(32, n - q0);
      auto lf = [&](int q) { return wl[q0 + q]; };
      auto rf = [&](int q) { return wc + (q0 + q) * k_pad; };
      if (warp_any_empty<DP>(mult, np, amask))
        dispatch_chunk<DP, TT, true>(w0 + q0, nq, true, ml_min, ml, kk, base, mult, plane, lf, rf, prow, words, s_sum, pbj,
                                     pl);
      else
        dispatch_chunk<DP, TT, false>(w0 + q0, nq, true, ml_min, ml, kk, base, mult, plane, lf, rf, prow, words, s_sum,
                                      pbj, pl);
      chunk_flush<DP, SH>(plane, nq, w0 + q0, np, mstride, mbits, cf);
    }
  }
  if (!live) return;
  s_sum[pbj * kDispatchThreads] += pl;  // the last decision's S_j
  uint64_t m = 0ull;
#pragma unroll
  for (int j = 0; j < DP; ++j)
    if (j < np) m = max(m, (uint64_t)base[j]);
  lb_out = m;
}

// Packed-key run (MODE 0: every load of the CTA < 2^(31 - SH)).  key_j = (C_j + E_j) << SH | j,
// so a candidate key is one IMAD, the argmin is a VIMNMX tree with no index bookkeeping and the
// winner's new key is the minimum itself.  Same decisions as dispatch_run, with a steady-state
// step of about half its instructions:
//  * feasibility is folded into the keys: a pipeline with MaxLen_j < l carries bit 31 in key_j
//    (it never wins while a feasible pipeline exists, and j = 0 always is), cleared on the rare
//    step where l drops to its MaxLen -- the canonical order makes the infeasible set a suffix,
//    so one compare per step against the largest pending MaxLen suffices;
//  * the empty-pipeline multiplier PP_j (Eq. 2's first-member term) matters only until every
//    pipeline of the thread holds a sequence; 32-step chunks run a multiplier-free step once the
//    whole warp is past that point (warp vote: no divergence);
//  * membership is kept as log2(DP) bit planes of j* (plane_b bit q = bit b of the q-th
//    decision), expanded into per-pipeline words once per chunk; the chunk's 32 decision bytes
//    leave as two 16-byte stores (one full sector);
//  * staged cost rows are transposed to [scheme][sequence] (odd row stride: no bank conflicts),
//    so a pipeline's costs for 4 consecutive sequences are one base register + immediates.
template <int DP, bool EMPTY>
__device__ __forceinline__ uint32_t packed_pick(const uint32_t (&tau)[DP], uint32_t (&key)[DP],
                                                uint32_t (&mults)[DP], uint32_t one_sh) {
  uint32_t m[DP];
#pragma unroll
  for (int j = 0; j < DP; ++j) m[j] = tau[j] * (EMPTY ? mults[j] : one_sh) + key[j];
  const uint32_t mk = min_tree3<DP>(m);
  const uint32_t bj = mk & (uint32_t)(DP - 1);
#pragma unroll
  for (int j = 0; j < DP; ++j) {
    const bool hit = (uint32_t)j == bj;
    key[j] = hit ? mk : key[j];
    if (EMPTY) mults[j] = hit ? one_sh : mults[j];
  }
  return bj;
}

// one decision: feasibility release (EMPTY phase only), pick, plane bits, S_j
template <int DP, int SH, bool EMPTY>
__device__ __forceinline__ uint32_t packed_step(uint32_t l, const uint32_t (&tau)[DP],
                                                uint32_t (&key)[DP], uint32_t (&mults)[DP],
                                                const uint32_t (&ml)[DP], int np, uint32_t& pend,
                                                uint32_t (&plane)[SH],
                                                unsigned long long* s_sum, uint32_t& pbj, uint32_t& pl) {
  // S_j one step late: the previous decision's column is loaded before this step's pick, so the
  // load's latency hides under it (same thread, program order: a repeat of the column is safe)
  const unsigned long long sold = s_sum[pbj * kDispatchThreads];
  if (EMPTY && l <= pend) {  // rare: pipelines become feasible as l drops to their MaxLen
    uint32_t np2 = 0u;
#pragma unroll
    for (int j = 0; j < DP; ++j) {
      if (j < np && (key[j] >> 31) != 0u) {
        if (ml[j] >= l) key[j] &= 0x7FFFFFFFu;
        else np2 = max(np2, ml[j]);
      }
    }
    pend = np2;
  }
  const uint32_t bj = packed_pick<DP, EMPTY>(tau, key, mults, 1u << SH);
#pragma unroll  // shift bit b of j* in from the top: after the chunk, bit q = decision q
  for (int b = 0; b < SH; ++b) plane[b] = __funnelshift_r(plane[b], bj >> b, 1);
  s_sum[pbj * kDispatchThreads] = sold + pl;  // S_j column of this thread
  pbj = bj;
  pl = l;
  return bj;
}

template <int OFF>
__device__ __forceinline__ uint32_t lds_off(uint32_t addr) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1+%2];" : "=r"(v) : "r"(addr), "n"(OFF));
  return v;
}

// TRANS: cost staged in smem as [lt][k][Bp] (cost(i, k) at ct[k * Bp + i] for this thread's lt);
// else global rows [t][i][k_pad].
template <int DP, bool TRANS>
__device__ __forceinline__ void packed_run(const uint32_t* __restrict__ sl,
                                           const uint32_t* __restrict__ cst, int B, int stride,
                                           const uint32_t (&ml)[DP], const uint32_t (&pp)[DP],
                                           const uint32_t (&kk)[DP], uint8_t* __restrict__ prow,
                                           unsigned long long* s_sum, uint32_t* __restrict__ mbits,
                                           int np, int mstride, uint64_t& lb_out,
                                           uint32_t (&base)[DP], uint32_t (&cf)[DP],
                                           unsigned amask) {
  constexpr int SH = DP <= 2 ? 1 : DP <= 4 ? 2 : DP <= 8 ? 3 : DP <= 16 ? 4 : 5;
  const uint32_t one_sh = 1u << SH;
  const uint32_t l0 = sl[0];
  uint32_t key[DP], mults[DP];
  uint32_t pend = 0u;  // largest MaxLen among still-infeasible pipelines (0: none)
  const uint32_t* pj[DP];  // TRANS: row of pipeline j's scheme; else column offset kk_j
#pragma unroll
  for (int j = 0; j < DP; ++j) {
    const bool used = j < np;
    const bool feas = used && ml[j] >= l0;
    key[j] = !used ? 0x7FFFFFFFu : feas ? (uint32_t)j : (0x80000000u | (uint32_t)j);
    mults[j] = used ? pp[j] << SH : 0u;
    if (used && !feas) pend = max(pend, ml[j]);
    cf[j] = 0u;
    pj[j] = TRANS ? cst + (size_t)kk[j] * stride : cst + kk[j];
  }
  uint32_t pa[DP];  // TRANS: the rows' shared-window addresses
#pragma unroll
  for (int j = 0; j < DP; ++j) pa[j] = TRANS ? (uint32_t)__cvta_generic_to_shared(pj[j]) : 0u;
  const bool full_sectors = (B & 31) == 0 && ((size_t)prow & 15) == 0;
  uint32_t pbj = 0u, pl = 0u;  // the decision whose S_j update is pending
  for (int i0 = 0; i0 < B; i0 += 32) {
    const int n = min(32, B - i0);
    bool empty = false;
#pragma unroll
    for (int j = 0; j < DP; ++j) empty |= j < np && (key[j] < one_sh || (key[j] >> 31) != 0u);
    const bool warp_empty = __any_sync(amask, empty);
    uint32_t plane[SH];
#pragma unroll
    for (int b = 0; b < SH; ++b) plane[b] = 0u;
    if (TRANS) {  // groups of 4 steps (uniform batches: B % 4 == 0), then the ragged remainder
      const int n4 = n & ~3;
      for (int g = 0; g < n4; g += 4) {
        const int i = i0 + g;
        const uint4 l4 = *reinterpret_cast<const uint4*>(sl + i);
        const uint32_t lq[4] = {l4.x, l4.y, l4.z, l4.w};
        uint32_t qa[DP];  // shared addresses of row j at sequence i: the 4 steps use immediate offsets
#pragma unroll
        for (int j = 0; j < DP; ++j) qa[j] = pa[j] + 4u * (uint32_t)i;
        auto step = [&](auto uc) {
          constexpr int U = decltype(uc)::value;
          uint32_t tau[DP];
#pragma unroll
          for (int j = 0; j < DP; ++j) tau[j] = lds_off<4 * U>(qa[j]);
          if (warp_empty)
            packed_step<DP, SH, true>(lq[U], tau, key, mults, ml, np, pend, plane, s_sum, pbj, pl);
          else
            packed_step<DP, SH, false>(lq[U], tau, key, mults, ml, np, pend, plane, s_sum, pbj, pl);
        };
        step(std::integral_constant<int, 0>{});
        step(std::integral_constant<int, 1>{});
        step(std::integral_constant<int, 2>{});
        step(std::integral_constant<int, 3>{});
      }
      for (int q = n4; q < n; ++q) {
        const int i = i0 + q;
        uint32_t tau[DP];
#pragma unroll
        for (int j = 0; j < DP; ++j) tau[j] = pj[j][i];
        if (warp_empty)
          packed_step<DP, SH, true>(sl[i], tau, key, mults, ml, np, pend, plane, s_sum, pbj, pl);
        else
          packed_step<DP, SH, false>(sl[i], tau, key, mults, ml, np, pend, plane, s_sum, pbj, pl);
      }
    } else {
      for (int q = 0; q < n; ++q) {
        const int i = i0 + q;
        const uint32_t l = sl[i];
        uint32_t tau[DP];
#pragma unroll
        for (int j = 0; j < DP; ++j) tau[j] = __ldg(pj[j] + (size_t)i * stride);
        if (warp_empty)
          packed_step<DP, SH, true>(l, tau, key, mults, ml, np, pend, plane, s_sum, pbj, pl);
        else
          packed_step<DP, SH, false>(l, tau, key, mults, ml, np, pend, plane, s_sum, pbj, pl);
      }
    }
    if (n < 32) {
#pragma unroll
      for (int b = 0; b < SH; ++b) plane[b] >>= 32 - n;
    }
    // decisions of the chunk: byte q = sum_b bit q of plane_b << b
    uint32_t wd[8];
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      uint32_t x = 0u;
#pragma unroll
      for (int b = 0; b < SH; ++b)
        x |= ((((plane[b] >> (4 * w)) & 0xFu) * 0x00204081u) & 0x01010101u) << b;
      wd[w] = x;
    }
    if (full_sectors) {
      uint4* dst = reinterpret_cast<uint4*>(prow + i0);
      dst[0] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
      dst[1] = make_uint4(wd[4], wd[5], wd[6], wd[7]);
    } else {
#pragma unroll
      for (int q = 0; q < 32; ++q)
        if (q < n) prow[i0 + q] = (uint8_t)(wd[q >> 2] >> (8 * (q & 3)));
    }
    // membership words (word-major: the chunk's words of all pipelines are contiguous, so with
    // mstride == DP they leave as full 32-byte sectors); U_j and first member in cf_j
    const uint32_t valid = n == 32 ? 0xFFFFFFFFu : (1u << n) - 1u;
    uint32_t xw[DP];
#pragma unroll
    for (int j = 0; j < DP; ++j) {
      uint32_t x = j < np ? valid : 0u;
#pragma unroll
      for (int b = 0; b < SH; ++b) x &= ((j >> b) & 1) ? plane[b] : ~plane[b];
      xw[j] = x;
      const uint32_t f = (cf[j] & 0xFFFFu) == 0u && x != 0u ? (uint32_t)i0 + __ffs(x) : 0u;
      cf[j] += (__popc(x) << 16) + f;
    }
    uint32_t* mrow = mbits + (size_t)(i0 >> 5) * mstride;
    if (DP >= 4 && mstride == DP) {
#pragma unroll
      for (int j = 0; j < DP; j += 4)
        *reinterpret_cast<uint4*>(mrow + j) = make_uint4(xw[j], xw[j + 1], xw[j + 2], xw[j + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < DP; ++j)
        if (j < np) mrow[j] = xw[j];
    }
  }
  s_sum[pbj * kDispatchThreads] += pl;  // the last decision's S_j
  uint64_t mx = 0ull;
#pragma unroll
  for (int j = 0; j < DP; ++j) {
    base[j] = j < np ? (key[j] & 0x7FFFFFFFu) >> SH : 0xFFFFFFFFu;  // never-feasible: 0
    if (j < np) mx = max(mx, (uint64_t)base[j]);
  }
  lb_out = mx;
}

// Per-iteration bound[t] = sum_i max_k tau_ik + max_ik tau_ik (PPmax - 1): no C_j + E_j (and no
// candidate load C_j + tau + e_j) of iteration t can exceed it.  One CTA per iteration.
__global__ void __launch_bounds__(256)
    k_iter_bound(const uint32_t* __restrict__ cost, int batch, const uint32_t* __restrict__ off,
                 int k_pad, const hyd_scheme* __restrict__ schemes, int n_schemes,
                 uint64_t* __restrict__ bound) {
  __shared__ unsigned long long s_part[8];
  __shared__ uint32_t s_top;
  const int t = blockIdx.x, tid = threadIdx.x;
  const uint32_t* c = cost + geo_base(off, batch, t) * k_pad;
  const int bt = geo_bt(off, batch, t);
  unsigned long long sum = 0ull;
  uint32_t top = 0u;
  for (int i = tid; i < bt; i += 256) {
    uint32_t m = 0u;
    for (int k = 0; k < n_schemes; ++k) m = max(m, __ldg(c + (size_t)i * k_pad + k));
    sum += m;
    top = max(top, m);
  }
  for (int o = 16; o > 0; o >>= 1) {
    sum += __shfl_xor_sync(HYD_FULL, sum, o);
    top = max(top, __shfl_xor_sync(HYD_FULL, top, o));
  }
  if (tid == 0) s_top = 0u;
  __syncthreads();
  if ((tid & 31) == 0) {
    s_part[tid >> 5] = sum;
    atomicMax(&s_top, top);
  }
  __syncthreads();
  if (tid == 0) {
    unsigned long long b = 0ull;
    for (int w = 0; w < 8; ++w) b += s_part[w];
    uint32_t ppmax = 1u;
    for (int k = 0; k < n_schemes; ++k) ppmax = max(ppmax, schemes[k].pp);
    bound[t] = b + (unsigned long long)s_top * (ppmax - 1u);
  }
}

int launch_iter_bound(const uint32_t* cost, int n_iter, int batch, const uint32_t* off, int k_pad,
                      const hyd_scheme* schemes, int n_schemes, uint64_t* bound, cudaStream_t s) {
  if (n_iter == 0) return HYD_OK;
  k_iter_bound<<<n_iter, 256, 0, s>>>(cost, batch, off, k_pad, schemes, n_schemes, bound);
  note_launch();
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HYD_OK : record_cuda_error(e);
}

// MODE 0: CTAs whose load bound admits packed keys; MODE 1: u32 sums; MODE 2: u64 sums.  All
// kernels are launched; each reads the same per-iteration bounds and leaves the other's CTAs
// alone (before staging anything), so the common packed case runs with the packed kernel's
// smaller register footprint.
template <int DP, bool STAGED, int MODE>
__global__ void __launch_bounds__(kDispatchThreads, (MODE == 0 && DP == 8) ? 5 : MODE == 1 ? 3 : 1)
    k_dispatch(const uint32_t* __restrict__ sorted_len, const uint32_t* __restrict__ cost,
               int n_iter, int batch, const uint32_t* __restrict__ off, size_t n_total, int k_pad,
               const hyd_scheme* __restrict__ schemes,
               int n_schemes, const uint8_t* __restrict__ cand, const uint8_t* __restrict__ cand_np,
               int n_cand, int max_np, int ct, int tt, uint8_t* __restrict__ pipe,
               uint64_t* __restrict__ lb, hyd_pipe_stats* __restrict__ stats,
               uint32_t* __restrict__ members, uint32_t* __restrict__ status,
               const uint64_t* __restrict__ bounds) {
  extern __shared__ __align__(16) uint32_t sm[];
  // dynamic smem: [stage if STAGED] [s_sum u64 columns]; stage = [tt][B] lengths, then the
  // costs: MODE 1 as global rows [tt][B][k_pad]; MODE 0 transposed [tt][k_pad][Bp], Bp = B | 1
  constexpr bool TRANS = STAGED && MODE == 0;
  // general sums on an iteration too long to stage: window staging (one iteration per CTA)
  constexpr bool WIN = !STAGED && MODE != 0;
  // ragged batches (off != nullptr) run with tt = 1: B = this iteration's sequences
  const int B = off ? geo_bt(off, batch, blockIdx.y) : batch;
  const int Bp = B | 1;
  const size_t stage_words =
      STAGED ? dispatch_stage_words(tt, batch, k_pad) : WIN ? (size_t)kDispatchWin * (1 + k_pad) : 0;
  unsigned long long* s_sum = reinterpret_cast<unsigned long long*>(sm + ((stage_words + 3) & ~(size_t)3));
  const int tid = threadIdx.x;
  const int c0 = blockIdx.x * ct, t0 = blockIdx.y * tt;
  const int ntt = min(tt, n_iter - t0);
  // every load of the CTA's threads is below the largest bound of its iterations
  unsigned long long bound = 0ull;
  for (int lt = 0; lt < ntt; ++lt) bound = max(bound, (unsigned long long)bounds[t0 + lt]);
  const bool narrow = bound < 0xFFFFFFFFull;
  constexpr int SHK = DP <= 2 ? 1 : DP <= 4 ? 2 : DP <= 8 ? 3 : DP <= 16 ? 4 : 5;
  const bool packed = bound < (1ull << (31 - SHK));  // keys (load << SHK | j) stay below 2^31
  if (MODE != (packed ? 0 : narrow ? 1 : 2)) return;  // another kernel owns this CTA
  const size_t base0 = geo_base(off, batch, t0);  // first row of the CTA's iterations
  if (STAGED && off) {  // ragged: rows need not be 16-byte aligned
    for (int e = tid; e < B; e += kDispatchThreads) sm[e] = __ldg(sorted_len + base0 + e);
    uint32_t* st = sm + (size_t)tt * B;
    const uint32_t* gc = cost + base0 * k_pad;
    for (int e = tid; e < B * k_pad; e += kDispatchThreads) {
      const int i = e / k_pad, k = e - i * k_pad;
      st[TRANS ? (size_t)k * Bp + i : (size_t)e] = __ldg(gc + e);
    }
  } else if (STAGED) {
    const uint4* gl = reinterpret_cast<const uint4*>(sorted_len + base0);
    uint4* sl4 = reinterpret_cast<uint4*>(sm);
    const int nl = ntt * B / 4;
    for (int e = tid; e < nl; e += kDispatchThreads) sl4[e] = __ldg(gl + e);
    const uint4* gc = reinterpret_cast<const uint4*>(cost + base0 * k_pad);
    const int nc = ntt * B * k_pad / 4;
    if (TRANS) {
      uint32_t* st = sm + (size_t)tt * B;
      for (int e = tid; e < nc; e += kDispatchThreads) {
        const uint4 v = __ldg(gc + e);
        const int f = e * 4;  // flat index (lt * B + i) * k_pad + k, k % 4 == 0
        const int row = f / k_pad, k = f - row * k_pad;
        const int lt = row / B, i = row - lt * B;
        uint32_t* d = st + ((size_t)lt * k_pad + k) * Bp + i;
        d[0] = v.x;
        d[Bp] = v.y;
        d[2 * Bp] = v.z;
        d[3 * Bp] = v.w;
      }
    } else {
      uint4* sc4 = reinterpret_cast<uint4*>(sm + (size_t)tt * B);
      for (int e = tid; e < nc; e += kDispatchThreads) sc4[e] = __ldg(gc + e);
    }
  }
#pragma unroll
  for (int j = 0; j < DP; ++j) s_sum[j * kDispatchThreads + tid] = 0ull;
  __syncthreads();

  const int lt = tid / ct, lc = tid - lt * ct;
  const int c = c0 + lc, t = t0 + lt;
  // (WIN: every thread stays for the CTA's window copies; tt == 1 there)
  const bool active = !(lt >= tt || c >= n_cand || t >= n_iter || B == 0);
  if (!WIN && !active) return;
  if (WIN && (B == 0 || t0 >= n_iter)) return;  // CTA-uniform

  const size_t tbase = geo_base(off, batch, t);
  const uint32_t* sl = STAGED ? sm + (size_t)lt * B : sorted_len + tbase;
  const uint32_t* cs = STAGED ? sm + (size_t)tt * B + (size_t)lt * B * k_pad : cost + tbase * k_pad;
  const size_t row = (size_t)c * n_iter + t;
  uint8_t* prow = pipe + (size_t)c * n_total + tbase;  // = row * B for uniform batches

  // candidate: pipelines in canonical order; unused lanes get MaxLen 0 (never feasible)
  const int np = active ? cand_np[c] : 0;
  uint32_t ml[DP], pp[DP], kk[DP];
  bool ok = np >= 1 && np <= DP;
  uint32_t prev_ml = 0xFFFFFFFFu, prev_k = 0;
#pragma unroll
  for (int j = 0; j < DP; ++j) {
    ml[j] = 0u;
    pp[j] = 1u;
    kk[j] = 0u;
    if (j < np) {
      const uint32_t k = cand[(size_t)c * HYD_MAX_PIPES + j];
      if (k < (uint32_t)n_schemes) {
        const uint32_t m = schemes[k].max_len;
        const uint32_t p = schemes[k].pp;
        ok = ok && (m < prev_ml || (m == prev_ml && k >= prev_k)) && p >= 1u && p <= HYD_MAX_PP &&
             m >= 1u;
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
  if (active && !ok) flag(status, HYD_F_NOT_CANONICAL);
  const size_t srow = (size_t)t * n_cand + c;  // iteration-major stats / members row
  const bool live = active && ok && sl[0] <= ml[0];
  if (active && !live) {  // infeasible candidate for this iteration
    for (int i = 0; i < B; ++i) prow[i] = 0xFF;
    lb[row] = ~0ull;
    stats[srow * max_np].u = 0xFFFFFFFFu;
  }
  if (!WIN && !live) return;
  const int nwords = (batch + 31) >> 5;  // row stride: words of the largest batch
  uint32_t* mbits = members + srow * max_np * nwords;  // word w of pipeline j at [w * max_np + j]
  unsigned long long* ssum = s_sum + tid;
  uint64_t lbv = 0ull;
  uint32_t cf[DP];
  hyd_pipe_stats* st = stats + srow * max_np;
  auto write_stats = [&](const auto& base) {
    lb[row] = lbv;
#pragma unroll
    for (int j = 0; j < DP; ++j) {
      if (j < np) {
        const uint32_t first = cf[j] & 0xFFFFu;  // 0: no member
        const uint32_t tm = !first ? 0u
                            : TRANS ? sm[(size_t)tt * B + ((size_t)lt * k_pad + kk[j]) * Bp + first - 1u]
                                    : cs[(size_t)(first - 1u) * k_pad + kk[j]];
        hyd_pipe_stats e;
        e.u = cf[j] >> 16;
        e.tau_max = tm;
        e.s = ssum[j * kDispatchThreads];
        e.sum_t = (uint64_t)base[j] - (uint64_t)tm * (pp[j] - 1u);  // base_j = C_j + E_j
        st[j] = e;
      }
    }
  };
  if constexpr (MODE == 0) {
    const unsigned amask = __activemask();
    const uint32_t* cst = TRANS ? sm + (size_t)tt * B + (size_t)lt * k_pad * Bp : cs;
    uint32_t base[DP];
    packed_run<DP, TRANS>(sl, cst, B, TRANS ? Bp : k_pad, ml, pp, kk, prow, ssum, mbits, np, max_np,
                          lbv, base, cf, amask);
    write_stats(base);
  } else if constexpr (WIN) {
    using TT = typename std::conditional<MODE == 1, uint32_t, uint64_t>::type;
    TT base[DP];
    // the CTA's iteration t0 (threads past n_cand have lt >= 1 and point elsewhere): windows of it
    dispatch_run_win<DP, TT>(live, sorted_len + base0, cost + base0 * k_pad, sm, B, k_pad, ml, pp, kk, prow, ssum,
                             mbits, np, max_np, lbv, base, cf);
    if (live) write_stats(base);
  } else if constexpr (MODE == 1) {
    uint32_t base[DP];
    dispatch_run<DP, uint32_t>(sl, cs, STAGED, B, k_pad, ml, pp, kk, prow, ssum, mbits, np, max_np, lbv, base,
                               cf);
    write_stats(base);
  } else {
    uint64_t base[DP];
    dispatch_run<DP, uint64_t>(sl, cs, STAGED, B, k_pad, ml, pp, kk, prow, ssum, mbits, np, max_np, lbv, base,
                               cf);
    write_stats(base);
  }
}

template <int DP, bool STAGED, int MODE>
static cudaError_t launch_mode(dim3 grid, size_t smem, cudaStream_t s, const uint32_t* sorted_len,
                               const uint32_t* cost, int n_iter, int batch, const uint32_t* off,
                               size_t n_total, int k_pad,
                               const hyd_scheme* schemes, int n_schemes, const uint8_t* cand,
                               const uint8_t* cand_np, int n_cand, int max_np, int ct, int tt,
                               uint8_t* pipe, uint64_t* lb, hyd_pipe_stats* stats, uint32_t* members,
                               uint32_t* status, const uint64_t* bounds) {
  cudaError_t e = cudaFuncSetAttribute(k_dispatch<DP, STAGED, MODE>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_dispatch<DP, STAGED, MODE><<<grid, kDispatchThreads, smem, s>>>(
      sorted_len, cost, n_iter, batch, off, n_total, k_pad, schemes, n_schemes, cand, cand_np, n_cand, max_np, ct,
      tt, pipe, lb, stats, members, status, bounds);
  note_launch();
  return cudaGetLastError();
}

template <int DP>
static cudaError_t launch_dp(bool staged, dim3 grid, size_t smem_stage, cudaStream_t s,
                             const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch,
                             const uint32_t* off, size_t n_total,
                             int k_pad, const hyd_scheme* schemes, int n_schemes,
                             const uint8_t* cand, const uint8_t* cand_np, int n_cand, int max_np,
                             int ct, int tt, uint8_t* pipe, uint64_t* lb, hyd_pipe_stats* stats,
                             uint32_t* members, uint32_t* status, const uint64_t* bounds) {
  const size_t cols = (size_t)DP * kDispatchThreads * 8;
  const size_t win = (((size_t)kDispatchWin * (1 + k_pad) * 4 + 15) & ~(size_t)15) + cols;  // MODE 1/2, not staged
  cudaError_t e;
#define HYD_LAUNCH_MODE(ST, MD)                                                                            \
  launch_mode<DP, ST, MD>(grid, ST ? ((smem_stage + 15) & ~(size_t)15) + cols : MD ? win : cols, s,      \
                          sorted_len, cost, n_iter, batch, off, n_total, k_pad, schemes,                  \
                          n_schemes, cand, cand_np, n_cand, max_np, ct, tt, pipe, lb, stats, members, status, \
                          bounds)
  if (staged) {
    e = HYD_LAUNCH_MODE(true, 0);
    if (e == cudaSuccess) e = HYD_LAUNCH_MODE(true, 1);
    if (e == cudaSuccess) e = HYD_LAUNCH_MODE(true, 2);
  } else {
    e = HYD_LAUNCH_MODE(false, 0);
    if (e == cudaSuccess) e = HYD_LAUNCH_MODE(false, 1);
    if (e == cudaSuccess) e = HYD_LAUNCH_MODE(false, 2);
  }
#undef HYD_LAUNCH_MODE
  return e;
}

size_t dispatch_workspace(int n_iter) { return ((size_t)n_iter * 8 + 255) & ~(size_t)255; }

int launch_dispatch(const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch,
                    const uint32_t* off, size_t n_total, int k_pad, const hyd_scheme* schemes, int n_schemes, const uint8_t* cand,
                    const uint8_t* cand_np, int n_cand, int max_np, uint8_t* pipe, uint64_t* lb,
                    hyd_pipe_stats* stats, uint32_t* members, uint32_t* status, void* ws,
                    cudaStream_t s) {
  if (n_iter == 0 || n_cand == 0) return HYD_OK;
  uint64_t* bounds = static_cast<uint64_t*>(ws);
  const int rb = launch_iter_bound(cost, n_iter, batch, off, k_pad, schemes, n_schemes, bounds, s);
  if (rb != HYD_OK) return rb;
  const int ct = n_cand < kDispatchThreads ? n_cand : kDispatchThreads;
  int tt = off ? 1 : kDispatchThreads / ct;  // ragged batches: one iteration per CTA
  const size_t smem = dispatch_stage_words(tt, batch, k_pad) * 4;
  const int dp = max_np <= 2 ? 2 : max_np <= 4 ? 4 : max_np <= 8 ? 8 : max_np <= 16 ? 16 : 32;
  const size_t static_smem = (size_t)dp * kDispatchThreads * 8 + 64;
  // stage when the rows fit comfortably (leaves room for several CTAs per SM)
  const bool staged = smem + static_smem <= 96 * 1024 && (off || (batch % 4) == 0);
  if (!staged) tt = 1;  // the window-staged general kernels take one iteration per CTA
  dim3 grid((n_cand + ct - 1) / ct, (n_iter + tt - 1) / tt);
  cudaError_t e;
  switch (dp) {
    case 2: e = launch_dp<2>(staged, grid, smem, s, sorted_len, cost, n_iter, batch, off, n_total, k_pad, schemes, n_schemes, cand, cand_np, n_cand, max_np, ct, tt, pipe, lb, stats, members, status, bounds); break;
    case 4: e = launch_dp<4>(staged, grid, smem, s, sorted_len, cost, n_iter, batch, off, n_total, k_pad, schemes, n_schemes, cand, cand_np, n_cand, max_np, ct, tt, pipe, lb, stats, members, status, bounds); break;
    case 8: e = launch_dp<8>(staged, grid, smem, s, sorted_len, cost, n_iter, batch, off, n_total, k_pad, schemes, n_schemes, cand, cand_np, n_cand, max_np, ct, tt, pipe, lb, stats, members, status, bounds); break;
    case 16: e = launch_dp<16>(staged, grid, smem, s, sorted_len, cost, n_iter, batch, off, n_total, k_pad, schemes, n_schemes, cand, cand_np, n_cand, max_np, ct, tt, pipe, lb, stats, members, status, bounds); break;
    default: e = launch_dp<32>(staged, grid, smem, s, sorted_len, cost, n_iter, batch, off, n_total, k_pad, schemes, n_schemes, cand, cand_np, n_cand, max_np, ct, tt, pipe, lb, stats, members, status, bounds); break;
  }
  return e == cudaSuccess ? HYD_OK : record_cuda_error(e);
}

}  // namespace hyd
