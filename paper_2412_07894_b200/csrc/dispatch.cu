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
// The sums run in u32 when a per-CTA bound proves every load < 2^32, else in u64.
// Outputs: pipe[c][t][i] (4 decisions per u32 store), lb[c][t] = max_j base_j, stats.
#include "hyd_internal.cuh"

namespace hyd {

constexpr int kDispatchThreads = 128;

// One sequence step: candidate loads, argmin (new_j, j), branch-free update of pipeline j*.
// FEAS: test MaxLen_j >= l (only needed while l exceeds the smallest MaxLen of the candidate;
// lengths are sorted descending, so the tail of the batch skips the test).
template <int DP, typename TT, bool FEAS>
__device__ __forceinline__ uint32_t dispatch_step(uint32_t l, const uint32_t* __restrict__ crow,
                                                  bool staged, const uint32_t (&ml)[DP],
                                                  const uint32_t (&kk)[DP], TT (&base)[DP],
                                                  uint32_t (&mult)[DP], uint32_t (&bits)[DP],
                                                  uint32_t bit) {
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
    mult[j] = hit ? 1u : mult[j];
    bits[j] |= hit ? bit : 0u;
  }
  return bj;
}

// Packed-key step (all loads < 2^(31 - SH)): key_j = (C_j + E_j) << SH | j, so the candidate
// key is one IMAD, the argmin is a VIMNMX tree with no index bookkeeping, and the winner's new
// key is the minimum itself.  FEAS masks pipelines with MaxLen_j < l via bit 31.
template <int DP, bool FEAS>
__device__ __forceinline__ uint32_t key_step(uint32_t l, const uint32_t* __restrict__ crow,
                                             bool staged, const uint32_t (&ml)[DP],
                                             const uint32_t (&kk)[DP], uint32_t (&key)[DP],
                                             uint32_t (&mults)[DP], uint32_t (&bits)[DP],
                                             uint32_t bit, uint32_t one_sh) {
  uint32_t m[DP];
#pragma unroll
  for (int j = 0; j < DP; ++j) {
    const uint32_t tau = staged ? crow[kk[j]] : __ldg(crow + kk[j]);
    m[j] = key[j] + tau * mults[j];
    if (FEAS) m[j] |= (l > ml[j]) ? 0x80000000u : 0u;
  }
#pragma unroll
  for (int w = DP / 2; w > 0; w >>= 1)
#pragma unroll
    for (int j = 0; j < w; ++j) m[j] = min(m[j], m[j + w]);
  const uint32_t mk = m[0];
  const uint32_t bj = mk & (uint32_t)(DP - 1);
#pragma unroll
  for (int j = 0; j < DP; ++j) {
    const bool hit = (uint32_t)j == bj;
    key[j] = hit ? mk : key[j];
    mults[j] = hit ? one_sh : mults[j];
    bits[j] |= hit ? bit : 0u;
  }
  return bj;
}

template <int DP, typename TT>
__device__ __forceinline__ void dispatch_run(const uint32_t* __restrict__ sl,
                                             const uint32_t* __restrict__ cs, bool staged, int B,
                                             int k_pad, const uint32_t (&ml)[DP],
                                             const uint32_t (&pp)[DP], const uint32_t (&kk)[DP],
                                             uint8_t* __restrict__ prow, unsigned long long* s_sum,
                                             uint32_t* __restrict__ mbits, int np, int nwords,
                                             uint64_t& lb_out, TT (&base)[DP], uint32_t (&cnt)[DP],
                                             uint32_t (&tmax)[DP], bool packed) {
  constexpr int SH = DP <= 2 ? 1 : DP <= 4 ? 2 : DP <= 8 ? 3 : DP <= 16 ? 4 : 5;
  uint32_t mult[DP], bits[DP];
  uint32_t ml_min = 0xFFFFFFFFu;
#pragma unroll
  for (int j = 0; j < DP; ++j) {  // unused slots: base = max, mult = 0 -> never strictly best
    base[j] = j < np ? (TT)0 : (TT)~(TT)0;
    mult[j] = j < np ? pp[j] : 0u;
    bits[j] = 0u;
    cnt[j] = 0u;
    tmax[j] = 0u;
    if (j < np) ml_min = min(ml_min, ml[j]);
  }
  uint32_t key[DP], mults[DP];
  if (packed) {
#pragma unroll
    for (int j = 0; j < DP; ++j) {
      key[j] = j < np ? (uint32_t)j : 0x7FFFFFFFu;  // unused slots never win (bit 31 clear, > any)
      mults[j] = mult[j] << SH;
    }
  }
  const bool words = (B & 3) == 0;
  uint32_t word = 0u;
  for (int i = 0; i < B; ++i) {
    const uint32_t l = sl[i];
    const uint32_t* crow = cs + (size_t)i * k_pad;
    const uint32_t bit = 1u << (i & 31);
    uint32_t bj;
    if (packed) {
      bj = l > ml_min ? key_step<DP, true>(l, crow, staged, ml, kk, key, mults, bits, bit, 1u << SH)
                      : key_step<DP, false>(l, crow, staged, ml, kk, key, mults, bits, bit, 1u << SH);
    } else {
      bj = l > ml_min ? dispatch_step<DP, TT, true>(l, crow, staged, ml, kk, base, mult, bits, bit)
                      : dispatch_step<DP, TT, false>(l, crow, staged, ml, kk, base, mult, bits, bit);
    }
    s_sum[bj * kDispatchThreads] += l;  // S_j column of this thread
    if ((i & 31) == 31 || i == B - 1) {  // flush one membership word per pipeline; U_j, tau_max_j
      const int w0 = i & ~31;
#pragma unroll
      for (int j = 0; j < DP; ++j) {
        if (j < np) {
          mbits[(size_t)j * nwords + (i >> 5)] = bits[j];
          if (cnt[j] == 0u && bits[j] != 0u) {  // first (= longest) member of pipeline j
            const uint32_t* frow = cs + (size_t)(w0 + __ffs(bits[j]) - 1) * k_pad;
            tmax[j] = staged ? frow[kk[j]] : __ldg(frow + kk[j]);
          }
          cnt[j] += __popc(bits[j]);
        }
        bits[j] = 0u;
      }
    }
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
  if (packed) {
#pragma unroll
    for (int j = 0; j < DP; ++j) base[j] = j < np ? (TT)(key[j] >> SH) : (TT)~(TT)0;
  }
  uint64_t m = 0ull;
#pragma unroll
  for (int j = 0; j < DP; ++j)
    if (j < np) m = max(m, (uint64_t)base[j]);
  lb_out = m;
}

template <int DP, bool STAGED>
__global__ void __launch_bounds__(kDispatchThreads)
    k_dispatch(const uint32_t* __restrict__ sorted_len, const uint32_t* __restrict__ cost,
               int n_iter, int batch, int k_pad, const hyd_scheme* __restrict__ schemes,
               int n_schemes, const uint8_t* __restrict__ cand, const uint8_t* __restrict__ cand_np,
               int n_cand, int max_np, int ct, int tt, uint8_t* __restrict__ pipe,
               uint64_t* __restrict__ lb, hyd_pipe_stats* __restrict__ stats,
               uint32_t* __restrict__ members, uint32_t* __restrict__ status) {
  extern __shared__ __align__(16) uint32_t sm[];
  // dynamic smem: [stage: tt*B*(1+k_pad) u32 if STAGED] [s_sum u64 columns]
  const size_t stage_words = STAGED ? (size_t)tt * batch * (1 + k_pad) : 0;
  unsigned long long* s_sum = reinterpret_cast<unsigned long long*>(sm + ((stage_words + 3) & ~(size_t)3));
  __shared__ unsigned long long s_bound[kDispatchThreads / 32];
  __shared__ uint32_t s_ppmax;
  const int B = batch;
  const int tid = threadIdx.x;
  const int c0 = blockIdx.x * ct, t0 = blockIdx.y * tt;
  const int ntt = min(tt, n_iter - t0);
  if (STAGED) {
    // [tt][B] lengths then [tt][B][k_pad] costs, both contiguous in global memory per t
    const uint4* gl = reinterpret_cast<const uint4*>(sorted_len + (size_t)t0 * B);
    uint4* sl4 = reinterpret_cast<uint4*>(sm);
    const int nl = ntt * B / 4;
    for (int e = tid; e < nl; e += kDispatchThreads) sl4[e] = __ldg(gl + e);
    const uint4* gc = reinterpret_cast<const uint4*>(cost + (size_t)t0 * B * k_pad);
    uint4* sc4 = reinterpret_cast<uint4*>(sm + (size_t)tt * B);
    const int nc = ntt * B * k_pad / 4;
    for (int e = tid; e < nc; e += kDispatchThreads) sc4[e] = __ldg(gc + e);
  }
  if (tid == 0) {
    uint32_t m = 1u;
    for (int k = 0; k < n_schemes; ++k) m = max(m, schemes[k].pp);
    s_ppmax = m;
  }
#pragma unroll
  for (int j = 0; j < DP; ++j) s_sum[j * kDispatchThreads + tid] = 0ull;
  __syncthreads();
  // u32 bound over the CTA's iterations: sum_i max_k tau_ik + max tau * (PPmax - 1) < 2^32-1
  //  =>  every base_j and new_j of every thread fits u32 (strictly below the u32 sentinel).
  unsigned long long bound = 0ull;
  for (int e = tid; e < ntt * B; e += kDispatchThreads) {
    const int lt = e / B, i = e - lt * B;
    const uint32_t* crow = STAGED ? sm + (size_t)tt * B + ((size_t)lt * B + i) * k_pad
                                  : cost + ((size_t)(t0 + lt) * B + i) * k_pad;
    uint32_t mx = 0u;
    for (int k = 0; k < n_schemes; ++k) mx = max(mx, STAGED ? crow[k] : __ldg(crow + k));
    unsigned long long v = (unsigned long long)mx;
    if (i == 0) v += (unsigned long long)mx * (s_ppmax - 1u);
    bound += v;
  }
  for (int o = 16; o > 0; o >>= 1) bound += __shfl_xor_sync(HYD_FULL, bound, o);
  if ((tid & 31) == 0) s_bound[tid >> 5] = bound;
  __syncthreads();
  bound = 0ull;
  for (int w = 0; w < kDispatchThreads / 32; ++w) bound += s_bound[w];
  const bool narrow = bound < 0xFFFFFFFFull;
  constexpr int SHK = DP <= 2 ? 1 : DP <= 4 ? 2 : DP <= 8 ? 3 : DP <= 16 ? 4 : 5;
  const bool packed = bound < (1ull << (31 - SHK));  // keys (load << SHK | j) stay below 2^31

  const int lt = tid / ct, lc = tid - lt * ct;
  const int c = c0 + lc, t = t0 + lt;
  if (lt >= tt || c >= n_cand || t >= n_iter) return;

  const uint32_t* sl = STAGED ? sm + (size_t)lt * B : sorted_len + (size_t)t * B;
  const uint32_t* cs = STAGED ? sm + (size_t)tt * B + (size_t)lt * B * k_pad
                              : cost + (size_t)t * B * k_pad;
  const size_t row = (size_t)c * n_iter + t;
  uint8_t* prow = pipe + row * B;

  // candidate: pipelines in canonical order; unused lanes get MaxLen 0 (never feasible)
  const int np = cand_np[c];
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
  if (!ok) flag(status, HYD_F_NOT_CANONICAL);
  const size_t srow = (size_t)t * n_cand + c;  // iteration-major stats / members row
  if (!ok || sl[0] > ml[0]) {  // infeasible candidate for this iteration
    for (int i = 0; i < B; ++i) prow[i] = 0xFF;
    lb[row] = ~0ull;
    stats[srow * max_np].u = 0xFFFFFFFFu;
    return;
  }
  const int nwords = (B + 31) >> 5;
  uint32_t* mbits = members + srow * max_np * nwords;
  unsigned long long* ssum = s_sum + tid;
  uint64_t lbv = 0ull;
  uint64_t base64[DP];
  uint32_t cnt[DP], tmx[DP];
  if (narrow) {
    uint32_t base[DP];
    dispatch_run<DP, uint32_t>(sl, cs, STAGED, B, k_pad, ml, pp, kk, prow, ssum, mbits, np, nwords,
                               lbv, base, cnt, tmx, packed);
#pragma unroll
    for (int j = 0; j < DP; ++j) base64[j] = base[j];
  } else {
    dispatch_run<DP, uint64_t>(sl, cs, STAGED, B, k_pad, ml, pp, kk, prow, ssum, mbits, np, nwords,
                               lbv, base64, cnt, tmx, false);
  }
  lb[row] = lbv;
  hyd_pipe_stats* st = stats + srow * max_np;
#pragma unroll
  for (int j = 0; j < DP; ++j) {
    if (j < np) {
      hyd_pipe_stats e;
      e.u = cnt[j];
      e.tau_max = tmx[j];
      e.s = ssum[j * kDispatchThreads];
      e.sum_t = base64[j] - (uint64_t)tmx[j] * (pp[j] - 1u);  // base_j = C_j + E_j
      st[j] = e;
    }
  }
}

template <int DP>
static cudaError_t launch_dp(bool staged, dim3 grid, size_t smem_stage, cudaStream_t s,
                             const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch,
                             int k_pad, const hyd_scheme* schemes, int n_schemes,
                             const uint8_t* cand, const uint8_t* cand_np, int n_cand, int max_np,
                             int ct, int tt, uint8_t* pipe, uint64_t* lb, hyd_pipe_stats* stats,
                             uint32_t* members, uint32_t* status) {
  const size_t cols = (size_t)DP * kDispatchThreads * 8;
  cudaError_t e;
  if (staged) {
    const size_t smem = ((smem_stage + 15) & ~(size_t)15) + cols;
    e = cudaFuncSetAttribute(k_dispatch<DP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_dispatch<DP, true><<<grid, kDispatchThreads, smem, s>>>(
        sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, max_np,
        ct, tt, pipe, lb, stats, members, status);
  } else {
    e = cudaFuncSetAttribute(k_dispatch<DP, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cols);
    if (e != cudaSuccess) return e;
    k_dispatch<DP, false><<<grid, kDispatchThreads, cols, s>>>(
        sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, max_np,
        ct, tt, pipe, lb, stats, members, status);
  }
  return cudaGetLastError();
}

int launch_dispatch(const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch,
                    int k_pad, const hyd_scheme* schemes, int n_schemes, const uint8_t* cand,
                    const uint8_t* cand_np, int n_cand, int max_np, uint8_t* pipe, uint64_t* lb,
                    hyd_pipe_stats* stats, uint32_t* members, uint32_t* status, cudaStream_t s) {
  if (n_iter == 0 || n_cand == 0) return HYD_OK;
  const int ct = n_cand < kDispatchThreads ? n_cand : kDispatchThreads;
  const int tt = kDispatchThreads / ct;
  const size_t smem = (size_t)tt * batch * 4 * (1 + (size_t)k_pad);
  const int dp = max_np <= 2 ? 2 : max_np <= 4 ? 4 : max_np <= 8 ? 8 : max_np <= 16 ? 16 : 32;
  const size_t static_smem = (size_t)dp * kDispatchThreads * 8 + 64;
  // stage when the rows fit comfortably (leaves room for several CTAs per SM)
  const bool staged = smem + static_smem <= 96 * 1024 && (batch % 4) == 0;
  dim3 grid((n_cand + ct - 1) / ct, (n_iter + tt - 1) / tt);
  cudaError_t e;
  switch (dp) {
    case 2: e = launch_dp<2>(staged, grid, smem, s, sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, max_np, ct, tt, pipe, lb, stats, members, status); break;
    case 4: e = launch_dp<4>(staged, grid, smem, s, sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, max_np, ct, tt, pipe, lb, stats, members, status); break;
    case 8: e = launch_dp<8>(staged, grid, smem, s, sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, max_np, ct, tt, pipe, lb, stats, members, status); break;
    case 16: e = launch_dp<16>(staged, grid, smem, s, sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, max_np, ct, tt, pipe, lb, stats, members, status); break;
    default: e = launch_dp<32>(staged, grid, smem, s, sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, max_np, ct, tt, pipe, lb, stats, members, status); break;
  }
  note_launch();
  return e == cudaSuccess ? HYD_OK : record_cuda_error(e);
}

}  // namespace hyd
