// dispatch.cu -- a3: stage 1 sequence dispatching across pipelines (§6.2).
//
// One thread per (candidate c, iteration t).  A CTA covers `ct` candidates x `tt`
// iterations (ct*tt <= 128), so every thread of a warp shares the iteration's sorted
// lengths and cost rows; when they fit, those rows are staged in shared memory once per
// CTA (16-byte copies) and each sequence step reads one <=64-word smem row (a single
// wavefront: the threads' scheme indices fall in one row).  Pipeline state lives in
// registers, unrolled over DP = next_pow2(max_np) lanes:
//   C_j (load_j, u64), E_j (extra_j, u64), an "occupied" bit, MaxLen_j, PP_j - 1, k_j.
// Per sequence i (longest first) and feasible j (MaxLen_j >= l_i, the horizon J_i of P:626):
//   e_j  = occupied ? E_j : tau * (PP_j - 1)       (Eq. 2 extra term; Alg. 1 l.10)
//   new_j = C_j + tau + e_j                          (Alg. 1 lines 9-11)
//   j* = argmin (new_j, j)                           (SURVEY §8(c) step 4 / reading 10)
// Decisions are packed 4 per u32 store.  Output: pipe[c][t][i], lb[c][t] = max_j C_j+E_j.
#include "hyd_internal.cuh"

namespace hyd {

constexpr int kDispatchThreads = 128;

template <int DP, bool STAGED>
__global__ void __launch_bounds__(kDispatchThreads)
    k_dispatch(const uint32_t* __restrict__ sorted_len, const uint32_t* __restrict__ cost,
               int n_iter, int batch, int k_pad, const hyd_scheme* __restrict__ schemes,
               int n_schemes, const uint8_t* __restrict__ cand, const uint8_t* __restrict__ cand_np,
               int n_cand, int ct, int tt, uint8_t* __restrict__ pipe, uint64_t* __restrict__ lb,
               uint32_t* __restrict__ status) {
  extern __shared__ __align__(16) uint32_t sm[];
  const int B = batch;
  const int tid = threadIdx.x;
  const int c0 = blockIdx.x * ct, t0 = blockIdx.y * tt;
  if (STAGED) {
    // [tt][B] lengths then [tt][B][k_pad] costs, both contiguous in global memory per t
    const int ntt = min(tt, n_iter - t0);
    const uint4* gl = reinterpret_cast<const uint4*>(sorted_len + (size_t)t0 * B);
    uint4* sl4 = reinterpret_cast<uint4*>(sm);
    const int nl = ntt * B / 4;
    for (int e = tid; e < nl; e += kDispatchThreads) sl4[e] = __ldg(gl + e);
    const uint4* gc = reinterpret_cast<const uint4*>(cost + (size_t)t0 * B * k_pad);
    uint4* sc4 = reinterpret_cast<uint4*>(sm + (size_t)tt * B);
    const int nc = ntt * B * k_pad / 4;
    for (int e = tid; e < nc; e += kDispatchThreads) sc4[e] = __ldg(gc + e);
    __syncthreads();
  }
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
  uint32_t ml[DP], ppm1[DP], kk[DP];
  bool ok = np >= 1 && np <= DP;
  uint32_t prev_ml = 0xFFFFFFFFu, prev_k = 0;
#pragma unroll
  for (int j = 0; j < DP; ++j) {
    ml[j] = 0u;
    ppm1[j] = 0u;
    kk[j] = 0u;
    if (j < np) {
      const uint32_t k = cand[(size_t)c * HYD_MAX_PIPES + j];
      if (k < (uint32_t)n_schemes) {
        const uint32_t m = schemes[k].max_len;
        const uint32_t pp = schemes[k].pp;
        ok = ok && (m < prev_ml || (m == prev_ml && k >= prev_k)) && pp >= 1u && pp <= HYD_MAX_PP &&
             m >= 1u;
        prev_ml = m;
        prev_k = k;
        ml[j] = m;
        ppm1[j] = pp - 1u;
        kk[j] = k;
      } else {
        ok = false;
      }
    }
  }
  if (!ok) flag(status, HYD_F_NOT_CANONICAL);
  if (!ok || sl[0] > ml[0]) {  // infeasible candidate for this iteration
    for (int i = 0; i < B; ++i) prow[i] = 0xFF;
    lb[row] = ~0ull;
    return;
  }

  uint64_t ld[DP], ex[DP];
#pragma unroll
  for (int j = 0; j < DP; ++j) {
    ld[j] = 0ull;
    ex[j] = 0ull;
  }
  uint32_t occ = 0u;
  const bool words = (B & 3) == 0;
  uint32_t word = 0u;
  for (int i = 0; i < B; ++i) {
    const uint32_t l = sl[i];
    const uint32_t* crow = cs + (size_t)i * k_pad;
    uint64_t best = ~0ull, btau = 0ull, be = 0ull;
    uint32_t bj = 0u;
#pragma unroll
    for (int j = 0; j < DP; ++j) {
      const uint32_t tau = STAGED ? crow[kk[j]] : __ldg(crow + kk[j]);
      const uint64_t e = ((occ >> j) & 1u) ? ex[j] : (uint64_t)tau * ppm1[j];
      const uint64_t nw = ld[j] + tau + e;
      if (l <= ml[j] && nw < best) {
        best = nw;
        bj = (uint32_t)j;
        btau = tau;
        be = e;
      }
    }
#pragma unroll
    for (int j = 0; j < DP; ++j)
      if ((uint32_t)j == bj) {
        ld[j] += btau;
        ex[j] = be;
      }
    occ |= 1u << bj;
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
  uint64_t m = 0ull;
#pragma unroll
  for (int j = 0; j < DP; ++j) m = max(m, ld[j] + ex[j]);
  lb[row] = m;
}

template <int DP>
static cudaError_t launch_dp(bool staged, dim3 grid, size_t smem, cudaStream_t s,
                             const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch,
                             int k_pad, const hyd_scheme* schemes, int n_schemes,
                             const uint8_t* cand, const uint8_t* cand_np, int n_cand, int ct,
                             int tt, uint8_t* pipe, uint64_t* lb, uint32_t* status) {
  if (staged) {
    cudaError_t e = cudaFuncSetAttribute(k_dispatch<DP, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_dispatch<DP, true><<<grid, kDispatchThreads, smem, s>>>(
        sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, ct, tt,
        pipe, lb, status);
  } else {
    k_dispatch<DP, false><<<grid, kDispatchThreads, 0, s>>>(
        sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, ct, tt,
        pipe, lb, status);
  }
  return cudaGetLastError();
}

int launch_dispatch(const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch,
                    int k_pad, const hyd_scheme* schemes, int n_schemes, const uint8_t* cand,
                    const uint8_t* cand_np, int n_cand, int max_np, uint8_t* pipe, uint64_t* lb,
                    uint32_t* status, cudaStream_t s) {
  if (n_iter == 0 || n_cand == 0) return HYD_OK;
  const int ct = n_cand < kDispatchThreads ? n_cand : kDispatchThreads;
  const int tt = kDispatchThreads / ct;
  const size_t smem = (size_t)tt * batch * 4 * (1 + (size_t)k_pad);
  // stage when the rows fit comfortably (leaves room for several CTAs per SM)
  const bool staged = smem <= 96 * 1024 && (batch % 4) == 0;
  dim3 grid((n_cand + ct - 1) / ct, (n_iter + tt - 1) / tt);
  cudaError_t e;
  const int dp = max_np <= 2 ? 2 : max_np <= 4 ? 4 : max_np <= 8 ? 8 : max_np <= 16 ? 16 : 32;
  switch (dp) {
    case 2: e = launch_dp<2>(staged, grid, smem, s, sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, ct, tt, pipe, lb, status); break;
    case 4: e = launch_dp<4>(staged, grid, smem, s, sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, ct, tt, pipe, lb, status); break;
    case 8: e = launch_dp<8>(staged, grid, smem, s, sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, ct, tt, pipe, lb, status); break;
    case 16: e = launch_dp<16>(staged, grid, smem, s, sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, ct, tt, pipe, lb, status); break;
    default: e = launch_dp<32>(staged, grid, smem, s, sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, ct, tt, pipe, lb, status); break;
  }
  note_launch();
  return e == cudaSuccess ? HYD_OK : record_cuda_error(e);
}

}  // namespace hyd
