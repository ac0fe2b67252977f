// alg1.cu -- NEXT-1: the paper's randomized greedy dispatcher, Alg. 1, on the GPU.
//
// Stage 1 alternative to dispatch.cu: T random-permutation trials per (c, t); in each trial the
// sequences arrive in the trial's order and go to the feasible pipeline minimising
//   O_max(j) = max(C_j' + E_j', C_k + E_k for k != j)        (Alg. 1 line 10)
// with the first j winning ties (strict <, line 11).  Because C_j' + E_j' >= C_j + E_j, that
// maximum equals max(new_j, M) with M = max_k (C_k + E_k) over all pipelines, one register.
// E_j' = T(l_max, P_j)(PP_j - 1) uses the running maximum cost on pipeline j (T is
// non-decreasing in l, so T(max l) = max T(l)).  The trial with the smallest (O_trial, trial)
// wins (lines 15-17).
//
// Kernels:
//   k_alg1_perm    thread per (t, trial): Fisher-Yates over the B sorted positions from
//                  Philox4x32-10 (the counter layout of include/hyd.h); order [It][T][B] u16.
//   (k_iter_bound of dispatch.cu: a per-iteration bound on every C + E, packed-key choice.)
//   k_alg1_trials  thread per (c, t, trial): lane = candidate, warp = trial, CTA = 8 trials of
//                  one iteration, whose lengths / cost rows / orders are staged in smem.
//                  MODE 0 packed u32 keys max(new_j, M) << SH | j, MODE 1 u64 (CTAs of the
//                  other mode exit at once).  atomicMin of (O_trial << 8 | trial) per (c, t).
//   k_alg1_replay  thread per (c, t): re-runs the winning trial writing pipe, then one pass in
//                  sorted order builds the statistics / membership rows the pack stage reads
//                  (same layouts as dispatch.cu).
#include "hyd_internal.cuh"

namespace hyd {

constexpr int kAlg1Warps = 8;  // trials per CTA
constexpr int kAlg1Threads = 32 * kAlg1Warps;
constexpr int kReplayThreads = 128;

// Philox4x32-10 (Salmon et al., SC'11), 10 rounds, key bumped by the Weyl constants
__device__ __forceinline__ uint4 philox4x32_10(uint4 x, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t lo0 = 0xD2511F53u * x.x, hi0 = __umulhi(0xD2511F53u, x.x);
    const uint32_t lo1 = 0xCD9E8D57u * x.z, hi1 = __umulhi(0xCD9E8D57u, x.z);
    x = make_uint4(hi1 ^ x.y ^ k0, lo1, hi0 ^ x.w ^ k1, lo0);
  }
  return x;
}

__global__ void k_alg1_perm(uint64_t seed, int n_iter, int batch, int trials,
                            uint16_t* __restrict__ order) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_iter * trials) return;
  const int t = g / trials, trial = g - t * trials;
  uint16_t* o = order + (size_t)g * batch;
  for (int i = 0; i < batch; ++i) o[i] = (uint16_t)i;
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  uint4 r = make_uint4(0, 0, 0, 0);
  for (int k = batch - 1; k >= 1; --k) {
    if (k == batch - 1 || (k & 3) == 3)
      r = philox4x32_10(make_uint4((uint32_t)k >> 2, (uint32_t)t, (uint32_t)trial, 0u), k0, k1);
    const uint32_t rk = (k & 3) == 0 ? r.x : (k & 3) == 1 ? r.y : (k & 3) == 2 ? r.z : r.w;
    const uint32_t j = __umulhi(rk, (uint32_t)k + 1u);  // (r * (k + 1)) >> 32
    const uint16_t a = o[k];
    o[k] = o[j];
    o[j] = a;
  }
}

int launch_iter_bound(const uint32_t* cost, int n_iter, int batch, const uint32_t* off, int k_pad,
                      const hyd_scheme* schemes, int n_schemes, uint64_t* bound, cudaStream_t s);

__host__ __device__ constexpr int alg1_sh(int dp) {
  return dp <= 2 ? 1 : dp <= 4 ? 2 : dp <= 8 ? 3 : dp <= 16 ? 4 : 5;
}

// packed keys need every max(new, M) <= 2^(32 - SH) - 2 (the infeasible key is 0xFFFFFFFF)
__host__ __device__ inline bool alg1_packed(uint64_t bound, int dp) {
  return bound < (1ull << (32 - alg1_sh(dp))) - 1ull;
}

// candidate row: canonical check, per-pipeline MaxLen / PP - 1 / scheme (unused slots: MaxLen 0)
template <int DP>
__device__ __forceinline__ bool load_candidate(const hyd_scheme* __restrict__ schemes, int n_schemes,
                                               const uint8_t* __restrict__ cand, int c, int np,
                                               uint32_t (&ml)[DP], uint32_t (&ppm1)[DP],
                                               uint32_t (&kk)[DP]) {
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
        const uint32_t m = schemes[k].max_len, p = schemes[k].pp;
        ok = ok && (m < prev_ml || (m == prev_ml && k >= prev_k)) && p >= 1u && p <= HYD_MAX_PP &&
             m >= 1u;
        prev_ml = m;
        prev_k = k;
        ml[j] = m;
        ppm1[j] = p - 1u;
        kk[j] = k;
      } else {
        ok = false;
      }
    }
  }
  return ok;
}

// One trial of Alg. 1 for candidate c; ~0 if the candidate is infeasible or not canonical.
template <int DP, bool STAGED, int MODE>
__device__ __forceinline__ uint64_t run_trial(const uint32_t* __restrict__ sorted_len,
                                              const uint32_t* __restrict__ cost, int t, int B,
                                              int k_pad, const hyd_scheme* __restrict__ schemes,
                                              int n_schemes, const uint8_t* __restrict__ cand,
                                              const uint8_t* __restrict__ cand_np, int c,
                                              int trials, int trial,
                                              const uint16_t* __restrict__ order,
                                              const uint32_t* s_len, const uint32_t* s_cost,
                                              const uint16_t* s_ord, int warp) {
  constexpr int SH = alg1_sh(DP);
  const int np = cand_np[c];
  uint32_t ml[DP], ppm1[DP], kk[DP];
  if (!load_candidate<DP>(schemes, n_schemes, cand, c, np, ml, ppm1, kk)) return ~0ull;  // replay flags
  const uint32_t* sl = STAGED ? s_len : sorted_len + (size_t)t * B;
  const uint32_t* cs = STAGED ? s_cost : cost + (size_t)t * B * k_pad;
  const uint16_t* ord = STAGED ? s_ord + (size_t)warp * B : order + ((size_t)t * trials + trial) * B;
  if (sl[0] > ml[0]) return ~0ull;  // infeasible candidate

  uint64_t o_trial;
  if constexpr (MODE == 0) {
    uint32_t C[DP], tm[DP];
#pragma unroll
    for (int j = 0; j < DP; ++j) {
      C[j] = 0u;
      tm[j] = 0u;
    }
    uint32_t M = 0u;
    for (int q = 0; q < B; ++q) {
      const uint32_t i = ord[q];
      const uint32_t l = sl[i];
      const uint32_t* row = cs + (size_t)i * k_pad;
      uint32_t tau[DP], key[DP];
#pragma unroll
      for (int j = 0; j < DP; ++j) {
        tau[j] = row[kk[j]];
        const uint32_t nw = C[j] + tau[j] + max(tm[j], tau[j]) * ppm1[j];
        const uint32_t o = max(nw, M);
        key[j] = l <= ml[j] ? (o << SH) | (uint32_t)j : 0xFFFFFFFFu;
      }
      uint32_t m[DP];
#pragma unroll
      for (int j = 0; j < DP; ++j) m[j] = key[j];
#pragma unroll
      for (int w = DP / 2; w > 0; w >>= 1)
#pragma unroll
        for (int j = 0; j < w; ++j) m[j] = min(m[j], m[j + w]);
      const uint32_t bj = m[0] & (uint32_t)(DP - 1);
      M = m[0] >> SH;
#pragma unroll
      for (int j = 0; j < DP; ++j) {
        const bool hit = (uint32_t)j == bj;
        C[j] = hit ? C[j] + tau[j] : C[j];
        tm[j] = hit ? max(tm[j], tau[j]) : tm[j];
      }
    }
    o_trial = M;
  } else {
    uint64_t C[DP];
    uint32_t tm[DP];
#pragma unroll
    for (int j = 0; j < DP; ++j) {
      C[j] = 0ull;
      tm[j] = 0u;
    }
    uint64_t M = 0ull;
    for (int q = 0; q < B; ++q) {
      const uint32_t i = ord[q];
      const uint32_t l = sl[i];
      const uint32_t* row = cs + (size_t)i * k_pad;
      uint32_t tau[DP];
      uint64_t best_o = ~0ull;
      uint32_t bj = 0u;
#pragma unroll
      for (int j = 0; j < DP; ++j) {
        tau[j] = row[kk[j]];
        const uint64_t nw = C[j] + tau[j] + (uint64_t)max(tm[j], tau[j]) * ppm1[j];
        const uint64_t o = max(nw, M);
        if (l <= ml[j] && o < best_o) {
          best_o = o;
          bj = (uint32_t)j;
        }
      }
      M = best_o;
#pragma unroll
      for (int j = 0; j < DP; ++j) {
        const bool hit = (uint32_t)j == bj;
        C[j] = hit ? C[j] + tau[j] : C[j];
        tm[j] = hit ? max(tm[j], tau[j]) : tm[j];
      }
    }
    o_trial = M;
  }
  return o_trial;
}

template <int DP, bool STAGED, int MODE>
__global__ void __launch_bounds__(kAlg1Threads)
    k_alg1_trials(const uint32_t* __restrict__ sorted_len, const uint32_t* __restrict__ cost,
                  int n_iter, int batch, int k_pad, const hyd_scheme* __restrict__ schemes,
                  int n_schemes, const uint8_t* __restrict__ cand,
                  const uint8_t* __restrict__ cand_np, int n_cand, int trials,
                  const uint16_t* __restrict__ order, const uint64_t* __restrict__ bound,
                  unsigned long long* __restrict__ best) {
  extern __shared__ __align__(16) uint32_t sm[];
  const int B = batch, t = blockIdx.y;
  if (alg1_packed(bound[t], DP) != (MODE == 0)) return;  // the other kernel owns this iteration
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tr0 = blockIdx.z * kAlg1Warps;
  const int ntr = min(kAlg1Warps, trials - tr0);
  // smem (STAGED): [B] lengths, [B][k_pad] costs, [kAlg1Warps][B] orders (u16)
  uint32_t* s_len = sm;
  uint32_t* s_cost = sm + B;
  uint16_t* s_ord = reinterpret_cast<uint16_t*>(sm + (size_t)B * (1 + k_pad));
  if (STAGED) {
    const uint4* gl = reinterpret_cast<const uint4*>(sorted_len + (size_t)t * B);
    for (int e = tid; e < B / 4; e += kAlg1Threads) reinterpret_cast<uint4*>(s_len)[e] = __ldg(gl + e);
    const uint4* gc = reinterpret_cast<const uint4*>(cost + (size_t)t * B * k_pad);
    for (int e = tid; e < B * k_pad / 4; e += kAlg1Threads)
      reinterpret_cast<uint4*>(s_cost)[e] = __ldg(gc + e);
    const uint4* go = reinterpret_cast<const uint4*>(order + ((size_t)t * trials + tr0) * B);
    for (int e = tid; e < ntr * B / 8; e += kAlg1Threads)
      reinterpret_cast<uint4*>(s_ord)[e] = __ldg(go + e);
    __syncthreads();
  }
  __shared__ unsigned long long s_best[32];  // per lane (candidate): min over the CTA's trials
  if (tid < 32) s_best[tid] = ~0ull;
  __syncthreads();
  const int c = blockIdx.x * 32 + lane, trial = tr0 + warp;
  const uint64_t o_trial = (c < n_cand && warp < ntr)
                               ? run_trial<DP, STAGED, MODE>(sorted_len, cost, t, B, k_pad, schemes,
                                                             n_schemes, cand, cand_np, c, trials,
                                                             trial, order, s_len, s_cost, s_ord, warp)
                               : ~0ull;
  if (o_trial != ~0ull) atomicMin(&s_best[lane], (unsigned long long)((o_trial << 8) | (uint64_t)trial));
  __syncthreads();
  if (tid < 32 && s_best[tid] != ~0ull)
    atomicMin(best + (size_t)(blockIdx.x * 32 + tid) * n_iter + t, s_best[tid]);
}


// Replay of the winning trial (u64 arithmetic, same decisions as k_alg1_trials), then the
// sorted-order pass: pipe row, lb, stats (U_j, tau_max_j, S_j, sum_t = C_j), membership words.
template <int DP>
__global__ void __launch_bounds__(kReplayThreads)
    k_alg1_replay(const uint32_t* __restrict__ sorted_len, const uint32_t* __restrict__ cost,
                  int n_iter, int batch, int k_pad, const hyd_scheme* __restrict__ schemes,
                  int n_schemes, const uint8_t* __restrict__ cand, const uint8_t* __restrict__ cand_np,
                  int n_cand, int max_np, int trials, const uint16_t* __restrict__ order,
                  unsigned long long* __restrict__ best, uint8_t* __restrict__ pipe,
                  uint64_t* __restrict__ lb, hyd_pipe_stats* __restrict__ stats,
                  uint32_t* __restrict__ members, uint32_t* __restrict__ status) {
  __shared__ unsigned long long s_sum[DP * kReplayThreads];
  const int tid = threadIdx.x;
  const int c = blockIdx.x * kReplayThreads + tid, t = blockIdx.y;
  if (c >= n_cand) return;
  const int B = batch;
  const size_t row = (size_t)c * n_iter + t;
  const size_t srow = (size_t)t * n_cand + c;
  uint8_t* prow = pipe + row * B;
  const int np = cand_np[c];
  uint32_t ml[DP], ppm1[DP], kk[DP];
  const bool ok = load_candidate<DP>(schemes, n_schemes, cand, c, np, ml, ppm1, kk);
  if (!ok) flag(status, HYD_F_NOT_CANONICAL);
  const uint32_t* sl = sorted_len + (size_t)t * B;
  const uint32_t* cs = cost + (size_t)t * B * k_pad;
  if (!ok || sl[0] > ml[0]) {  // infeasible candidate for this iteration
    for (int i = 0; i < B; ++i) prow[i] = 0xFF;
    lb[row] = ~0ull;
    best[row] = ~0ull;
    stats[srow * max_np].u = 0xFFFFFFFFu;
    return;
  }
  const unsigned long long bk = best[row];
  const int trial = (int)(bk & 0xFFu);
  const uint16_t* ord = order + ((size_t)t * trials + trial) * B;
  uint64_t C[DP];
  uint32_t tm[DP];
#pragma unroll
  for (int j = 0; j < DP; ++j) {
    C[j] = 0ull;
    tm[j] = 0u;
  }
  uint64_t M = 0ull;
  for (int q = 0; q < B; ++q) {
    const uint32_t i = __ldg(ord + q);
    const uint32_t l = __ldg(sl + i);
    const uint32_t* crow = cs + (size_t)i * k_pad;
    uint32_t tau[DP];
    uint64_t best_o = ~0ull;
    uint32_t bj = 0u;
#pragma unroll
    for (int j = 0; j < DP; ++j) {
      tau[j] = __ldg(crow + kk[j]);
      const uint64_t nw = C[j] + tau[j] + (uint64_t)max(tm[j], tau[j]) * ppm1[j];
      const uint64_t o = max(nw, M);
      if (l <= ml[j] && o < best_o) {
        best_o = o;
        bj = (uint32_t)j;
      }
    }
    M = best_o;
#pragma unroll
    for (int j = 0; j < DP; ++j) {
      const bool hit = (uint32_t)j == bj;
      C[j] = hit ? C[j] + tau[j] : C[j];
      tm[j] = hit ? max(tm[j], tau[j]) : tm[j];
    }
    prow[i] = (uint8_t)bj;
  }
  lb[row] = M;
  // sorted-order pass: S_j, U_j, first (longest) member, membership words
  const int nwords = (B + 31) >> 5;
  uint32_t* mbits = members + srow * max_np * nwords;
#pragma unroll
  for (int j = 0; j < DP; ++j) s_sum[j * kReplayThreads + tid] = 0ull;
  uint32_t bits[DP], cnt[DP], first[DP];
#pragma unroll
  for (int j = 0; j < DP; ++j) {
    bits[j] = 0u;
    cnt[j] = 0u;
    first[j] = 0xFFFFFFFFu;
  }
  for (int i = 0; i < B; ++i) {
    const uint32_t j0 = prow[i];
    s_sum[j0 * kReplayThreads + tid] += __ldg(sl + i);
#pragma unroll
    for (int j = 0; j < DP; ++j) {
      const bool hit = (uint32_t)j == j0;
      bits[j] |= hit ? 1u << (i & 31) : 0u;
      first[j] = hit && first[j] == 0xFFFFFFFFu ? (uint32_t)i : first[j];
    }
    if ((i & 31) == 31 || i == B - 1) {
#pragma unroll
      for (int j = 0; j < DP; ++j) {
        if (j < np) mbits[(size_t)(i >> 5) * max_np + j] = bits[j];  // word-major
        cnt[j] += __popc(bits[j]);
        bits[j] = 0u;
      }
    }
  }
  hyd_pipe_stats* st = stats + srow * max_np;
#pragma unroll
  for (int j = 0; j < DP; ++j) {
    if (j < np) {
      hyd_pipe_stats e;
      e.u = cnt[j];
      e.tau_max = cnt[j] ? __ldg(cs + (size_t)first[j] * k_pad + kk[j]) : 0u;
      e.s = s_sum[j * kReplayThreads + tid];
      e.sum_t = C[j];
      st[j] = e;
    }
  }
}

int launch_alg1_perm(uint64_t seed, int n_iter, int batch, int trials, uint16_t* order,
                     cudaStream_t s) {
  const int n = n_iter * trials;
  if (n == 0) return HYD_OK;
  k_alg1_perm<<<(n + 127) / 128, 128, 0, s>>>(seed, n_iter, batch, trials, order);
  note_launch();
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HYD_OK : record_cuda_error(e);
}

size_t alg1_stage_bytes(int batch, int k_pad) {
  return (size_t)batch * (1 + k_pad) * 4 + (size_t)kAlg1Warps * batch * 2;
}

template <int DP, bool STAGED, int MODE>
static cudaError_t launch_trials(dim3 grid, size_t smem, cudaStream_t s, const uint32_t* sorted_len,
                                 const uint32_t* cost, int n_iter, int batch, int k_pad,
                                 const hyd_scheme* schemes, int n_schemes, const uint8_t* cand,
                                 const uint8_t* cand_np, int n_cand, int trials,
                                 const uint16_t* order, const uint64_t* bound, uint64_t* best) {
  cudaError_t e = cudaFuncSetAttribute(k_alg1_trials<DP, STAGED, MODE>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_alg1_trials<DP, STAGED, MODE><<<grid, kAlg1Threads, smem, s>>>(
      sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, trials,
      order, bound, reinterpret_cast<unsigned long long*>(best));
  note_launch();
  return cudaGetLastError();
}

template <int DP>
static cudaError_t launch_alg1_dp(const uint32_t* sorted_len, const uint32_t* cost, int n_iter,
                                  int batch, int k_pad, const hyd_scheme* schemes, int n_schemes,
                                  const uint8_t* cand, const uint8_t* cand_np, int n_cand,
                                  int max_np, int trials, const uint16_t* order, uint64_t* bound,
                                  uint64_t* best, uint8_t* pipe, uint64_t* lb,
                                  hyd_pipe_stats* stats, uint32_t* members, uint32_t* status,
                                  cudaStream_t s) {
  if (launch_iter_bound(cost, n_iter, batch, nullptr, k_pad, schemes, n_schemes, bound, s) != HYD_OK)
    return cudaGetLastError();
  cudaError_t e = cudaMemsetAsync(best, 0xFF, (size_t)n_cand * n_iter * 8, s);
  if (e != cudaSuccess) return e;
  const size_t stage = alg1_stage_bytes(batch, k_pad);
  const bool staged = stage <= 160 * 1024 && (batch % 8) == 0;
  const dim3 grid((n_cand + 31) / 32, n_iter, (trials + kAlg1Warps - 1) / kAlg1Warps);
  if (staged) {
    e = launch_trials<DP, true, 0>(grid, stage, s, sorted_len, cost, n_iter, batch, k_pad, schemes,
                                   n_schemes, cand, cand_np, n_cand, trials, order, bound, best);
    if (e == cudaSuccess)
      e = launch_trials<DP, true, 1>(grid, stage, s, sorted_len, cost, n_iter, batch, k_pad,
                                     schemes, n_schemes, cand, cand_np, n_cand, trials, order,
                                     bound, best);
  } else {
    e = launch_trials<DP, false, 0>(grid, 0, s, sorted_len, cost, n_iter, batch, k_pad, schemes,
                                    n_schemes, cand, cand_np, n_cand, trials, order, bound, best);
    if (e == cudaSuccess)
      e = launch_trials<DP, false, 1>(grid, 0, s, sorted_len, cost, n_iter, batch, k_pad, schemes,
                                      n_schemes, cand, cand_np, n_cand, trials, order, bound,
                                      best);
  }
  if (e != cudaSuccess) return e;
  const dim3 rgrid((n_cand + kReplayThreads - 1) / kReplayThreads, n_iter);
  k_alg1_replay<DP><<<rgrid, kReplayThreads, 0, s>>>(
      sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, max_np,
      trials, order, reinterpret_cast<unsigned long long*>(best), pipe, lb, stats, members, status);
  note_launch();
  return cudaGetLastError();
}

size_t alg1_workspace(int n_iter) { return ((size_t)n_iter * 8 + 255) & ~(size_t)255; }

int launch_alg1(const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch, int k_pad,
                const hyd_scheme* schemes, int n_schemes, const uint8_t* cand,
                const uint8_t* cand_np, int n_cand, int max_np, int trials, const uint16_t* order,
                uint64_t* best, uint8_t* pipe, uint64_t* lb, hyd_pipe_stats* stats,
                uint32_t* members, uint32_t* status, void* ws, cudaStream_t s) {
  if (n_iter == 0 || n_cand == 0) return HYD_OK;
  uint64_t* bound = static_cast<uint64_t*>(ws);
  const int dp = max_np <= 2 ? 2 : max_np <= 4 ? 4 : max_np <= 8 ? 8 : max_np <= 16 ? 16 : 32;
  cudaError_t e;
  switch (dp) {
    case 2: e = launch_alg1_dp<2>(sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, max_np, trials, order, bound, best, pipe, lb, stats, members, status, s); break;
    case 4: e = launch_alg1_dp<4>(sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, max_np, trials, order, bound, best, pipe, lb, stats, members, status, s); break;
    case 8: e = launch_alg1_dp<8>(sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, max_np, trials, order, bound, best, pipe, lb, stats, members, status, s); break;
    case 16: e = launch_alg1_dp<16>(sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, max_np, trials, order, bound, best, pipe, lb, stats, members, status, s); break;
    default: e = launch_alg1_dp<32>(sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, max_np, trials, order, bound, best, pipe, lb, stats, members, status, s); break;
  }
  return e == cudaSuccess ? HYD_OK : record_cuda_error(e);
}

}  // namespace hyd
