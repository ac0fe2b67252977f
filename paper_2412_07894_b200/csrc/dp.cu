// dp.cu -- NEXT-3: the strategy-proposal dynamic programme (§5) on the GPU.
//
//   t[n][l] = min( t[n-1][l], min_{(k,d), l'} max( t[n - d N(P_k)][l - l'], (1/d) W_k(l - l', l) ) )
//   over MaxLen(P_k) >= l, d N(P_k) <= n, l' < l;  t[n][0] = 0, t[0][l > 0] = inf,
// with l = j step and n, d on a grid of 1/scale GPU (scale 1: the integer DP; scale 10: the
// continuous relaxation of P:701-713), W_k(a, b) = sum of T(x, P_k) over the dataset lengths
// in (a, b] (truncated to the context J step).  Values are exact rationals scale W / mu
// (128-bit cross-multiplied comparisons), ties broken by (carry, k, mu, j') ascending.
//
// Kernels: k_dp_hist (per-CTA shared histograms of sum T per (scheme, length bucket), one
// pass over the lengths), k_dp_scan (prefix sums per scheme), k_dp_solve (cooperative: one CTA
// per l, all levels n in order with a grid barrier between them -- level n reads only levels
// < n; the CTA's threads split the (k, d) pairs, each finds its best l' by binary search on the
// monotone halves of max(t, W/d), and the CTA reduces the lexicographic (value, choice) minimum), k_dp_strategy (thread per l: follow the recorded choices from
// (N, l), per-scheme d totals), k_dp_round (thread per l: floor/ceil of every d, within N GPUs),
// k_dp_unique (first occurrence of each rounded candidate).
#include <cooperative_groups.h>

#include "hyd_internal.cuh"

namespace cg = cooperative_groups;

namespace hyd {

constexpr int kDpThreads = 512;

// rationals num/den, den == 0: infinity
__device__ __forceinline__ bool q_less(uint64_t an, uint64_t ad, uint64_t bn, uint64_t bd) {
  if (bd == 0ull) return ad != 0ull;
  if (ad == 0ull) return false;
  uint64_t h1, l1, h2, l2;
  mul128(an, bd, h1, l1);
  mul128(bn, ad, h2, l2);
  return h1 < h2 || (h1 == h2 && l1 < l2);
}

// (value, choice) lexicographic
__device__ __forceinline__ bool key_less(uint64_t an, uint64_t ad, int32_t ac, uint64_t bn,
                                         uint64_t bd, int32_t bc) {
  if (q_less(an, ad, bn, bd)) return true;
  if (q_less(bn, bd, an, ad)) return false;
  return ac < bc;
}

__global__ void __launch_bounds__(256)
    k_dp_hist(const uint32_t* __restrict__ lengths, int n_seq, const hyd_scheme* __restrict__ schemes,
              int K, int step, int J, unsigned long long* __restrict__ bucket,
              uint32_t* __restrict__ status) {
  extern __shared__ unsigned long long s_b[];  // [K][J + 1]
  const int nb = K * (J + 1);
  for (int e = threadIdx.x; e < nb; e += blockDim.x) s_b[e] = 0ull;
  __syncthreads();
  const uint32_t lmax = (uint32_t)J * (uint32_t)step;
  uint32_t st = 0u;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_seq; i += gridDim.x * blockDim.x) {
    const uint32_t x0 = __ldg(lengths + i);
    const uint32_t x = x0 < lmax ? x0 : lmax;  // truncated to the context
    const int j = (int)((x + (uint32_t)step - 1u) / (uint32_t)step);
    for (int k = 0; k < K; ++k) {
      const uint32_t t = eval_cost(schemes[k].a_q32, schemes[k].b_q32, schemes[k].c_q32, x, st);
      atomicAdd(&s_b[k * (J + 1) + j], (unsigned long long)t);
    }
  }
  flag_warp(status, st);
  __syncthreads();
  for (int e = threadIdx.x; e < nb; e += blockDim.x)
    if (s_b[e]) atomicAdd(&bucket[e], s_b[e]);
}

__global__ void k_dp_scan(unsigned long long* __restrict__ pre, int J) {  // one warp per scheme
  unsigned long long* p = pre + (size_t)blockIdx.x * (J + 1);
  const int lane = threadIdx.x;
  unsigned long long carry = 0ull;
  for (int j0 = 0; j0 <= J; j0 += 32) {
    const int j = j0 + lane;
    unsigned long long v = j <= J ? p[j] : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(HYD_FULL, v, o);
      if (lane >= o) v += y;
    }
    v += carry;
    if (j <= J) p[j] = v;
    carry = __shfl_sync(HYD_FULL, v, 31);
  }
}

__global__ void __launch_bounds__(kDpThreads)
    k_dp_solve(const unsigned long long* __restrict__ pre, const hyd_scheme* __restrict__ schemes,
               int K, int step, int J, int NV, int scale, unsigned long long* __restrict__ t_num,
               unsigned long long* __restrict__ t_den, int32_t* __restrict__ choice) {
  extern __shared__ unsigned long long s_pre[];  // [K][J + 1]
  __shared__ uint32_t s_g[HYD_MAX_SCHEMES];
  __shared__ unsigned char s_ok[HYD_MAX_SCHEMES];
  __shared__ unsigned long long s_rn[kDpThreads / 32], s_rd[kDpThreads / 32];
  __shared__ int32_t s_rc[kDpThreads / 32];
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t W1 = (size_t)J + 1;
  for (int e = tid; e < K * (J + 1); e += kDpThreads) s_pre[e] = pre[e];
  for (int k = tid; k < K; k += kDpThreads) s_g[k] = schemes[k].tp * schemes[k].pp * schemes[k].cp;
  // level 0 and column 0; the CTA owns buckets j = blockIdx.x + 1 + r gridDim.x
  for (int j = blockIdx.x + 1 + tid * gridDim.x; j <= J; j += kDpThreads * gridDim.x) {
    t_num[j] = 1ull;
    t_den[j] = 0ull;
    choice[j] = -2;
  }
  if (blockIdx.x == 0)
    for (int nu = tid; nu <= NV; nu += kDpThreads) {
      t_num[(size_t)nu * W1] = 0ull;
      t_den[(size_t)nu * W1] = 1ull;
      choice[(size_t)nu * W1] = -2;
    }
  __syncthreads();
  grid.sync();
  for (int nu = 1; nu <= NV; ++nu) {
   for (int j = blockIdx.x + 1; j <= J; j += gridDim.x) {
    __syncthreads();
    for (int k = tid; k < K; k += kDpThreads)
      s_ok[k] = schemes[k].max_len >= (uint32_t)j * (uint32_t)step;  // MaxLen(P_k) >= l
    __syncthreads();
    // candidate: carry t[nu - 1][j] (choice -1), then every (k, mu, j')
    uint64_t bn = t_num[(size_t)(nu - 1) * W1 + j], bd = t_den[(size_t)(nu - 1) * W1 + j];
    int32_t bc = -1;
    // (k, mu) pairs split over the threads; for each pair the best l' by binary search:
    // f(j') = t[nu - mu N_k][j - j'] is non-increasing in j' (t is non-decreasing in l) and
    // g(j') = scale W_k(j - j', j) / mu non-decreasing, so max(f, g) falls then rises -- its
    // minimum is at the first j' with g >= f (value g) or just before it (value f, taken at the
    // first j' of f's plateau); the smaller (value, j') of the two is the exact argmin the
    // enumeration of every j' would return (ties: smaller j', as the choice code orders them).
    const unsigned long long* ppre = s_pre;
    int pair = 0;
    for (int k = 0; k < K; ++k) {
      if (!s_ok[k]) continue;
      const int mumax = nu / (int)s_g[k];
      const unsigned long long* pk = ppre + (size_t)k * W1;
      const unsigned long long pj = pk[j];
      const uint64_t g1 = (uint64_t)scale * (pj - pk[j - 1]);  // mu g(1): W_k over the last bucket
      for (int mu = 1 + ((tid - pair) % kDpThreads + kDpThreads) % kDpThreads; mu <= mumax;
           mu += kDpThreads) {
        // every value of the pair is >= g(1) = g1 / mu (g is non-decreasing in j', f >= 0): a pair
        // whose bound already exceeds this thread's best cannot win, nor tie (exact pruning)
        if (q_less(bn, bd, g1, (uint64_t)mu)) continue;
        const size_t rbase = (size_t)(nu - mu * (int)s_g[k]) * W1 + j;  // f(j') = t[rbase - j']
        auto f_at = [&](int jp, uint64_t& fn, uint64_t& fd) {
          fn = t_num[rbase - jp];
          fd = t_den[rbase - jp];
        };
        auto g_at = [&](int jp, uint64_t& gn, uint64_t& gd) {
          gn = (uint64_t)scale * (pj - pk[j - jp]);
          gd = (uint64_t)mu;
        };
        // c = first j' in [1, j] with g >= f (j + 1 if none)
        int lo = 1, hi = j + 1;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          uint64_t fn, fd, gn, gd;
          f_at(mid, fn, fd);
          g_at(mid, gn, gd);
          if (!q_less(gn, gd, fn, fd)) hi = mid;
          else lo = mid + 1;
        }
        const int c = lo;
        const uint32_t codebase = ((uint32_t)k << 24) | ((uint32_t)mu << 12);
        if (c <= j) {  // candidate A: j' = c, value g(c)
          uint64_t gn, gd;
          g_at(c, gn, gd);
          const int32_t code = (int32_t)(codebase | (uint32_t)c);
          if (key_less(gn, gd, code, bn, bd, bc)) {
            bn = gn;
            bd = gd;
            bc = code;
          }
        }
        if (c > 1) {  // candidate B: value f(c - 1), at the first j' of its plateau
          uint64_t vn, vd;
          f_at(c - 1, vn, vd);
          int l2 = 1, h2 = c - 1;  // first j' in [1, c - 1] with f(j') <= f(c - 1)
          while (l2 < h2) {
            const int mid = (l2 + h2) >> 1;
            uint64_t fn, fd;
            f_at(mid, fn, fd);
            if (!q_less(vn, vd, fn, fd)) h2 = mid;  // f(mid) <= v
            else l2 = mid + 1;
          }
          const int32_t code = (int32_t)(codebase | (uint32_t)l2);
          if (key_less(vn, vd, code, bn, bd, bc)) {
            bn = vn;
            bd = vd;
            bc = code;
          }
        }
      }
      pair += mumax;
    }
    // block-wide lexicographic minimum
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t on = __shfl_xor_sync(HYD_FULL, bn, o), od = __shfl_xor_sync(HYD_FULL, bd, o);
      const int32_t oc = __shfl_xor_sync(HYD_FULL, bc, o);
      if (key_less(on, od, oc, bn, bd, bc)) {
        bn = on;
        bd = od;
        bc = oc;
      }
    }
    if (lane == 0) {
      s_rn[warp] = bn;
      s_rd[warp] = bd;
      s_rc[warp] = bc;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < kDpThreads / 32; ++w)
        if (key_less(s_rn[w], s_rd[w], s_rc[w], bn, bd, bc)) {
          bn = s_rn[w];
          bd = s_rd[w];
          bc = s_rc[w];
        }
      t_num[(size_t)nu * W1 + j] = bn;
      t_den[(size_t)nu * W1 + j] = bd;
      choice[(size_t)nu * W1 + j] = bc;
    }
   }
    grid.sync();  // level nu complete everywhere before level nu + 1 reads it
  }
}

// thread per j: S[N][j step] -> per-scheme d totals (1/scale units), scheme of the longest interval
__global__ void k_dp_strategy(const int32_t* __restrict__ choice,
                              const unsigned long long* __restrict__ t_den,
                              const hyd_scheme* __restrict__ schemes, int K, int J, int NV,
                              uint16_t* __restrict__ counts, uint8_t* __restrict__ top) {
  const int j0 = blockIdx.x * blockDim.x + threadIdx.x;
  if (j0 > J) return;
  uint16_t* cnt = counts + (size_t)j0 * K;
  for (int k = 0; k < K; ++k) cnt[k] = 0;
  top[j0] = 0xFF;
  const size_t W1 = (size_t)J + 1;
  if (j0 == 0 || t_den[(size_t)NV * W1 + j0] == 0ull) return;
  int nu = NV, j = j0;
  while (j > 0) {
    const int32_t c = choice[(size_t)nu * W1 + j];
    if (c == -1) {
      --nu;
      continue;
    }
    const uint32_t k = (uint32_t)c >> 24, mu = ((uint32_t)c >> 12) & 0xFFFu, jp = (uint32_t)c & 0xFFFu;
    if (top[j0] == 0xFF) top[j0] = (uint8_t)k;
    cnt[k] = (uint16_t)(cnt[k] + mu);
    nu -= (int)(mu * schemes[k].tp * schemes[k].pp * schemes[k].cp);
    j -= (int)jp;
  }
}

// thread per j: integer candidates near the relaxed strategy (reading 27): every
// scheme with d_k > 0 takes floor or ceil of d_k (combinations in binary order over the used
// schemes, ascending k), kept if within N GPUs and the longest interval's scheme keeps a pipeline
__global__ void k_dp_round(const uint16_t* __restrict__ counts, const uint8_t* __restrict__ top,
                           const hyd_scheme* __restrict__ schemes, int K, int J, int n_gpus,
                           int scale, uint8_t* __restrict__ rows, uint8_t* __restrict__ valid,
                           uint32_t* __restrict__ status) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j > J) return;
  const uint16_t* cnt = counts + (size_t)j * K;
  uint8_t* out = rows + (size_t)j * HYD_DP_MAX_ROUND * K;
  uint8_t* ok = valid + (size_t)j * HYD_DP_MAX_ROUND;
  for (int r = 0; r < HYD_DP_MAX_ROUND; ++r) ok[r] = 0;
  if (top[j] == 0xFF) return;
  int frac_k[HYD_MAX_SCHEMES];
  int nf = 0;
  for (int k = 0; k < K; ++k)
    if (cnt[k] % scale != 0) frac_k[nf++] = k;  // schemes whose d is not an integer
  if ((1 << min(nf, 30)) > HYD_DP_MAX_ROUND) {
    flag(status, HYD_F_OVERFLOW);
    return;
  }
  for (int m = 0; m < (1 << nf); ++m) {
    uint8_t* row = out + (size_t)m * K;
    uint64_t g = 0ull;
    int q = 0;
    for (int k = 0; k < K; ++k) {
      int n = cnt[k] / scale;
      if (q < nf && frac_k[q] == k) {
        n += (m >> q) & 1;  // bit q of m: ceil for the q-th fractional scheme
        ++q;
      }
      row[k] = (uint8_t)min(n, 255);
      g += (uint64_t)n * schemes[k].tp * schemes[k].pp * schemes[k].cp;
    }
    ok[m] = g <= (uint64_t)n_gpus && row[top[j]] >= 1;
  }
}

// first occurrence (in (j, r) order) of every valid rounded candidate
__global__ void k_dp_unique(const uint8_t* __restrict__ rows, const uint8_t* __restrict__ valid,
                            int K, int M, uint8_t* __restrict__ keep) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  if (!valid[m]) {
    keep[m] = 0;
    return;
  }
  const uint8_t* a = rows + (size_t)m * K;
  for (int p = 0; p < m; ++p) {
    if (!valid[p]) continue;
    const uint8_t* b = rows + (size_t)p * K;
    bool same = true;
    for (int k = 0; k < K && same; ++k) same = a[k] == b[k];
    if (same) {
      keep[m] = 0;
      return;
    }
  }
  keep[m] = 1;
}

// The proposed subset (keep = 1, in (j, r) order) as candidate tables the assignment takes:
// pipelines in canonical order (MaxLen non-increasing, scheme index ascending: P:623), each
// scheme repeated by its pipeline count.  One CTA: a block-wide exclusive scan of keep gives
// each kept row its output index; a row with more than HYD_MAX_PIPES pipelines gets cand_np 0.
constexpr int kDpCandThreads = 1024;
__global__ void __launch_bounds__(kDpCandThreads)
    k_dp_candidates(const uint8_t* __restrict__ rows, const uint8_t* __restrict__ keep, int M,
                    const hyd_scheme* __restrict__ schemes, int K, uint8_t* __restrict__ cand,
                    uint8_t* __restrict__ cand_np, int32_t* __restrict__ n_out) {
  __shared__ uint8_t s_order[HYD_MAX_SCHEMES];  // canonical position -> scheme
  __shared__ int s_warp[kDpCandThreads / 32];
  __shared__ int s_base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < K) {  // rank of scheme tid in (MaxLen desc, k asc)
    const uint32_t m = schemes[tid].max_len;
    int r = 0;
    for (int q = 0; q < K; ++q) {
      const uint32_t mq = schemes[q].max_len;
      r += (mq > m || (mq == m && q < tid)) ? 1 : 0;
    }
    s_order[r] = (uint8_t)tid;
  }
  if (tid == 0) s_base = 0;
  __syncthreads();
  for (int m0 = 0; m0 < M; m0 += kDpCandThreads) {
    const int m = m0 + tid;
    const int kp = (m < M && keep[m]) ? 1 : 0;
    const unsigned bal = __ballot_sync(HYD_FULL, kp);
    if (lane == 0) s_warp[warp] = __popc(bal);
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the warp counts
      int x = s_warp[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(HYD_FULL, x, o);
        if (lane >= o) x += y;
      }
      s_warp[lane] = x - s_warp[lane];
    }
    __syncthreads();
    const int at = s_base + s_warp[warp] + __popc(bal & ((1u << lane) - 1u));
    if (kp) {
      const uint8_t* row = rows + (size_t)m * K;
      uint8_t* out = cand + (size_t)at * HYD_MAX_PIPES;
      int n = 0;
      for (int q = 0; q < K; ++q) {
        const int k = s_order[q];
        for (int r = 0; r < (int)row[k]; ++r, ++n)
          if (n < HYD_MAX_PIPES) out[n] = (uint8_t)k;
      }
      for (int q = n; q < HYD_MAX_PIPES; ++q) out[q] = 0xFF;
      cand_np[at] = n <= HYD_MAX_PIPES ? (uint8_t)n : 0;
    }
    __syncthreads();
    if (tid == kDpCandThreads - 1) s_base = at + kp;
    __syncthreads();
  }
  if (tid == 0) *n_out = s_base;
}

int launch_dp_candidates(const uint8_t* rows, const uint8_t* keep, int J, const hyd_scheme* schemes, int K,
                         uint8_t* cand, uint8_t* cand_np, int32_t* n_out, cudaStream_t s) {
  const int M = (J + 1) * HYD_DP_MAX_ROUND;
  k_dp_candidates<<<1, kDpCandThreads, 0, s>>>(rows, keep, M, schemes, K, cand, cand_np, n_out);
  note_launch();
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HYD_OK : record_cuda_error(e);
}

size_t dp_workspace(int K, int J) {
  return ((size_t)K * (J + 1) * 8 + 255) & ~(size_t)255;  // prefix sums
}

int launch_dp(const uint32_t* lengths, int n_seq, const hyd_scheme* schemes, int K, int step,
              int J, int n_gpus, int scale, uint64_t* t_num, uint64_t* t_den, int32_t* choice,
              uint16_t* counts, uint8_t* rows, uint8_t* valid, uint8_t* keep, uint32_t* status,
              void* ws, cudaStream_t s) {
  auto* pre = static_cast<unsigned long long*>(ws);
  const size_t npre = (size_t)K * (J + 1);
  cudaError_t e = cudaMemsetAsync(pre, 0, npre * 8, s);
  if (e != cudaSuccess) return record_cuda_error(e);
  const size_t smem = npre * 8;
  e = cudaFuncSetAttribute(k_dp_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return record_cuda_error(e);
  const int hb = max(1, min(296, (n_seq + 255) / 256));
  k_dp_hist<<<hb, 256, smem, s>>>(lengths, n_seq, schemes, K, step, J, pre, status);
  note_launch();
  k_dp_scan<<<K, 32, 0, s>>>(pre, J);
  note_launch();
  e = cudaFuncSetAttribute(k_dp_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return record_cuda_error(e);
  const int NV = n_gpus * scale;
  const unsigned long long* pre_c = pre;
  auto* tn = reinterpret_cast<unsigned long long*>(t_num);
  auto* td = reinterpret_cast<unsigned long long*>(t_den);
  void* args[] = {(void*)&pre_c, (void*)&schemes, (void*)&K, (void*)&step, (void*)&J,
                  (void*)&NV, (void*)&scale, (void*)&tn, (void*)&td, (void*)&choice};
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dp_solve, kDpThreads, smem);
  if (e != cudaSuccess || per_sm < 1) return record_cuda_error(e != cudaSuccess ? e : cudaErrorInvalidConfiguration);
  const int grid = min(J, per_sm * sms);  // co-resident for the grid barrier
  e = cudaLaunchCooperativeKernel((const void*)k_dp_solve, dim3(grid), dim3(kDpThreads), args, smem, s);
  note_launch();
  if (e != cudaSuccess) return record_cuda_error(e);
  const int tb = (J + 1 + 127) / 128;
  k_dp_strategy<<<tb, 128, 0, s>>>(choice, td, schemes, K, J, NV, counts, reinterpret_cast<uint8_t*>(keep));
  note_launch();
  // `keep` doubles as the top-scheme scratch until the rounding consumed it
  k_dp_round<<<tb, 128, 0, s>>>(counts, keep, schemes, K, J, n_gpus, scale, rows, valid, status);
  note_launch();
  const int M = (J + 1) * HYD_DP_MAX_ROUND;
  k_dp_unique<<<(M + 255) / 256, 256, 0, s>>>(rows, valid, K, M, keep);
  note_launch();
  e = cudaGetLastError();
  return e == cudaSuccess ? HYD_OK : record_cuda_error(e);
}

}  // namespace hyd
