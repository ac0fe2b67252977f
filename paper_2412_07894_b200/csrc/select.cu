// select.cu -- a5: per-iteration argmin of makespan over candidates (step ④),
// and the winner gather used by the end-to-end call.
//
// k_select: one warp per iteration, lanes stride the makespan row (coalesced 8-byte
// loads), key = makespan << 20 | c_global (argmin of (makespan, c) == min key), then a
// 5-step shuffle min.  k_select_cta: rows of more than 512 candidates get a CTA each
// (~16 candidates per thread, shuffle + shared-memory min), so few long rows (config 5: 16
// iterations x 16 384 candidates) do not serialise on 16 warps.  Across GPUs the caller
// allreduces key with MIN over NCCL.
#include "hyd_internal.cuh"

namespace hyd {

__global__ void __launch_bounds__(256) k_select(const uint64_t* __restrict__ makespan, int n_iter,
                                                int n_cand, int cand_offset,
                                                int64_t* __restrict__ key,
                                                uint32_t* __restrict__ status) {
  const int w = (int)((blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= n_iter) return;
  const uint64_t* row = makespan + (size_t)w * n_cand;
  long long best = 0x7FFFFFFFFFFFFFFFll;
  uint32_t st = 0;
  for (int c = lane; c < n_cand; c += 32) {
    const uint64_t m = __ldg(reinterpret_cast<const unsigned long long*>(row) + c);
    if (m == ~0ull) continue;  // infeasible candidate
    if (m >= HYD_MAKESPAN_LIMIT) {
      st |= HYD_F_KEY_RANGE;
      continue;
    }
    const long long k = (long long)((m << HYD_KEY_SHIFT) | (uint64_t)(c + cand_offset));
    best = k < best ? k : best;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long y = __shfl_xor_sync(HYD_FULL, best, o);
    best = y < best ? y : best;
  }
  st = __reduce_or_sync(HYD_FULL, st);
  if (lane == 0) {
    key[w] = best;
    if (st) atomicOr(status, st);
  }
}

__device__ __forceinline__ long long select_key(uint64_t m, int c, int cand_offset, uint32_t& st) {
  if (m == ~0ull) return 0x7FFFFFFFFFFFFFFFll;  // infeasible candidate
  if (m >= HYD_MAKESPAN_LIMIT) {
    st |= HYD_F_KEY_RANGE;
    return 0x7FFFFFFFFFFFFFFFll;
  }
  return (long long)((m << HYD_KEY_SHIFT) | (uint64_t)(c + cand_offset));
}

__global__ void __launch_bounds__(1024) k_select_cta(const uint64_t* __restrict__ makespan, int n_iter,
                                                     int n_cand, int cand_offset,
                                                     int64_t* __restrict__ key,
                                                     uint32_t* __restrict__ status) {
  __shared__ long long s_best[32];
  __shared__ uint32_t s_st;
  const int t = blockIdx.x, tid = threadIdx.x, lane = tid & 31, nt = blockDim.x;
  const unsigned long long* row = reinterpret_cast<const unsigned long long*>(makespan) + (size_t)t * n_cand;
  if (tid == 0) s_st = 0u;
  long long best = 0x7FFFFFFFFFFFFFFFll;
  uint32_t st = 0;
  int c = tid;
  for (; c + 3 * nt < n_cand; c += 4 * nt) {  // four independent loads in flight per thread
    const uint64_t m0 = __ldg(row + c), m1 = __ldg(row + c + nt), m2 = __ldg(row + c + 2 * nt),
                   m3 = __ldg(row + c + 3 * nt);
    best = min(best, min(min(select_key(m0, c, cand_offset, st), select_key(m1, c + nt, cand_offset, st)),
                         min(select_key(m2, c + 2 * nt, cand_offset, st), select_key(m3, c + 3 * nt, cand_offset, st))));
  }
  for (; c < n_cand; c += nt) best = min(best, select_key(__ldg(row + c), c, cand_offset, st));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(HYD_FULL, best, o));
  st = __reduce_or_sync(HYD_FULL, st);
  __syncthreads();  // s_st initialised
  if (lane == 0) {
    s_best[tid >> 5] = best;
    if (st) atomicOr(&s_st, st);
  }
  __syncthreads();
  if (tid < 32) {
    best = tid < (nt >> 5) ? s_best[tid] : 0x7FFFFFFFFFFFFFFFll;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(HYD_FULL, best, o));
    if (tid == 0) {
      key[t] = best;
      if (s_st) atomicOr(status, s_st);
    }
  }
}

__global__ void __launch_bounds__(256) k_gather(const int64_t* __restrict__ key,
                                                const uint32_t* __restrict__ perm,
                                                const uint8_t* __restrict__ pipe,
                                                const uint16_t* __restrict__ mb,
                                                const uint16_t* __restrict__ v,
                                                const uint64_t* __restrict__ ptime, int n_iter,
                                                int batch, const uint32_t* __restrict__ off,
                                                size_t n_total, int n_cand, int cand_offset,
                                                uint8_t* __restrict__ win_pipe,
                                                uint16_t* __restrict__ win_mb,
                                                uint16_t* __restrict__ win_v,
                                                uint64_t* __restrict__ win_ptime) {
  const int t = blockIdx.x;
  const long long k = key[t];
  if (k == 0x7FFFFFFFFFFFFFFFll) return;
  const int c = (int)(k & ((1ll << HYD_KEY_SHIFT) - 1)) - cand_offset;
  if (c < 0 || c >= n_cand) return;  // another rank owns the winner
  const size_t row = (size_t)c * n_iter + t;
  const size_t base = geo_base(off, batch, t);
  const int bt = geo_bt(off, batch, t);
  const uint32_t* pr = perm + base;
  const size_t src = (size_t)c * n_total + base;
  for (int i = threadIdx.x; i < bt; i += blockDim.x) {
    const uint32_t o = pr[i];
    win_pipe[base + o] = pipe[src + i];
    win_mb[base + o] = mb[src + i];
  }
  if (threadIdx.x < HYD_MAX_PIPES) {
    win_v[(size_t)t * HYD_MAX_PIPES + threadIdx.x] = v[row * HYD_MAX_PIPES + threadIdx.x];
    win_ptime[(size_t)t * HYD_MAX_PIPES + threadIdx.x] = ptime[row * HYD_MAX_PIPES + threadIdx.x];
  }
}

int launch_select(const uint64_t* makespan, int n_iter, int n_cand, int cand_offset, int64_t* key,
                  uint32_t* status, cudaStream_t s) {
  if (n_iter == 0) return HYD_OK;
  if (n_cand > 512) {
    const int nt = min(1024, ((n_cand + 16 * 32 - 1) / (16 * 32)) * 32);  // ~16 candidates per thread
    k_select_cta<<<n_iter, nt, 0, s>>>(makespan, n_iter, n_cand, cand_offset, key, status);
  } else {
    const int blocks = (n_iter * 32 + 255) / 256;
    k_select<<<blocks, 256, 0, s>>>(makespan, n_iter, n_cand, cand_offset, key, status);
  }
  note_launch();
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HYD_OK : record_cuda_error(e);
}

int launch_gather(const int64_t* key, const uint32_t* perm, const uint8_t* pipe, const uint16_t* mb,
                  const uint16_t* v, const uint64_t* ptime, int n_iter, int batch,
                  const uint32_t* off, size_t n_total, int n_cand, int cand_offset, uint8_t* win_pipe, uint16_t* win_mb, uint16_t* win_v,
                  uint64_t* win_ptime, cudaStream_t s) {
  if (n_iter == 0) return HYD_OK;
  k_gather<<<n_iter, 256, 0, s>>>(key, perm, pipe, mb, v, ptime, n_iter, batch, off, n_total, n_cand, cand_offset,
                                  win_pipe, win_mb, win_v, win_ptime);
  note_launch();
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HYD_OK : record_cuda_error(e);
}

}  // namespace hyd
