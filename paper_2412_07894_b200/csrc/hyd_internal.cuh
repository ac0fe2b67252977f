// hyd_internal.cuh -- device helpers shared by the libhyd.so kernels (product path only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/hyd.h"

#define HYD_FULL 0xFFFFFFFFu
#define HYD_LEN_LIMIT (1u << 24)
#define HYD_MAKESPAN_LIMIT (1ull << 43)

// Debug builds (libhyd_debug.so, -DHYD_DEBUG_CHECKS; tools/sanitize_cases.py): bounds checks on
// the shared-memory and global indices the kernels compute; a failed check prints its site and
// traps the kernel (the call then returns HYD_E_CUDA).  compute-sanitizer is closed on this GPU
// pool, so this build is the memory-safety check of the test plan.
#ifdef HYD_DEBUG_CHECKS
#include <cstdio>
#define HYD_CHECK(cond)                                                                      \
  do {                                                                                       \
    if (!(cond)) {                                                                           \
      printf("HYD_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
             (int)blockIdx.x, (int)threadIdx.x);                                             \
      __trap();                                                                              \
    }                                                                                        \
  } while (0)
#else
#define HYD_CHECK(cond) \
  do {                  \
  } while (0)
#endif

namespace hyd {

// Launch bookkeeping (diagnostics only): counts kernels this library launched.
void note_launch();
int record_cuda_error(cudaError_t e);

__device__ __forceinline__ void flag(uint32_t* status, uint32_t bits) {
  if (bits) atomicOr(status, bits);
}

// Warp-aggregated status OR: one atomic per warp per distinct call site.
__device__ __forceinline__ void flag_warp(uint32_t* status, uint32_t bits) {
  uint32_t all = __reduce_or_sync(__activemask(), bits);
  if (all && (threadIdx.x & 31) == __ffs(__activemask()) - 1) atomicOr(status, all);
}

// 64x64 -> 128-bit product as (hi, lo)
__device__ __forceinline__ void mul128(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
  lo = a * b;
  hi = __umul64hi(a, b);
}

// (ahi:alo) > (bhi:blo)
__device__ __forceinline__ bool gt128(uint64_t ahi, uint64_t alo, uint64_t bhi, uint64_t blo) {
  return ahi > bhi || (ahi == bhi && alo > blo);
}

// Batch geometry (NEXT-2, token-budget batches): iteration t holds geo_bt(t) sequences whose rows
// start at geo_base(t) in every iteration-indexed array ([N_total] lengths, [C][N_total] pipe/mb,
// ...).  off = nullptr: the uniform case, B sequences per iteration; otherwise off[0..It] are CSR
// offsets and B is the largest batch (bt is clamped to [0, B]; sort_cost flags violations).
__device__ __forceinline__ int geo_bt(const uint32_t* off, int B, int t) {
  if (!off) return B;
  const int d = (int)(__ldg(off + t + 1) - __ldg(off + t));
  return d < 0 ? 0 : (d > B ? B : d);
}
__device__ __forceinline__ size_t geo_base(const uint32_t* off, int B, int t) {
  return off ? (size_t)__ldg(off + t) : (size_t)t * B;
}
__device__ __forceinline__ size_t geo_total(const uint32_t* off, int B, int n_iter) {
  return off ? (size_t)__ldg(off + n_iter) : (size_t)n_iter * B;
}

// T(l) with a 128-bit intermediate; status bits per include/hyd.h.
__device__ __forceinline__ uint32_t eval_cost(uint64_t a, uint64_t b, uint64_t c, uint32_t l,
                                              uint32_t& st) {
  if (l == 0u || l > HYD_LEN_LIMIT) {
    st |= HYD_F_BAD_LENGTH;
    return 0xFFFFFFFFu;
  }
  const uint64_t l2 = (uint64_t)l * (uint64_t)l;  // < 2^49
  uint64_t hi1, lo1, hi2, lo2;
  mul128(a, l2, hi1, lo1);
  mul128(b, (uint64_t)l, hi2, lo2);
  uint64_t lo = lo1 + lo2;
  uint64_t hi = hi1 + hi2 + (lo < lo1 ? 1ull : 0ull);
  const uint64_t lo3 = lo + c;
  hi += (lo3 < lo) ? 1ull : 0ull;
  // T = (hi:lo3) >> 32 = hi * 2^32 + (lo3 >> 32): fits u32 iff hi == 0
  if (hi != 0ull) {
    st |= HYD_F_OVERFLOW;
    return 0xFFFFFFFFu;
  }
  const uint32_t t = (uint32_t)(lo3 >> 32);
  if (t == 0u) st |= HYD_F_ZERO_COST;
  return t;
}

// min of m[0..N) as a ternary tree: ptxas fuses min(min(a, b), c) into one 3-input VIMNMX3, so
// N keys take about N/2 instructions instead of N - 1 (e.g. 8 -> 4, 16 -> 8, 32 -> 17).
// Overwrites m.
template <int N, int A>
__device__ __forceinline__ uint32_t min_tree3(uint32_t (&m)[A]) {
  static_assert(N >= 1 && N <= A, "min_tree3 size");
  if constexpr (N == 1) {
    return m[0];
  } else if constexpr (N == 2) {
    return min(m[0], m[1]);
  } else {
#pragma unroll
    for (int i = 0; i < N / 3; ++i) m[i] = min(min(m[3 * i], m[3 * i + 1]), m[3 * i + 2]);
    if constexpr (N % 3 == 1) m[N / 3] = m[N - 1];
    if constexpr (N % 3 == 2) m[N / 3] = min(m[N - 2], m[N - 1]);
    return min_tree3<(N + 2) / 3, A>(m);
  }
}

__device__ __forceinline__ int next_pow2_ge(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

}  // namespace hyd
