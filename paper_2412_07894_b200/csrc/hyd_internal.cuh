// hyd_internal.cuh -- device helpers shared by the libhyd.so kernels (product path only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/hyd.h"

#define HYD_FULL 0xFFFFFFFFu
#define HYD_LEN_LIMIT (1u << 24)
#define HYD_MAKESPAN_LIMIT (1ull << 43)

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

__device__ __forceinline__ int next_pow2_ge(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

}  // namespace hyd
