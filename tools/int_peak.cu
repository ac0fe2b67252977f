// int_peak.cu -- integer-issue ceiling of the B200 for the instruction mix of the LPT bin loops
// (the "alu" roofline denominator of bench.py; tools/int_peak.py runs it and writes
// profiles/rNN/int_peak.json).
//
// Every kernel runs a loop of independent 32-bit integer chains (8 per thread, so dependent
// latency never binds) at full occupancy (148 x 8 CTAs of 256 threads) and counts lane-ops:
//   mix_pack:  one LPT bin evaluation per chain and step as k_pack_lanes issues it -- capacity
//              mask (IADD3 rem-l, LOP3 & 2^31 | key), a min (IMNMX), a compare + predicated
//              placement (ISETP + 2 predicated IADD3)  = 6 ops;
//   iadd3:     IADD3 only;   imnmx: min (ptxas: VIMNMX3, 3-input);   lop3: LOP3 only;
//   isetp_sel: ISETP + predicated LOP3 pairs (compare, then a predicated update).
// The values depend on a runtime seed and are stored, so nothing folds away; the SASS is
// checked by tools/int_peak.py (cuobjdump) to hold the intended instruction classes.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {
constexpr int kChains = 8;

__global__ void __launch_bounds__(256) k_mix_pack(uint32_t seed, int iters, uint32_t* out) {
  uint32_t key[kChains], rem[kChains], mk[kChains];
  const uint32_t l = (seed >> 3) | 1u, tau = seed & 0xFFu;
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    key[c] = seed * (c + 1) + threadIdx.x;
    rem[c] = seed ^ (c * 977u);
    mk[c] = seed + c;
  }
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      const uint32_t m = key[c] | ((rem[c] - l) & 0x80000000u);  // IADD3 + LOP3
      mk[c] = min(mk[c], m);                                     // IMNMX
      asm volatile("{\n\t.reg .pred p;\n\t"                    // ISETP + 2 predicated IADD3
                   "setp.eq.u32 p, %0, %2;\n\t"
                   "@p add.u32 %0, %0, %3;\n\t"
                   "@p sub.u32 %1, %1, %4;\n\t}"
                   : "+r"(key[c]), "+r"(rem[c])
                   : "r"(mk[c]), "r"(tau), "r"(l));
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc ^= key[c] + rem[c] + mk[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int OP>
__global__ void __launch_bounds__(256) k_single(uint32_t seed, int iters, uint32_t* out) {
  uint32_t x[kChains];
  const uint32_t a = seed | 1u, b = seed >> 7;
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = seed * (c + 3) + threadIdx.x;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        if constexpr (OP == 0) {
          asm volatile("add.u32 %0, %0, %1;" : "+r"(x[c]) : "r"(a));
        } else if constexpr (OP == 1) {
          asm volatile("min.u32 %0, %0, %1;" : "+r"(x[c]) : "r"(a + (uint32_t)r));
        } else if constexpr (OP == 2) {
          asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(a), "r"(b));
        } else {
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, %1;\n\t@p xor.b32 %0, %0, %2;\n\t}"
                       : "+r"(x[c]) : "r"(a + (uint32_t)r), "r"(b));
        }
      }
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc ^= x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
}  // namespace

extern "C" {
// kind: 0 mix_pack, 1 iadd3, 2 imnmx, 3 lop3, 4 isetp_sel.  Returns lane-ops per thread per
// iteration (the caller multiplies by threads x iters), or -1 on a launch error.
int int_peak_launch(int kind, int blocks, int iters, uint32_t seed, uint32_t* out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  switch (kind) {
    case 0: k_mix_pack<<<blocks, 256, 0, s>>>(seed, iters, out); break;
    case 1: k_single<0><<<blocks, 256, 0, s>>>(seed, iters, out); break;
    case 2: k_single<1><<<blocks, 256, 0, s>>>(seed, iters, out); break;
    case 3: k_single<2><<<blocks, 256, 0, s>>>(seed, iters, out); break;
    case 4: k_single<3><<<blocks, 256, 0, s>>>(seed, iters, out); break;
    default: return -1;
  }
  if (cudaGetLastError() != cudaSuccess) return -1;
  // lane-ops per thread and iteration: mix 7 per chain + 1 (mk ^= it); singles 4 (isetp_sel 8)
  return kind == 0 ? 6 * kChains : kind == 4 ? 8 * kChains : 4 * kChains;
}
}
