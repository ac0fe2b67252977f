// search.cuh -- the exact pruned search over V of App. D's range for one pipeline,
// shared by the packing kernels (pack.cu: k_pack_lanes / k_pack_big; small.cu: the fused
// small-batch kernel).  See pack.cu's header comment for the pruning argument.
#pragma once
#include "hyd_internal.cuh"

namespace hyd {

// ------------------------------------------------------------------ exact V search state
struct Search {
  uint64_t S, sumT, best;
  uint32_t U, M, P, UL, tau_max, vlo, vhi, va, cursor, vbest;
  int phase;
  bool have;
};

__device__ __forceinline__ uint32_t ceil_div_small(uint64_t n, uint32_t d) {
  // n / d rounded up, with a 32-bit division when n fits
  return n < 0xFFFFFFFFull - d ? ((uint32_t)n + d - 1u) / d : (uint32_t)((n + d - 1) / d);
}

__device__ __forceinline__ void search_init(Search& s) {
  const uint32_t vlo = max(ceil_div_small(s.S, s.M), 1u);
  uint32_t vhi = s.U;
  if (s.UL) {
    const uint64_t q = s.S < 0xFFFFFFFFull ? (uint64_t)((uint32_t)s.S / s.UL) : s.S / s.UL;
    vhi = q < (uint64_t)s.U ? (uint32_t)q : s.U;
  }
  if (vhi < vlo) vhi = vlo;
  s.vlo = vlo;
  s.vhi = vhi;
  uint32_t va = s.vlo;
  if (s.P > 1 && s.tau_max > 0) {
    const float vc = (float)s.sumT / (float)s.tau_max;
    const float vcl = fminf(fmaxf(vc + 0.5f, (float)s.vlo), (float)s.vhi);
    va = (uint32_t)vcl;
    va = min(max(va, s.vlo), s.vhi);
  }
  s.va = va;
  s.cursor = s.vlo;
  s.phase = 0;
  s.have = false;
  s.best = 0;
  s.vbest = 0;
}

// next V to evaluate, 0 when the search is complete
__device__ __forceinline__ uint32_t search_next(Search& s) {
  if (s.phase == 0) {
    s.phase = 1;
    return s.va;
  }
  if (s.phase == 1) {
    while (s.cursor <= s.vhi) {
      const uint32_t V = s.cursor++;
      if (V == s.va) continue;
      if (s.have) {
        const uint64_t m = (uint64_t)(s.P - 1 + V);
        const uint64_t tb = (uint64_t)s.tau_max * m;
        if (tb > s.best || (tb >= s.best && V > s.vbest)) {
          s.cursor = s.vhi + 1;  // tau_max (PP-1+V) grows with V: no later V can win
          break;
        }
        uint64_t ah, al, bh, bl;
        mul128(s.sumT, m, ah, al);
        mul128(s.best, (uint64_t)V, bh, bl);
        if (gt128(ah, al, bh, bl)) continue;                          // LB(V) > best
        if (!gt128(bh, bl, ah, al) && V > s.vbest) continue;          // LB(V) >= best, larger V
      }
      return V;
    }
    s.phase = 2;
    s.cursor = s.vhi + 1;
  }
  if (s.phase == 2) {
    if (!s.have && s.cursor <= s.U) return s.cursor++;  // extension above the range (reading 5)
    s.phase = 3;
  }
  return 0;
}

// A bin-time ceiling for early abort that is never below the exact one (the exact test
// is repeated when a run completes): floor(best/(PP-1+V)) estimated in fp32 with slack.
__device__ __forceinline__ uint64_t search_thr_approx(const Search& s, uint32_t V) {
  if (!s.have) return ~0ull;
  const float q = (float)s.best / (float)(s.P - 1 + V);
  return (uint64_t)(q * 1.0001f) + 2ull;
}

// exact: does LPT(V) with this max bin time improve (best, V_best)?
__device__ __forceinline__ bool search_improves(const Search& s, uint32_t V, uint64_t maxbin) {
  if (!s.have) return true;
  const uint64_t obj = maxbin * (uint64_t)(s.P - 1 + V);
  return obj < s.best || (obj == s.best && V < s.vbest);
}

__device__ __forceinline__ void search_take(Search& s, uint32_t V, uint64_t maxbin) {
  s.best = maxbin * (uint64_t)(s.P - 1 + V);
  s.vbest = V;
  s.have = true;
  // every V < ceil(sumT (PP-1) / (best - sumT)) has sumT (PP-1+V) > best V: jump past them
  // (fp32 estimate minus a margin of 2; the exact per-V tests in search_next stay in force)
  if (s.phase == 1 && s.P > 1) {
    if (s.best <= s.sumT) {
      s.cursor = s.vhi + 1;
    } else {
      const float est = (float)s.sumT * (float)(s.P - 1) / (float)(s.best - s.sumT);
      const float lo = est - 2.0f;
      if (lo > (float)s.cursor) s.cursor = lo >= (float)s.vhi ? s.vhi + 1 : (uint32_t)lo;
    }
  }
}

}  // namespace hyd
