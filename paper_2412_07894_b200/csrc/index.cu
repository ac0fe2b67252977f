// index.cu -- the stage-1 -> stage-2 interface built from an arbitrary assignment `pipe`.
//
// Eq. 3 states stage 1's result as the matrix m_ij (sequence i on pipeline j, with
// j in J_i = {j : MaxLen(P_j) >= l_i}); stage 2 (Eq. 1) packs each
// pipeline's sequences.  hyd_dispatch emits that matrix as membership bitmaps plus per-pipeline
// sums while it decides; k_pipe_index derives the same (stats, members) from any `pipe` row --
// e.g. a host Alg. 1 or the caller's own dispatch -- so hyd_pack can pack it, and it
// checks the row is an assignment: every entry names a pipeline of the candidate that can hold
// the sequence (J_i), or the whole row is 0xFF for a pair that is infeasible (l_0 > MaxLen_0,
// S:371).  Anything else sets HYD_F_BAD_PIPE and the pair is treated as infeasible.
//
// One warp per (c, t): lane j < np holds pipeline j's scheme; 32 sorted positions per step
// (coalesced pipe / length loads, one cost word per lane); per pipeline a ballot gives the
// membership word and warp reductions give the token and cost sums (costs split in 16-bit
// halves so the 32-lane sums fit u32).  lb = Eq. 2's max_j (sum T + T(first)(PP_j - 1)).
#include "hyd_internal.cuh"

namespace hyd {

constexpr int kIndexWarps = 8;

__global__ void __launch_bounds__(kIndexWarps * 32)
    k_pipe_index(const uint32_t* __restrict__ sorted_len, const uint32_t* __restrict__ cost, int n_iter,
                 int batch, const uint32_t* __restrict__ off, size_t n_total, int k_pad,
                 const hyd_scheme* __restrict__ schemes, int n_schemes, const uint8_t* __restrict__ cand,
                 const uint8_t* __restrict__ cand_np, int n_cand, int max_np, const uint8_t* __restrict__ pipe,
                 uint64_t* __restrict__ lb, hyd_pipe_stats* __restrict__ stats, uint32_t* __restrict__ members,
                 uint32_t* __restrict__ status) {
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * kIndexWarps + (threadIdx.x >> 5);
  const int t = blockIdx.y;
  if (c >= n_cand || t >= n_iter) return;
  const int B = geo_bt(off, batch, t);
  const size_t tbase = geo_base(off, batch, t);
  const int np = cand_np[c];
  // lane j: pipeline j's scheme (canonical order checked as hyd_dispatch does)
  uint32_t k = 0, ml = 0, pp = 1;
  bool ok = np >= 1 && np <= max_np && np <= HYD_MAX_PIPES;
  if (lane < np) {
    k = cand[(size_t)c * HYD_MAX_PIPES + lane];
    if (k < (uint32_t)n_schemes) {
      ml = schemes[k].max_len;
      pp = schemes[k].pp;
      ok = ok && ml >= 1u && pp >= 1u && pp <= HYD_MAX_PP;
    } else {
      ok = false;
    }
  }
  const uint32_t prev_ml = __shfl_up_sync(HYD_FULL, ml, 1), prev_k = __shfl_up_sync(HYD_FULL, k, 1);
  if (lane >= 1 && lane < np) ok = ok && (ml < prev_ml || (ml == prev_ml && k >= prev_k));
  ok = __all_sync(HYD_FULL, ok);
  if (!ok) {
    if (lane == 0) flag(status, HYD_F_NOT_CANONICAL);
  }
  const size_t srow = (size_t)t * n_cand + c;
  const uint8_t* prow = pipe + (size_t)c * n_total + tbase;
  const uint32_t* sl = sorted_len + tbase;
  const uint32_t* cs = cost + tbase * k_pad;
  const uint32_t ml0 = __shfl_sync(HYD_FULL, ml, 0);
  const bool infeasible = !ok || B == 0 || sl[0] > ml0;
  const int nwords = (batch + 31) >> 5;  // member row stride (largest batch)
  uint32_t* mbits = members + srow * (size_t)max_np * nwords;
  bool bad = false, any_ff = false, any_set = false;
  uint32_t u = 0, first = 0xFFFFFFFFu;
  uint64_t s_sum = 0, t_sum = 0;
  for (int w = 0; w * 32 < B; ++w) {
    const int i = w * 32 + lane;
    const bool in = i < B;
    const uint32_t p = in ? (uint32_t)prow[i] : 0xFEu;
    const uint32_t l = in ? sl[i] : 0u;
    const uint32_t pl = p & 31u;
    const uint32_t mlp = __shfl_sync(HYD_FULL, ml, pl);
    const uint32_t kp_ = __shfl_sync(HYD_FULL, k, pl);
    if (in) {
      if (p == 0xFFu) any_ff = true;
      else if (p >= (uint32_t)np || mlp < l) bad = true;  // not a pipeline of c, or not in J_i
      else any_set = true;
    }
    const bool mine = in && p < (uint32_t)np && mlp >= l;
    const uint32_t tau = mine ? __ldg(cs + (size_t)i * k_pad + kp_) : 0u;
    for (int j = 0; j < np; ++j) {
      const bool hit = mine && p == (uint32_t)j;
      const uint32_t m = __ballot_sync(HYD_FULL, hit);
      const uint32_t sl_ = __reduce_add_sync(HYD_FULL, hit ? l : 0u);
      const uint32_t tlo = __reduce_add_sync(HYD_FULL, hit ? (tau & 0xFFFFu) : 0u);
      const uint32_t thi = __reduce_add_sync(HYD_FULL, hit ? (tau >> 16) : 0u);
      if (lane == j) {
        if (m && first == 0xFFFFFFFFu) first = (uint32_t)(w * 32 + __ffs(m) - 1);
        u += __popc(m);
        s_sum += sl_;
        t_sum += (uint64_t)tlo + ((uint64_t)thi << 16);
        HYD_CHECK(j < max_np && w < nwords);
        if (!infeasible) mbits[(size_t)w * max_np + j] = m;
      }
    }
  }
  bad = __any_sync(HYD_FULL, bad);
  any_ff = __any_sync(HYD_FULL, any_ff);
  any_set = __any_sync(HYD_FULL, any_set);
  // a feasible pair needs every sequence assigned; an infeasible one an all-0xFF row
  const bool invalid = ok && (infeasible ? (bad || any_set) : (bad || any_ff));
  if (invalid && lane == 0) flag(status, HYD_F_BAD_PIPE);
  if (infeasible || invalid) {
    if (lane == 0) {
      stats[srow * max_np].u = 0xFFFFFFFFu;
      if (lb) lb[(size_t)c * n_iter + t] = ~0ull;
    }
    return;
  }
  const uint32_t tm = (lane < np && first != 0xFFFFFFFFu) ? __ldg(cs + (size_t)first * k_pad + k) : 0u;
  uint64_t base = lane < np ? t_sum + (uint64_t)tm * (pp - 1u) : 0ull;  // C_j + E_j (Eq. 2)
  if (lane < np) {
    hyd_pipe_stats e;
    e.u = u;
    e.tau_max = tm;
    e.s = s_sum;
    e.sum_t = t_sum;
    stats[srow * max_np + lane] = e;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) base = max(base, __shfl_xor_sync(HYD_FULL, base, o));
  if (lb && lane == 0) lb[(size_t)c * n_iter + t] = base;
}

int launch_pipe_index(const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch,
                      const uint32_t* off, size_t n_total, int k_pad, const hyd_scheme* schemes,
                      int n_schemes, const uint8_t* cand, const uint8_t* cand_np, int n_cand, int max_np,
                      const uint8_t* pipe, uint64_t* lb, hyd_pipe_stats* stats, uint32_t* members,
                      uint32_t* status, cudaStream_t s) {
  if (n_iter == 0 || n_cand == 0) return HYD_OK;
  const dim3 grid((n_cand + kIndexWarps - 1) / kIndexWarps, n_iter);
  k_pipe_index<<<grid, kIndexWarps * 32, 0, s>>>(sorted_len, cost, n_iter, batch, off, n_total, k_pad, schemes,
                                                 n_schemes, cand, cand_np, n_cand, max_np, pipe, lb, stats,
                                                 members, status);
  note_launch();
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HYD_OK : record_cuda_error(e);
}

}  // namespace hyd
