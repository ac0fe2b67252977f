// bb.cu -- NEXT-4: exact optimum of Eq. 3 for small batches, branch-and-bound on
// the GPU, to measure the heuristics' optimality gap at scale.
//
// One thread per (candidate, iteration) instance: iterative depth-first search over the
// sequences in sorted (longest-first) order, each sequence on a feasible pipeline
// (MaxLen_j >= l).  Because the first sequence a pipeline receives is its longest, the
// pipeline's Eq. 2 bound is C_j + E_j with E_j = tau_first (PP_j - 1) fixed at its first
// member, so a node costs D additions.  Pruning (never loses an optimum):
//   * the partial maximum of C_j + E_j already reaches the incumbent (C_j + E_j never decrease);
//   * the average bound: (sum_j (C_j + E_j) + sum of the remaining sequences' cheapest
//     feasible cost) / D reaches the incumbent (the final maximum is at least the final mean);
//   * symmetry: among empty pipelines of the same scheme only the first is tried.
// The incumbent starts at the greedy HYD-H1 dispatch (the LPT rule of dispatch.cu), so an
// instance whose greedy is optimal proves it without improving.  A node budget bounds the
// search; exhausted instances report the incumbent and proved = 0.
#include "hyd_internal.cuh"

namespace hyd {

constexpr int kBBThreads = 128;
constexpr int kBBMaxB = HYD_BB_MAX_BATCH;
constexpr int kBBMaxD = 8;

__global__ void __launch_bounds__(kBBThreads)
    k_eq3_exact(const uint32_t* __restrict__ sorted_len, const uint32_t* __restrict__ cost,
                int n_iter, int batch, int k_pad, const hyd_scheme* __restrict__ schemes,
                int n_schemes, const uint8_t* __restrict__ cand, const uint8_t* __restrict__ cand_np,
                int n_cand, const int32_t* __restrict__ pair_c, const int32_t* __restrict__ pair_t,
                int n_pairs, unsigned long long node_limit, uint64_t* __restrict__ value,
                uint8_t* __restrict__ pipe, uint64_t* __restrict__ nodes_out,
                uint8_t* __restrict__ proved, uint32_t* __restrict__ status) {
  const int p = blockIdx.x * kBBThreads + threadIdx.x;
  if (p >= n_pairs) return;
  const int c = pair_c[p], t = pair_t[p];
  const int B = batch;
  uint8_t* prow = pipe + (size_t)p * B;
  const uint32_t* sl = sorted_len + (size_t)t * B;
  const uint32_t* cs = cost + (size_t)t * B * k_pad;
  const int np = cand_np[c];
  uint32_t ml[kBBMaxD], pm1[kBBMaxD], kk[kBBMaxD];
  bool ok = np >= 1 && np <= kBBMaxD && c < n_cand && t < n_iter;
  for (int j = 0; j < kBBMaxD; ++j) {
    ml[j] = 0u;
    pm1[j] = 0u;
    kk[j] = 0u;
    if (j < np) {
      const uint32_t k = cand[(size_t)c * HYD_MAX_PIPES + j];
      if (k < (uint32_t)n_schemes) {
        ml[j] = schemes[k].max_len;
        pm1[j] = schemes[k].pp - 1u;
        kk[j] = k;
      } else {
        ok = false;
      }
    }
  }
  if (!ok || sl[0] > ml[0]) {  // not canonical / infeasible candidate for this iteration
    value[p] = ~0ull;
    nodes_out[p] = 0ull;
    proved[p] = 0;
    for (int i = 0; i < B; ++i) prow[i] = 0xFF;
    if (!ok) flag(status, HYD_F_NOT_CANONICAL);
    return;
  }
  // suffix sums of the cheapest feasible cost of the remaining sequences
  uint64_t rem[kBBMaxB + 1];
  rem[B] = 0ull;
  for (int i = B - 1; i >= 0; --i) {
    uint32_t m = 0xFFFFFFFFu;
    for (int j = 0; j < np; ++j)
      if (sl[i] <= ml[j]) m = min(m, cs[(size_t)i * k_pad + kk[j]]);
    rem[i] = rem[i + 1] + m;
  }
  // incumbent: the HYD-H1 greedy dispatch (argmin of the own new load, smallest j)
  uint64_t C[kBBMaxD], E[kBBMaxD];
  uint32_t cnt[kBBMaxD];
  for (int j = 0; j < kBBMaxD; ++j) {
    C[j] = 0ull;
    E[j] = 0ull;
    cnt[j] = 0u;
  }
  uint8_t best_pipe[kBBMaxB], cur[kBBMaxB], next[kBBMaxB];
  for (int i = 0; i < B; ++i) {
    int bj = -1;
    uint64_t bv = 0ull;
    for (int j = 0; j < np; ++j) {
      if (sl[i] > ml[j]) continue;
      const uint64_t tau = cs[(size_t)i * k_pad + kk[j]];
      const uint64_t nw = C[j] + tau + (cnt[j] ? E[j] : tau * pm1[j]);
      if (bj < 0 || nw < bv) {
        bj = j;
        bv = nw;
      }
    }
    const uint64_t tau = cs[(size_t)i * k_pad + kk[bj]];
    if (cnt[bj] == 0u) E[bj] = tau * pm1[bj];
    C[bj] += tau;
    ++cnt[bj];
    best_pipe[i] = (uint8_t)bj;
  }
  uint64_t best = 0ull;
  for (int j = 0; j < np; ++j) best = max(best, C[j] + E[j]);
  for (int j = 0; j < kBBMaxD; ++j) {
    C[j] = 0ull;
    E[j] = 0ull;
    cnt[j] = 0u;
  }
  // depth-first search; next[i] = next pipeline to try at depth i
  unsigned long long nodes = 0ull;
  bool exhausted = false;
  int i = 0;
  next[0] = 0;
  while (i >= 0) {
    if (i == B) {  // leaf: strictly better than the incumbent by construction of the pruning
      uint64_t m = 0ull;
      for (int j = 0; j < np; ++j) m = max(m, C[j] + E[j]);
      if (m < best) {
        best = m;
        for (int q = 0; q < B; ++q) best_pipe[q] = cur[q];
      }
      --i;
      if (i >= 0) {  // undo cur[i]
        const int j = cur[i];
        C[j] -= cs[(size_t)i * k_pad + kk[j]];
        if (--cnt[j] == 0u) E[j] = 0ull;
        next[i] = (uint8_t)(j + 1);
      }
      continue;
    }
    if (++nodes > node_limit) {
      exhausted = true;
      break;
    }
    uint64_t pmax = 0ull, psum = 0ull;
    for (int j = 0; j < np; ++j) {
      pmax = max(pmax, C[j] + E[j]);
      psum += C[j] + E[j];
    }
    const uint32_t l = sl[i];
    int taken = -1;
    for (int j = next[i]; j < np; ++j) {
      if (l > ml[j]) continue;
      if (cnt[j] == 0u) {  // symmetry: the first empty pipeline of each scheme only
        bool dup = false;
        for (int q = 0; q < j; ++q) dup |= cnt[q] == 0u && kk[q] == kk[j];
        if (dup) continue;
      }
      const uint64_t tau = cs[(size_t)i * k_pad + kk[j]];
      const uint64_t add = cnt[j] ? tau : tau + tau * pm1[j];
      const uint64_t nv = C[j] + E[j] + add;
      if (max(pmax, nv) >= best) continue;
      // average bound over the final loads (cheapest costs for the rest)
      const uint64_t fsum = psum + add + rem[i + 1];
      if ((fsum + (uint64_t)np - 1ull) / (uint64_t)np >= best) continue;
      taken = j;
      break;
    }
    if (taken < 0) {  // backtrack
      --i;
      if (i >= 0) {
        const int j = cur[i];
        C[j] -= cs[(size_t)i * k_pad + kk[j]];
        if (--cnt[j] == 0u) E[j] = 0ull;
        next[i] = (uint8_t)(j + 1);
      }
      continue;
    }
    const uint64_t tau = cs[(size_t)i * k_pad + kk[taken]];
    if (cnt[taken] == 0u) E[taken] = tau * pm1[taken];
    C[taken] += tau;
    ++cnt[taken];
    cur[i] = (uint8_t)taken;
    ++i;
    if (i < B) next[i] = 0;
  }
  value[p] = best;
  nodes_out[p] = nodes;
  proved[p] = exhausted ? 0 : 1;
  for (int q = 0; q < B; ++q) prow[q] = best_pipe[q];
}

int launch_eq3_exact(const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch,
                     int k_pad, const hyd_scheme* schemes, int n_schemes, const uint8_t* cand,
                     const uint8_t* cand_np, int n_cand, const int32_t* pair_c,
                     const int32_t* pair_t, int n_pairs, unsigned long long node_limit,
                     uint64_t* value, uint8_t* pipe, uint64_t* nodes, uint8_t* proved,
                     uint32_t* status, cudaStream_t s) {
  if (n_pairs == 0) return HYD_OK;
  k_eq3_exact<<<(n_pairs + kBBThreads - 1) / kBBThreads, kBBThreads, 0, s>>>(
      sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np, n_cand, pair_c,
      pair_t, n_pairs, node_limit, value, pipe, nodes, proved, status);
  note_launch();
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HYD_OK : record_cuda_error(e);
}

}  // namespace hyd
