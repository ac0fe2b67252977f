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

namespace hyd {

// Exact Eq. 1 for one pipeline per thread: the items (the pipeline's sequences in
// sorted order, from the membership words) split into V micro-batches within MaxLen, min over V
// of (max micro-batch time)(PP - 1 + V) over App. D's range (upward extension while none is
// feasible), ties to the smaller V.  Per V: iterative depth-first search item by item over the
// bins, started from the LPT(V) packing as incumbent; pruned by the partial maximum, by LB(V) =
// max(ceil(sum T / V), tau_max)(PP-1+V) against the best objective so far, and by symmetry (an
// item goes to the first empty bin only); leaves must fill all V bins.
constexpr int kE1Max = 32;  // items and micro-batches per instance

__global__ void __launch_bounds__(128)
    k_eq1_exact(const uint32_t* __restrict__ sorted_len, const uint32_t* __restrict__ cost,
                int n_iter, int batch, int k_pad, const hyd_scheme* __restrict__ schemes,
                int n_schemes, const uint8_t* __restrict__ cand, int n_cand, int max_np,
                const uint32_t* __restrict__ members, const int32_t* __restrict__ pair_c,
                const int32_t* __restrict__ pair_t, const int32_t* __restrict__ pair_j, int n_pairs,
                unsigned long long node_limit, uint32_t* __restrict__ v_out,
                uint64_t* __restrict__ obj_out, uint64_t* __restrict__ nodes_out,
                uint8_t* __restrict__ proved, uint32_t* __restrict__ status) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_pairs) return;
  const int c = pair_c[p], t = pair_t[p], j = pair_j[p];
  const int B = batch;
  const uint32_t k = cand[(size_t)c * HYD_MAX_PIPES + j];
  const uint32_t* sl = sorted_len + (size_t)t * B;
  const uint32_t* cs = cost + (size_t)t * B * k_pad;
  const int nwords = (B + 31) >> 5;
  const uint32_t* mw = members + ((size_t)t * n_cand + c) * nwords * max_np + j;  // word-major
  uint32_t ell[kE1Max], tau[kE1Max];
  int U = 0;
  uint64_t S = 0, sumT = 0;
  uint32_t tmax = 0;
  bool too_big = false;
  for (int w = 0; w < nwords; ++w) {
    uint32_t bits = mw[(size_t)w * max_np];
    while (bits) {
      const int i = w * 32 + __ffs(bits) - 1;
      bits &= bits - 1u;
      if (U == kE1Max) {
        too_big = true;
        break;
      }
      ell[U] = sl[i];
      tau[U] = cs[(size_t)i * k_pad + k];
      S += ell[U];
      sumT += tau[U];
      tmax = max(tmax, tau[U]);
      ++U;
    }
  }
  v_out[p] = 0;
  obj_out[p] = 0;
  nodes_out[p] = 0;
  proved[p] = 0;
  if (too_big || k >= (uint32_t)n_schemes) {
    flag(status, too_big ? 0u : HYD_F_NOT_CANONICAL);
    return;
  }
  if (U == 0) {
    proved[p] = 1;
    return;
  }
  const uint32_t M = schemes[k].max_len, P = schemes[k].pp, UL = schemes[k].util_len;
  uint32_t vlo = (uint32_t)((S + M - 1) / M);
  if (vlo < 1) vlo = 1;
  uint32_t vhi = (uint32_t)U;
  if (UL) vhi = (uint32_t)min((uint64_t)U, S / UL);
  if (vhi < vlo) vhi = vlo;
  uint64_t best = ~0ull;
  uint32_t vbest = 0;
  unsigned long long nodes = 0;
  bool exhausted = false;
  uint64_t bt[kE1Max];
  uint32_t bk[kE1Max];
  uint8_t nxt[kE1Max];
  for (uint32_t V = vlo; V <= (uint32_t)U && !exhausted; ++V) {
    if (V > vhi && vbest != 0) break;  // extension only while nothing in range is feasible
    const uint64_t m = (uint64_t)(P - 1u + V);
    const uint64_t lbv = max((sumT + V - 1) / V, (uint64_t)tmax);
    if (vbest != 0 && lbv * m >= best) continue;  // cannot beat (or tie at smaller V) the best
    // incumbent: LPT(V) with capacity (least-time fitting bin, smallest index)
    for (uint32_t b = 0; b < V; ++b) {
      bt[b] = 0;
      bk[b] = 0;
    }
    uint64_t inc = 0;
    bool lpt_ok = true;
    for (int i = 0; i < U && lpt_ok; ++i) {
      int bb = -1;
      for (uint32_t b = 0; b < V; ++b)
        if (bk[b] + ell[i] <= M && (bb < 0 || bt[b] < bt[bb])) bb = (int)b;
      if (bb < 0) {
        lpt_ok = false;
        break;
      }
      bt[bb] += tau[i];
      bk[bb] += ell[i];
      inc = max(inc, bt[bb]);
    }
    uint64_t bestV = lpt_ok ? inc : ~0ull;  // best max micro-batch time for this V
    // depth-first search for a strictly better split
    for (uint32_t b = 0; b < V; ++b) {
      bt[b] = 0;
      bk[b] = 0;
    }
    int i = 0;
    nxt[0] = 0;
    uint64_t pm[kE1Max + 1];
    pm[0] = 0;
    uint32_t empty = V;  // bins still empty
    uint8_t cur[kE1Max];
    while (i >= 0) {
      if (i == U) {
        if (empty == 0 && pm[U] < bestV) bestV = pm[U];
        --i;
        if (i >= 0) {
          const int b = cur[i];
          bt[b] -= tau[i];
          bk[b] -= ell[i];
          if (bk[b] == 0) ++empty;
          nxt[i] = (uint8_t)(b + 1);
        }
        continue;
      }
      if (++nodes > node_limit) {
        exhausted = true;
        break;
      }
      int taken = -1;
      for (int b = nxt[i]; b < (int)V; ++b) {
        if (bk[b] + ell[i] > M) continue;
        if (bk[b] == 0) {  // the first empty bin only
          bool earlier = false;
          for (int q = 0; q < b; ++q) earlier |= bk[q] == 0;
          if (earlier) continue;
        }
        if ((uint32_t)(U - i - 1) < empty - (bk[b] == 0 ? 1u : 0u)) continue;  // bins left unfillable
        const uint64_t nm = max(pm[i], bt[b] + tau[i]);
        if (nm >= bestV) continue;
        taken = b;
        break;
      }
      if (taken < 0) {
        --i;
        if (i >= 0) {
          const int b = cur[i];
          bt[b] -= tau[i];
          bk[b] -= ell[i];
          if (bk[b] == 0) ++empty;
          nxt[i] = (uint8_t)(b + 1);
        }
        continue;
      }
      if (bk[taken] == 0) --empty;
      bt[taken] += tau[i];
      bk[taken] += ell[i];
      pm[i + 1] = max(pm[i], bt[taken]);
      cur[i] = (uint8_t)taken;
      ++i;
      if (i < U) nxt[i] = 0;
    }
    if (bestV != ~0ull) {
      const uint64_t obj = bestV * m;
      if (obj < best) {
        best = obj;
        vbest = V;
      }
    }
  }
  v_out[p] = vbest;
  obj_out[p] = vbest ? best : ~0ull;
  nodes_out[p] = nodes;
  proved[p] = !exhausted && vbest != 0;
}

int launch_eq1_exact(const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch,
                     int k_pad, const hyd_scheme* schemes, int n_schemes, const uint8_t* cand,
                     int n_cand, int max_np, const uint32_t* members, const int32_t* pair_c,
                     const int32_t* pair_t, const int32_t* pair_j, int n_pairs,
                     unsigned long long node_limit, uint32_t* v, uint64_t* obj, uint64_t* nodes,
                     uint8_t* proved, uint32_t* status, cudaStream_t s) {
  if (n_pairs == 0) return HYD_OK;
  k_eq1_exact<<<(n_pairs + 127) / 128, 128, 0, s>>>(sorted_len, cost, n_iter, batch, k_pad, schemes,
                                                    n_schemes, cand, n_cand, max_np, members, pair_c,
                                                    pair_t, pair_j, n_pairs, node_limit, v, obj,
                                                    nodes, proved, status);
  note_launch();
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HYD_OK : record_cuda_error(e);
}

}  // namespace hyd
