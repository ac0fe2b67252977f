// sort_cost.cu -- a1 + a2: per-iteration stable radix sort of the lengths (length
// descending, original index ascending) fused with the Q32 fixed-point cost table
// T(l, P_k) = floor((a_k l^2 + b_k l + c_k) / 2^32)  (App. C.2).
//
// By batch size: B <= 32 a warp per iteration ranks by shuffles; B <= 256 a warp per iteration
// runs a register bitonic sort on distinct keys; larger batches use one CTA per iteration t.
// There the B lengths stay in shared memory; an LSD radix sort
// over 4-bit digits (as many passes as the iteration's largest length needs) permutes
// a u16 index array, blocked arrangement + digit-major block scan => stable.  The
// cost rows are then written as 16-byte vector stores, consecutive threads writing
// consecutive 16 B (k_pad % 4 == 0).  HBM traffic per t: 4B read + 8B + 4*B*k_pad write.
#include "hyd_internal.cuh"

namespace hyd {


template <int NT>
__global__ void __launch_bounds__(NT) k_sort_cost(const uint32_t* __restrict__ len, int batch,
                                                  const uint32_t* __restrict__ off,
                                                  const hyd_scheme* __restrict__ schemes,
                                                  int n_schemes, int k_pad,
                                                  uint32_t* __restrict__ sorted_len,
                                                  uint32_t* __restrict__ perm,
                                                  uint32_t* __restrict__ cost,
                                                  uint32_t* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int t = blockIdx.x;
  const int tid = threadIdx.x;
  const int B = geo_bt(off, batch, t);  // this iteration's sequences (<= batch)
  const size_t base = geo_base(off, batch, t);
  if (off && tid == 0) {  // ragged batches: 1 <= B_t <= batch
    const int d = (int)(__ldg(off + t + 1) - __ldg(off + t));
    if (d < 1 || d > batch) atomicOr(status, HYD_F_BAD_LENGTH);
  }
  // layout (sized for `batch`): lens[B] u32 | hist[16*NT] u32 | idxA[B] u16 | idxB[B] u16 | coef
  uint32_t* lens = reinterpret_cast<uint32_t*>(smem_raw);
  uint32_t* hist = lens + batch;
  uint16_t* idxA = reinterpret_cast<uint16_t*>(hist + 16 * NT);
  uint16_t* idxB = idxA + batch;
  uint64_t* coef = reinterpret_cast<uint64_t*>(smem_raw + (((size_t)batch * 4 + 16 * NT * 4 + (size_t)batch * 4 + 15) & ~(size_t)15));
  __shared__ uint32_t s_or[NT / 32];
  __shared__ uint32_t s_wsum[NT / 32];

  const uint32_t* lrow = len + base;
  uint32_t orv = 0;
  for (int i = tid; i < B; i += NT) {
    const uint32_t l = __ldg(lrow + i);
    lens[i] = l;
    idxA[i] = (uint16_t)i;
    orv |= l;
  }
  for (int k = tid; k < n_schemes; k += NT) {
    coef[3 * k + 0] = schemes[k].a_q32;
    coef[3 * k + 1] = schemes[k].b_q32;
    coef[3 * k + 2] = schemes[k].c_q32;
  }
  orv = __reduce_or_sync(HYD_FULL, orv);
  if ((tid & 31) == 0) s_or[tid >> 5] = orv;
  __syncthreads();
  if (tid < 32) {
    uint32_t v = tid < NT / 32 ? s_or[tid] : 0u;
    v = __reduce_or_sync(HYD_FULL, v);
    if (tid == 0) s_or[0] = v;
  }
  __syncthreads();
  const uint32_t all_or = s_or[0];
  const int nbits = all_or ? 32 - __clz(all_or) : 1;
  const int passes = (nbits + 3) >> 2;

  const int ipt = (B + NT - 1) / NT;  // blocked arrangement: thread owns [lo, hi)
  const int lo = min(B, tid * ipt), hi = min(B, lo + ipt);
  uint16_t* src = idxA;
  uint16_t* dst = idxB;
  for (int p = 0; p < passes; ++p) {
    const int shift = 4 * p;
#pragma unroll
    for (int d = 0; d < 16; ++d) hist[d * NT + tid] = 0u;
    for (int q = lo; q < hi; ++q) {
      const uint32_t d = 15u - ((lens[src[q]] >> shift) & 15u);  // descending digits
      hist[d * NT + tid] += 1u;
    }
    __syncthreads();
    // exclusive scan of hist (digit-major) : thread tid scans entries [16*tid, 16*tid+16)
    uint32_t run = 0;
#pragma unroll
    for (int e = 0; e < 16; ++e) run += hist[16 * tid + e];
    uint32_t incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(HYD_FULL, incl, o);
      if ((tid & 31) >= o) incl += y;
    }
    if ((tid & 31) == 31) s_wsum[tid >> 5] = incl;
    __syncthreads();
    if (tid < 32) {
      uint32_t v = tid < NT / 32 ? s_wsum[tid] : 0u;
      uint32_t inc2 = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(HYD_FULL, inc2, o);
        if (tid >= o) inc2 += y;
      }
      if (tid < NT / 32) s_wsum[tid] = inc2 - v;  // exclusive warp offsets
    }
    __syncthreads();
    uint32_t base = s_wsum[tid >> 5] + incl - run;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const uint32_t h = hist[16 * tid + e];
      hist[16 * tid + e] = base;
      base += h;
    }
    __syncthreads();
    for (int q = lo; q < hi; ++q) {
      const uint16_t ix = src[q];
      const uint32_t d = 15u - ((lens[ix] >> shift) & 15u);
      const uint32_t pos = hist[d * NT + tid];
      hist[d * NT + tid] = pos + 1u;
      dst[pos] = ix;
    }
    __syncthreads();
    uint16_t* tmp = src;
    src = dst;
    dst = tmp;
  }

  uint32_t* srow = sorted_len + base;
  uint32_t* prow = perm + base;
  for (int i = tid; i < B; i += NT) {
    const uint32_t ix = src[i];
    srow[i] = lens[ix];
    prow[i] = ix;
  }
  // cost rows: thread handles (i, quad) pairs, consecutive threads -> consecutive 16 B
  uint32_t st = 0;
  const int quads = k_pad >> 2;
  uint4* crow = reinterpret_cast<uint4*>(cost + base * k_pad);
  for (int e = tid; e < B * quads; e += NT) {
    const int i = e / quads, q = e - i * quads;
    const uint32_t l = lens[src[i]];
    uint32_t out[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int k = 4 * q + r;
      out[r] = k < n_schemes ? eval_cost(coef[3 * k], coef[3 * k + 1], coef[3 * k + 2], l, st) : 0u;
    }
    crow[e] = make_uint4(out[0], out[1], out[2], out[3]);
  }
  st = __reduce_or_sync(HYD_FULL, st);
  if (st && (tid & 31) == 0) atomicOr(status, st);
}

// Batches of at most 32 sequences (configuration 1): a WARP per iteration.  Lane i holds l_i; its
// sorted position is the number of (l_j > l_i) or (l_j == l_i, j < i) over the row (32 shuffles),
// which is the same stable order; the lane then writes its length, index and cost row there.
__global__ void __launch_bounds__(256) k_sort_cost_warp(const uint32_t* __restrict__ len, int batch,
                                                        const uint32_t* __restrict__ off,
                                                        const hyd_scheme* __restrict__ schemes,
                                                        int n_schemes, int k_pad, int n_iter,
                                                        uint32_t* __restrict__ sorted_len,
                                                        uint32_t* __restrict__ perm,
                                                        uint32_t* __restrict__ cost,
                                                        uint32_t* __restrict__ status) {
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= n_iter) return;
  const int B = geo_bt(off, batch, t);
  const size_t base = geo_base(off, batch, t);
  if (off && lane == 0) {  // ragged batches: 1 <= B_t <= batch
    const int d = (int)(__ldg(off + t + 1) - __ldg(off + t));
    if (d < 1 || d > batch) atomicOr(status, HYD_F_BAD_LENGTH);
  }
  const bool mine = lane < B;
  const uint32_t l = mine ? __ldg(len + base + lane) : 0u;
  uint32_t rank = 0;
  for (int j = 0; j < 32; ++j) {
    const uint32_t lj = __shfl_sync(HYD_FULL, l, j);
    rank += (j < B && (lj > l || (lj == l && j < lane))) ? 1u : 0u;
  }
  uint32_t st = 0;
  if (mine) {
    sorted_len[base + rank] = l;
    perm[base + rank] = (uint32_t)lane;
    uint4* crow = reinterpret_cast<uint4*>(cost + (base + rank) * k_pad);
    for (int q = 0; q < (k_pad >> 2); ++q) {
      uint32_t out[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int k = 4 * q + r;
        out[r] = k < n_schemes ? eval_cost(schemes[k].a_q32, schemes[k].b_q32, schemes[k].c_q32, l, st) : 0u;
      }
      crow[q] = make_uint4(out[0], out[1], out[2], out[3]);
    }
  }
  st = __reduce_or_sync(HYD_FULL, st);
  if (st && lane == 0) atomicOr(status, st);
}

// Batches of 33 .. 256 sequences (configurations 2 and 6): a WARP per
// iteration, a bitonic sort of u64 keys (~l_i) << 32 | i in registers (E per lane, element
// i = lane * E + e; padding keys ~0 sort last).  The keys are distinct, so ascending key order is
// exactly (length descending, index ascending) -- the radix sort's stable order -- with no
// shared memory and no barriers (the CTA radix sort's passes are latency-bound at these sizes).
template <int E>
__device__ __forceinline__ void bitonic_warp(uint64_t (&k)[E], int lane) {
  constexpr int N = 32 * E;
#pragma unroll
  for (int size = 2; size <= N; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= E) {  // partner in lane ^ (stride / E), same e
        const int lm = stride / E;
        const bool lower = (lane & lm) == 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int i = lane * E + e;
          const bool asc = (i & size) == 0;
          const uint64_t o = __shfl_xor_sync(HYD_FULL, k[e], lm);
          k[e] = (lower == asc) ? min(k[e], o) : max(k[e], o);
        }
      } else {  // partner e ^ stride in the same lane
#pragma unroll
        for (int e = 0; e < E; ++e) {
          if ((e & stride) == 0) {
            const int i = lane * E + e;
            const bool asc = (i & size) == 0;
            const uint64_t x = k[e], y = k[e ^ stride];
            const uint64_t lo = min(x, y), hi = max(x, y);
            k[e] = asc ? lo : hi;
            k[e ^ stride] = asc ? hi : lo;
          }
        }
      }
    }
  }
}

template <int E>
__global__ void __launch_bounds__(128) k_sort_cost_bitonic(const uint32_t* __restrict__ len, int batch,
                                                           const uint32_t* __restrict__ off,
                                                           const hyd_scheme* __restrict__ schemes,
                                                           int n_schemes, int k_pad, int n_iter,
                                                           uint32_t* __restrict__ sorted_len,
                                                           uint32_t* __restrict__ perm,
                                                           uint32_t* __restrict__ cost,
                                                           uint32_t* __restrict__ status) {
  const int t = blockIdx.x * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= n_iter) return;
  const int B = geo_bt(off, batch, t);
  const size_t base = geo_base(off, batch, t);
  if (off && lane == 0) {  // ragged batches: 1 <= B_t <= batch
    const int d = (int)(__ldg(off + t + 1) - __ldg(off + t));
    if (d < 1 || d > batch) atomicOr(status, HYD_F_BAD_LENGTH);
  }
  uint64_t k[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = lane * E + e;
    k[e] = i < B ? ((uint64_t)(~__ldg(len + base + i)) << 32) | (uint32_t)i : ~0ull;
  }
  bitonic_warp<E>(k, lane);
  uint32_t st = 0;
  const int quads = k_pad >> 2;
  for (int q = 0; q < quads; ++q) {
    uint64_t ca[4], cb[4], cc[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int kk = 4 * q + r;
      ca[r] = kk < n_schemes ? schemes[kk].a_q32 : 0ull;
      cb[r] = kk < n_schemes ? schemes[kk].b_q32 : 0ull;
      cc[r] = kk < n_schemes ? schemes[kk].c_q32 : 0ull;
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = lane * E + e;
      if (i < B) {
        const uint32_t l = ~(uint32_t)(k[e] >> 32);
        uint32_t out[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) out[r] = 4 * q + r < n_schemes ? eval_cost(ca[r], cb[r], cc[r], l, st) : 0u;
        reinterpret_cast<uint4*>(cost + (base + i) * k_pad)[q] = make_uint4(out[0], out[1], out[2], out[3]);
      }
    }
  }
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = lane * E + e;
    if (i < B) {
      sorted_len[base + i] = ~(uint32_t)(k[e] >> 32);
      perm[base + i] = (uint32_t)(k[e] & 0xFFFFFFFFu);
    }
  }
  st = __reduce_or_sync(HYD_FULL, st);
  if (st && lane == 0) atomicOr(status, st);
}

size_t sort_cost_smem(int batch, int nt, int n_schemes) {
  return (((size_t)batch * 4 + 16 * (size_t)nt * 4 + (size_t)batch * 4 + 15) & ~(size_t)15) +
         (size_t)n_schemes * 24;
}

int launch_sort_cost(const uint32_t* len, int n_iter, int batch, const uint32_t* off,
                     const hyd_scheme* schemes, int n_schemes, int k_pad, uint32_t* sorted_len,
                     uint32_t* perm, uint32_t* cost, uint32_t* status, cudaStream_t s) {
  if (n_iter == 0) return HYD_OK;
  cudaError_t e;
  if (batch <= 32) {
    k_sort_cost_warp<<<(n_iter + 7) / 8, 256, 0, s>>>(len, batch, off, schemes, n_schemes, k_pad, n_iter,
                                                      sorted_len, perm, cost, status);
  } else if (batch <= 256) {  // (at 512 the CTA radix sort is as fast: few warps, long chains)
    const int g = (n_iter + 3) / 4;
    if (batch <= 64)
      k_sort_cost_bitonic<2><<<g, 128, 0, s>>>(len, batch, off, schemes, n_schemes, k_pad, n_iter, sorted_len, perm, cost, status);
    else if (batch <= 128)
      k_sort_cost_bitonic<4><<<g, 128, 0, s>>>(len, batch, off, schemes, n_schemes, k_pad, n_iter, sorted_len, perm, cost, status);
    else
      k_sort_cost_bitonic<8><<<g, 128, 0, s>>>(len, batch, off, schemes, n_schemes, k_pad, n_iter, sorted_len, perm, cost, status);
  } else if (batch <= 2048) {
    const size_t sm = sort_cost_smem(batch, 256, n_schemes);
    e = cudaFuncSetAttribute(k_sort_cost<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return record_cuda_error(e);
    k_sort_cost<256><<<n_iter, 256, sm, s>>>(len, batch, off, schemes, n_schemes, k_pad, sorted_len,
                                              perm, cost, status);
  } else {
    const size_t sm = sort_cost_smem(batch, 1024, n_schemes);
    e = cudaFuncSetAttribute(k_sort_cost<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return record_cuda_error(e);
    k_sort_cost<1024><<<n_iter, 1024, sm, s>>>(len, batch, off, schemes, n_schemes, k_pad, sorted_len,
                                                perm, cost, status);
  }
  note_launch();
  e = cudaGetLastError();
  return e == cudaSuccess ? HYD_OK : record_cuda_error(e);
}

}  // namespace hyd
