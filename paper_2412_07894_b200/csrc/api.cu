// api.cu -- the extern "C" boundary of libhyd.so (include/hyd.h): host-side validation,
// launch planning, workspace layout and the end-to-end host-buffer call.
#include <atomic>
#include <cstring>

#include "hyd_internal.cuh"

namespace hyd {

int launch_sort_cost(const uint32_t*, int, int, const uint32_t*, const hyd_scheme*, int, int, uint32_t*, uint32_t*,
                     uint32_t*, uint32_t*, cudaStream_t);
size_t dispatch_workspace(int);
int launch_dispatch(const uint32_t*, const uint32_t*, int, int, const uint32_t*, size_t, int, const hyd_scheme*, int,
                    const uint8_t*, const uint8_t*, int, int, uint8_t*, uint64_t*, hyd_pipe_stats*,
                    uint32_t*, uint32_t*, void*, cudaStream_t);
size_t pack_workspace(int, int, int, int);
int launch_pack(const uint32_t*, const uint32_t*, int, int, const uint32_t*, size_t, int, const hyd_scheme*, int,
                const uint8_t*, const uint8_t*, int, int, const uint8_t*, const hyd_pipe_stats*,
                const uint32_t*, uint16_t*, uint16_t*, uint64_t*, uint64_t*, uint32_t*, void*, size_t,
                cudaStream_t);
int launch_pipe_index(const uint32_t*, const uint32_t*, int, int, const uint32_t*, size_t, int, const hyd_scheme*,
                      int, const uint8_t*, const uint8_t*, int, int, const uint8_t*, uint64_t*, hyd_pipe_stats*,
                      uint32_t*, uint32_t*, cudaStream_t);
int launch_small(const uint32_t*, const uint32_t*, int, int, const uint32_t*, size_t, int, const hyd_scheme*, int,
                 const uint8_t*, const uint8_t*, int, int, uint8_t*, uint64_t*, uint16_t*, uint16_t*, uint64_t*,
                 uint64_t*, uint32_t*, void*, cudaStream_t);
int launch_select(const uint64_t*, int, int, int, int64_t*, uint32_t*, cudaStream_t);
int launch_gather(const int64_t*, const uint32_t*, const uint8_t*, const uint16_t*, const uint16_t*,
                  const uint64_t*, int, int, const uint32_t*, size_t, int, int, uint8_t*, uint16_t*,
                  uint16_t*, uint64_t*, cudaStream_t);

int launch_alg1_perm(uint64_t, int, int, int, uint16_t*, cudaStream_t);
size_t alg1_workspace(int);
int launch_alg1(const uint32_t*, const uint32_t*, int, int, int, const hyd_scheme*, int,
                const uint8_t*, const uint8_t*, int, int, int, const uint16_t*, uint64_t*, uint8_t*,
                uint64_t*, hyd_pipe_stats*, uint32_t*, uint32_t*, void*, cudaStream_t);

int launch_eq3_exact(const uint32_t*, const uint32_t*, int, int, int, const hyd_scheme*, int,
                     const uint8_t*, const uint8_t*, int, const int32_t*, const int32_t*, int,
                     unsigned long long, uint64_t*, uint8_t*, uint64_t*, uint8_t*, uint32_t*,
                     cudaStream_t);
int launch_eq1_exact(const uint32_t*, const uint32_t*, int, int, int, const hyd_scheme*, int,
                     const uint8_t*, int, int, const uint32_t*, const int32_t*, const int32_t*,
                     const int32_t*, int, unsigned long long, uint32_t*, uint64_t*, uint64_t*,
                     uint8_t*, uint32_t*, cudaStream_t);
size_t dp_workspace(int, int);
int launch_dp_candidates(const uint8_t*, const uint8_t*, int, const hyd_scheme*, int, uint8_t*, uint8_t*, int32_t*,
                         cudaStream_t);
int launch_dp(const uint32_t*, int, const hyd_scheme*, int, int, int, int, int, uint64_t*, uint64_t*,
              int32_t*, uint16_t*, uint8_t*, uint8_t*, uint8_t*, uint32_t*, void*, cudaStream_t);

static std::atomic<int> g_launches{0};
static thread_local char g_err[256] = "no CUDA error";

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int record_cuda_error(cudaError_t e) {
  std::strncpy(g_err, cudaGetErrorString(e), sizeof(g_err) - 1);
  g_err[sizeof(g_err) - 1] = 0;
  return HYD_E_CUDA;
}

static bool common_ok(int n_iter, int batch, int n_schemes, int k_pad) {
  return n_iter >= 0 && n_iter <= HYD_MAX_ITER && batch >= 1 && batch <= HYD_MAX_BATCH && n_schemes >= 1 &&
         n_schemes <= HYD_MAX_SCHEMES && k_pad >= n_schemes && (k_pad % 4) == 0 &&
         k_pad <= HYD_MAX_SCHEMES;
}

static bool cand_ok(int n_cand, int max_np) {
  return n_cand >= 0 && n_cand < (1 << HYD_KEY_SHIFT) && max_np >= 1 && max_np <= HYD_MAX_PIPES;
}

static size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

struct AssignLayout {
  size_t off, len, schemes, cand, cand_np, sorted, perm, cost, pipe, lb, stats, members, mb, v, ptime, makespan, key,
      status, win_pipe, win_mb, win_v, win_ptime, disp_ws, pack_ws, pack_bytes, total;
};

// n_total: rows of the iteration-indexed arrays (n_iter * batch for uniform batches); batch: the
// largest batch (member row stride, workspace sizing)
static AssignLayout assign_layout(int n_iter, size_t n_total, int batch, int n_schemes, int k_pad,
                                  int n_cand, int max_np) {
  AssignLayout L;
  const size_t It = (size_t)n_iter, B = (size_t)batch, Cn = (size_t)n_cand, N = n_total;
  size_t o = 0;
  auto put = [&](size_t bytes) {
    const size_t at = o;
    o += al(bytes);
    return at;
  };
  L.off = put((It + 1) * 4);
  L.len = put(N * 4);
  L.schemes = put((size_t)n_schemes * sizeof(hyd_scheme));
  L.cand = put(Cn * HYD_MAX_PIPES);
  L.cand_np = put(Cn);
  L.sorted = put(N * 4);
  L.perm = put(N * 4);
  L.cost = put(N * (size_t)k_pad * 4);
  L.pipe = put(Cn * N);
  L.lb = put(Cn * It * 8);
  L.stats = put(Cn * It * (size_t)max_np * sizeof(hyd_pipe_stats));
  L.members = put(Cn * It * (size_t)max_np * ((B + 31) / 32) * 4);
  L.mb = put(Cn * N * 2);
  L.v = put(Cn * It * HYD_MAX_PIPES * 2);
  L.ptime = put(Cn * It * HYD_MAX_PIPES * 8);
  L.makespan = put(It * Cn * 8);
  L.key = put(It * 8);
  L.status = put(4);
  L.win_pipe = put(N);
  L.win_mb = put(N * 2);
  L.win_v = put(It * HYD_MAX_PIPES * 2);
  L.win_ptime = put(It * HYD_MAX_PIPES * 8);
  L.disp_ws = put(dispatch_workspace(n_iter));
  L.pack_bytes = pack_workspace(n_iter, batch, n_cand, max_np);
  L.pack_ws = put(L.pack_bytes);
  L.total = o;
  return L;
}

}  // namespace hyd

using namespace hyd;

extern "C" {

const char* hyd_status_string(int code) {
  switch (code) {
    case HYD_OK: return "ok";
    case HYD_E_INVALID: return "invalid argument (null pointer, size or limit)";
    case HYD_E_NOT_CANONICAL: return "candidate pipelines not in canonical (MaxLen desc, index asc) order";
    case HYD_E_OVERFLOW: return "cost overflow";
    case HYD_E_ZERO_COST: return "zero cost";
    case HYD_E_CUDA: return "CUDA error";
    case HYD_E_WORKSPACE: return "workspace missing or too small";
    case HYD_E_REDUCE: return "allreduce callback failed";
    default: return "unknown status";
  }
}

const char* hyd_last_cuda_error(void) { return g_err; }

int hyd_kernel_launches(void) { return g_launches.load(); }

int hyd_check_candidates(const uint8_t* cand_host, const uint8_t* cand_np_host, int n_cand,
                         const hyd_scheme* schemes_host, int n_schemes, int* max_np_out) {
  if (!cand_host || !cand_np_host || !schemes_host || n_cand < 0 || n_schemes < 1 ||
      n_schemes > HYD_MAX_SCHEMES)
    return HYD_E_INVALID;
  int mx = 0;
  for (int c = 0; c < n_cand; ++c) {
    const int np = cand_np_host[c];
    if (np < 1 || np > HYD_MAX_PIPES) return HYD_E_INVALID;
    mx = np > mx ? np : mx;
    for (int j = 0; j < np; ++j) {
      const int k = cand_host[(size_t)c * HYD_MAX_PIPES + j];
      if (k >= n_schemes) return HYD_E_INVALID;
      const hyd_scheme& s = schemes_host[k];
      if (s.max_len < 1 || s.pp < 1 || s.pp > HYD_MAX_PP) return HYD_E_INVALID;
      if (j > 0) {
        const int kp = cand_host[(size_t)c * HYD_MAX_PIPES + j - 1];
        const uint32_t mp = schemes_host[kp].max_len;
        if (s.max_len > mp || (s.max_len == mp && k < kp)) return HYD_E_NOT_CANONICAL;
      }
    }
  }
  if (max_np_out) *max_np_out = mx;
  return HYD_OK;
}

int hyd_cost_table(const uint32_t* len, int n_iter, int batch, const hyd_scheme* schemes,
                   int n_schemes, int k_pad, uint32_t* sorted_len, uint32_t* perm, uint32_t* cost,
                   uint32_t* status, void* stream) {
  if (!len || !schemes || !sorted_len || !perm || !cost || !status ||
      !common_ok(n_iter, batch, n_schemes, k_pad))
    return HYD_E_INVALID;
  return launch_sort_cost(len, n_iter, batch, nullptr, schemes, n_schemes, k_pad, sorted_len, perm,
                          cost, status, (cudaStream_t)stream);
}

int hyd_cost_table_ragged(const uint32_t* len, int n_iter, const uint32_t* offsets, int n_total,
                          int batch_max, const hyd_scheme* schemes, int n_schemes, int k_pad,
                          uint32_t* sorted_len, uint32_t* perm, uint32_t* cost, uint32_t* status,
                          void* stream) {
  if (!len || !offsets || !schemes || !sorted_len || !perm || !cost || !status || n_total < 0 ||
      !common_ok(n_iter, batch_max, n_schemes, k_pad))
    return HYD_E_INVALID;
  return launch_sort_cost(len, n_iter, batch_max, offsets, schemes, n_schemes, k_pad, sorted_len,
                          perm, cost, status, (cudaStream_t)stream);
}

size_t hyd_dispatch_workspace(int n_iter) {
  if (n_iter < 0) return 0;
  return dispatch_workspace(n_iter);
}

int hyd_dispatch(const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch,
                 int k_pad, const hyd_scheme* schemes, int n_schemes, const uint8_t* cand,
                 const uint8_t* cand_np, int n_cand, int max_np, uint8_t* pipe, uint64_t* lb,
                 hyd_pipe_stats* stats, uint32_t* members, uint32_t* status, void* ws,
                 size_t ws_bytes, void* stream) {
  if (!sorted_len || !cost || !schemes || !cand || !cand_np || !pipe || !lb || !stats || !members || !status ||
      !common_ok(n_iter, batch, n_schemes, k_pad) || !cand_ok(n_cand, max_np))
    return HYD_E_INVALID;
  if (!ws || ws_bytes < dispatch_workspace(n_iter)) return HYD_E_WORKSPACE;
  return launch_dispatch(sorted_len, cost, n_iter, batch, nullptr, (size_t)n_iter * batch, k_pad,
                         schemes, n_schemes, cand, cand_np, n_cand, max_np, pipe, lb, stats, members,
                         status, ws, (cudaStream_t)stream);
}

int hyd_dispatch_ragged(const uint32_t* sorted_len, const uint32_t* cost, int n_iter,
                        const uint32_t* offsets, int n_total, int batch_max, int k_pad,
                        const hyd_scheme* schemes, int n_schemes, const uint8_t* cand,
                        const uint8_t* cand_np, int n_cand, int max_np, uint8_t* pipe, uint64_t* lb,
                        hyd_pipe_stats* stats, uint32_t* members, uint32_t* status, void* ws,
                        size_t ws_bytes, void* stream) {
  if (!sorted_len || !cost || !offsets || !schemes || !cand || !cand_np || !pipe || !lb || !stats ||
      !members || !status || n_total < 0 || !common_ok(n_iter, batch_max, n_schemes, k_pad) ||
      !cand_ok(n_cand, max_np))
    return HYD_E_INVALID;
  if (!ws || ws_bytes < dispatch_workspace(n_iter)) return HYD_E_WORKSPACE;
  return launch_dispatch(sorted_len, cost, n_iter, batch_max, offsets, (size_t)n_total, k_pad,
                         schemes, n_schemes, cand, cand_np, n_cand, max_np, pipe, lb, stats, members,
                         status, ws, (cudaStream_t)stream);
}

int hyd_pipe_index(const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch, int k_pad,
                   const hyd_scheme* schemes, int n_schemes, const uint8_t* cand, const uint8_t* cand_np,
                   int n_cand, int max_np, const uint8_t* pipe, uint64_t* lb, hyd_pipe_stats* stats,
                   uint32_t* members, uint32_t* status, void* stream) {
  if (!sorted_len || !cost || !schemes || !cand || !cand_np || !pipe || !stats || !members || !status ||
      !common_ok(n_iter, batch, n_schemes, k_pad) || !cand_ok(n_cand, max_np))
    return HYD_E_INVALID;
  return launch_pipe_index(sorted_len, cost, n_iter, batch, nullptr, (size_t)n_iter * batch, k_pad, schemes,
                           n_schemes, cand, cand_np, n_cand, max_np, pipe, lb, stats, members, status,
                           (cudaStream_t)stream);
}

int hyd_pipe_index_ragged(const uint32_t* sorted_len, const uint32_t* cost, int n_iter,
                          const uint32_t* offsets, int n_total, int batch_max, int k_pad,
                          const hyd_scheme* schemes, int n_schemes, const uint8_t* cand,
                          const uint8_t* cand_np, int n_cand, int max_np, const uint8_t* pipe,
                          uint64_t* lb, hyd_pipe_stats* stats, uint32_t* members, uint32_t* status,
                          void* stream) {
  if (!sorted_len || !cost || !offsets || !schemes || !cand || !cand_np || !pipe || !stats || !members ||
      !status || n_total < 0 || !common_ok(n_iter, batch_max, n_schemes, k_pad) || !cand_ok(n_cand, max_np))
    return HYD_E_INVALID;
  return launch_pipe_index(sorted_len, cost, n_iter, batch_max, offsets, (size_t)n_total, k_pad, schemes,
                           n_schemes, cand, cand_np, n_cand, max_np, pipe, lb, stats, members, status,
                           (cudaStream_t)stream);
}

size_t hyd_alg1_workspace(int n_iter) {
  if (n_iter < 0) return 0;
  return alg1_workspace(n_iter);
}

int hyd_alg1_permutations(uint64_t seed, int n_iter, int batch, int trials, uint16_t* order,
                          void* stream) {
  if (!order || n_iter < 0 || n_iter > HYD_MAX_ITER || batch < 1 || batch > HYD_MAX_BATCH || trials < 1 ||
      trials > HYD_MAX_TRIALS)
    return HYD_E_INVALID;
  return launch_alg1_perm(seed, n_iter, batch, trials, order, (cudaStream_t)stream);
}

int hyd_dispatch_alg1(const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch,
                      int k_pad, const hyd_scheme* schemes, int n_schemes, const uint8_t* cand,
                      const uint8_t* cand_np, int n_cand, int max_np, int trials,
                      const uint16_t* order, uint64_t* best, uint8_t* pipe, uint64_t* lb,
                      hyd_pipe_stats* stats, uint32_t* members, uint32_t* status, void* ws,
                      size_t ws_bytes, void* stream) {
  if (!sorted_len || !cost || !schemes || !cand || !cand_np || !order || !best || !pipe || !lb ||
      !stats || !members || !status || !common_ok(n_iter, batch, n_schemes, k_pad) ||
      !cand_ok(n_cand, max_np) || trials < 1 || trials > HYD_MAX_TRIALS)
    return HYD_E_INVALID;
  if (!ws || ws_bytes < alg1_workspace(n_iter)) return HYD_E_WORKSPACE;
  return launch_alg1(sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np,
                     n_cand, max_np, trials, order, best, pipe, lb, stats, members, status, ws,
                     (cudaStream_t)stream);
}

int hyd_eq3_exact(const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch, int k_pad,
                  const hyd_scheme* schemes, int n_schemes, const uint8_t* cand,
                  const uint8_t* cand_np, int n_cand, const int32_t* pair_c, const int32_t* pair_t,
                  int n_pairs, uint64_t node_limit, uint64_t* value, uint8_t* pipe, uint64_t* nodes,
                  uint8_t* proved, uint32_t* status, void* stream) {
  if (!sorted_len || !cost || !schemes || !cand || !cand_np || !pair_c || !pair_t || !value ||
      !pipe || !nodes || !proved || !status || n_pairs < 0 || batch > HYD_BB_MAX_BATCH ||
      !common_ok(n_iter, batch, n_schemes, k_pad) || n_cand < 0)
    return HYD_E_INVALID;
  return launch_eq3_exact(sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, cand_np,
                          n_cand, pair_c, pair_t, n_pairs, node_limit, value, pipe, nodes, proved,
                          status, (cudaStream_t)stream);
}

int hyd_eq1_exact(const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch, int k_pad,
                  const hyd_scheme* schemes, int n_schemes, const uint8_t* cand, int n_cand,
                  int max_np, const uint32_t* members, const int32_t* pair_c, const int32_t* pair_t,
                  const int32_t* pair_j, int n_pairs, uint64_t node_limit, uint32_t* v,
                  uint64_t* obj, uint64_t* nodes, uint8_t* proved, uint32_t* status, void* stream) {
  if (!sorted_len || !cost || !schemes || !cand || !members || !pair_c || !pair_t || !pair_j ||
      !v || !obj || !nodes || !proved || !status || n_pairs < 0 ||
      !common_ok(n_iter, batch, n_schemes, k_pad) || !cand_ok(n_cand, max_np))
    return HYD_E_INVALID;
  return launch_eq1_exact(sorted_len, cost, n_iter, batch, k_pad, schemes, n_schemes, cand, n_cand,
                          max_np, members, pair_c, pair_t, pair_j, n_pairs, node_limit, v, obj,
                          nodes, proved, status, (cudaStream_t)stream);
}

size_t hyd_dp_workspace(int n_schemes, int J) {
  if (n_schemes < 1 || J < 1) return 0;
  return dp_workspace(n_schemes, J);
}

int hyd_dp_propose(const uint32_t* lengths, int n_seq, const hyd_scheme* schemes, int n_schemes,
                   int step, int J, int n_gpus, int scale, uint64_t* t_num, uint64_t* t_den,
                   int32_t* choice, uint16_t* counts, uint8_t* rows, uint8_t* valid, uint8_t* keep,
                   uint32_t* status, void* ws, size_t ws_bytes, void* stream) {
  if (!lengths || !schemes || !t_num || !t_den || !choice || !counts || !rows || !valid || !keep ||
      !status || n_seq < 0 || n_schemes < 1 || n_schemes > HYD_MAX_SCHEMES || step < 1 || J < 1 ||
      J > 4095 || n_gpus < 1 || scale < 1 || (long long)n_gpus * scale > 4095 ||
      (long long)J * step > HYD_LEN_LIMIT)
    return HYD_E_INVALID;
  if (!ws || ws_bytes < dp_workspace(n_schemes, J)) return HYD_E_WORKSPACE;
  return launch_dp(lengths, n_seq, schemes, n_schemes, step, J, n_gpus, scale, t_num, t_den, choice,
                   counts, rows, valid, keep, status, ws, (cudaStream_t)stream);
}

int hyd_dp_candidates(const uint8_t* rows, const uint8_t* keep, int J, const hyd_scheme* schemes,
                      int n_schemes, uint8_t* cand, uint8_t* cand_np, int32_t* n_out, void* stream) {
  if (!rows || !keep || !schemes || !cand || !cand_np || !n_out || J < 1 || J > 4095 || n_schemes < 1 ||
      n_schemes > HYD_MAX_SCHEMES)
    return HYD_E_INVALID;
  return launch_dp_candidates(rows, keep, J, schemes, n_schemes, cand, cand_np, n_out, (cudaStream_t)stream);
}

size_t hyd_pack_workspace(int n_iter, int batch, int n_cand, int max_np) {
  if (n_iter < 0 || batch < 1 || n_cand < 0 || max_np < 1) return 0;
  return pack_workspace(n_iter, batch, n_cand, max_np);
}

int hyd_pack(const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch, int k_pad,
             const hyd_scheme* schemes, int n_schemes, const uint8_t* cand, const uint8_t* cand_np,
             int n_cand, int max_np, const uint8_t* pipe, const hyd_pipe_stats* stats,
             const uint32_t* members, uint16_t* mb, uint16_t* v, uint64_t* ptime, uint64_t* makespan,
             uint32_t* status, void* ws, size_t ws_bytes, void* stream) {
  if (!sorted_len || !cost || !schemes || !cand || !cand_np || !pipe || !stats || !members || !mb || !v || !ptime ||
      !makespan || !status || !common_ok(n_iter, batch, n_schemes, k_pad) ||
      !cand_ok(n_cand, max_np))
    return HYD_E_INVALID;
  if (!ws || ws_bytes < pack_workspace(n_iter, batch, n_cand, max_np)) return HYD_E_WORKSPACE;
  return launch_pack(sorted_len, cost, n_iter, batch, nullptr, (size_t)n_iter * batch, k_pad,
                     schemes, n_schemes, cand, cand_np, n_cand, max_np, pipe, stats, members, mb, v,
                     ptime, makespan, status, ws, ws_bytes, (cudaStream_t)stream);
}

int hyd_pack_ragged(const uint32_t* sorted_len, const uint32_t* cost, int n_iter,
                    const uint32_t* offsets, int n_total, int batch_max, int k_pad,
                    const hyd_scheme* schemes, int n_schemes, const uint8_t* cand,
                    const uint8_t* cand_np, int n_cand, int max_np, const uint8_t* pipe,
                    const hyd_pipe_stats* stats, const uint32_t* members, uint16_t* mb, uint16_t* v,
                    uint64_t* ptime, uint64_t* makespan, uint32_t* status, void* ws,
                    size_t ws_bytes, void* stream) {
  if (!sorted_len || !cost || !offsets || !schemes || !cand || !cand_np || !pipe || !stats ||
      !members || !mb || !v || !ptime || !makespan || !status || n_total < 0 ||
      !common_ok(n_iter, batch_max, n_schemes, k_pad) || !cand_ok(n_cand, max_np))
    return HYD_E_INVALID;
  if (!ws || ws_bytes < pack_workspace(n_iter, batch_max, n_cand, max_np)) return HYD_E_WORKSPACE;
  return launch_pack(sorted_len, cost, n_iter, batch_max, offsets, (size_t)n_total, k_pad, schemes,
                     n_schemes, cand, cand_np, n_cand, max_np, pipe, stats, members, mb, v, ptime,
                     makespan, status, ws, ws_bytes, (cudaStream_t)stream);
}

size_t hyd_dispatch_pack_workspace(void) { return 256; }

static bool small_ok(int batch, int max_np) { return batch <= HYD_SMALL_MAX_BATCH && max_np <= 16; }

int hyd_dispatch_pack(const uint32_t* sorted_len, const uint32_t* cost, int n_iter, int batch, int k_pad,
                      const hyd_scheme* schemes, int n_schemes, const uint8_t* cand, const uint8_t* cand_np,
                      int n_cand, int max_np, uint8_t* pipe, uint64_t* lb, uint16_t* mb, uint16_t* v,
                      uint64_t* ptime, uint64_t* makespan, uint32_t* status, void* ws, size_t ws_bytes,
                      void* stream) {
  if (!sorted_len || !cost || !schemes || !cand || !cand_np || !pipe || !lb || !mb || !v || !ptime || !makespan ||
      !status || !common_ok(n_iter, batch, n_schemes, k_pad) || !cand_ok(n_cand, max_np) || !small_ok(batch, max_np))
    return HYD_E_INVALID;
  if (!ws || ws_bytes < hyd_dispatch_pack_workspace()) return HYD_E_WORKSPACE;
  return launch_small(sorted_len, cost, n_iter, batch, nullptr, (size_t)n_iter * batch, k_pad, schemes, n_schemes,
                      cand, cand_np, n_cand, max_np, pipe, lb, mb, v, ptime, makespan, status, ws,
                      (cudaStream_t)stream);
}

int hyd_dispatch_pack_ragged(const uint32_t* sorted_len, const uint32_t* cost, int n_iter,
                             const uint32_t* offsets, int n_total, int batch_max, int k_pad,
                             const hyd_scheme* schemes, int n_schemes, const uint8_t* cand,
                             const uint8_t* cand_np, int n_cand, int max_np, uint8_t* pipe, uint64_t* lb,
                             uint16_t* mb, uint16_t* v, uint64_t* ptime, uint64_t* makespan,
                             uint32_t* status, void* ws, size_t ws_bytes, void* stream) {
  if (!sorted_len || !cost || !offsets || !schemes || !cand || !cand_np || !pipe || !lb || !mb || !v || !ptime ||
      !makespan || !status || n_total < 0 || !common_ok(n_iter, batch_max, n_schemes, k_pad) ||
      !cand_ok(n_cand, max_np) || !small_ok(batch_max, max_np))
    return HYD_E_INVALID;
  if (!ws || ws_bytes < hyd_dispatch_pack_workspace()) return HYD_E_WORKSPACE;
  return launch_small(sorted_len, cost, n_iter, batch_max, offsets, (size_t)n_total, k_pad, schemes, n_schemes,
                      cand, cand_np, n_cand, max_np, pipe, lb, mb, v, ptime, makespan, status, ws,
                      (cudaStream_t)stream);
}

int hyd_select_best(const uint64_t* makespan, int n_iter, int n_cand, int cand_offset,
                    int64_t* key, uint32_t* status, void* stream) {
  if (!makespan || !key || !status || n_iter < 0 || n_iter > HYD_MAX_ITER || n_cand < 0 || cand_offset < 0 ||
      (long long)n_cand + cand_offset > (1ll << HYD_KEY_SHIFT) - 1)
    return HYD_E_INVALID;
  return launch_select(makespan, n_iter, n_cand, cand_offset, key, status, (cudaStream_t)stream);
}

int hyd_gather_winners(const int64_t* key, const uint32_t* perm, const uint8_t* pipe,
                       const uint16_t* mb, const uint16_t* v, const uint64_t* ptime, int n_iter,
                       int batch, int n_cand, int cand_offset, uint8_t* win_pipe, uint16_t* win_mb,
                       uint16_t* win_v, uint64_t* win_ptime, void* stream) {
  if (!key || !perm || !pipe || !mb || !v || !ptime || !win_pipe || !win_mb || !win_v ||
      !win_ptime || n_iter < 0 || n_iter > HYD_MAX_ITER || batch < 1 || batch > HYD_MAX_BATCH || n_cand < 0 ||
      cand_offset < 0)
    return HYD_E_INVALID;
  return launch_gather(key, perm, pipe, mb, v, ptime, n_iter, batch, nullptr, (size_t)n_iter * batch,
                       n_cand, cand_offset, win_pipe, win_mb, win_v, win_ptime, (cudaStream_t)stream);
}

int hyd_gather_winners_ragged(const int64_t* key, const uint32_t* perm, const uint8_t* pipe,
                              const uint16_t* mb, const uint16_t* v, const uint64_t* ptime,
                              int n_iter, const uint32_t* offsets, int n_total, int batch_max,
                              int n_cand, int cand_offset, uint8_t* win_pipe, uint16_t* win_mb,
                              uint16_t* win_v, uint64_t* win_ptime, void* stream) {
  if (!key || !perm || !pipe || !mb || !v || !ptime || !offsets || !win_pipe || !win_mb ||
      !win_v || !win_ptime || n_iter < 0 || n_iter > HYD_MAX_ITER || n_total < 0 || batch_max < 1 ||
      batch_max > HYD_MAX_BATCH || n_cand < 0 || cand_offset < 0)
    return HYD_E_INVALID;
  return launch_gather(key, perm, pipe, mb, v, ptime, n_iter, batch_max, offsets, (size_t)n_total,
                       n_cand, cand_offset, win_pipe, win_mb, win_v, win_ptime, (cudaStream_t)stream);
}

size_t hyd_assign_workspace(int n_iter, int batch, int n_schemes, int k_pad, int n_cand, int max_np) {
  if (!common_ok(n_iter, batch, n_schemes, k_pad) || !cand_ok(n_cand, max_np)) return 0;
  return assign_layout(n_iter, (size_t)n_iter * batch, batch, n_schemes, k_pad, n_cand, max_np).total;
}

size_t hyd_assign_key_offset(int n_iter, int batch, int n_schemes, int k_pad, int n_cand, int max_np) {
  return assign_layout(n_iter, (size_t)n_iter * batch, batch, n_schemes, k_pad, n_cand, max_np).key;
}

size_t hyd_assign_workspace_ragged(int n_iter, int n_total, int batch_max, int n_schemes, int k_pad,
                                   int n_cand, int max_np) {
  if (n_total < 0 || !common_ok(n_iter, batch_max, n_schemes, k_pad) || !cand_ok(n_cand, max_np))
    return 0;
  return assign_layout(n_iter, (size_t)n_total, batch_max, n_schemes, k_pad, n_cand, max_np).total;
}

size_t hyd_assign_key_offset_ragged(int n_iter, int n_total, int batch_max, int n_schemes,
                                    int k_pad, int n_cand, int max_np) {
  return assign_layout(n_iter, (size_t)n_total, batch_max, n_schemes, k_pad, n_cand, max_np).key;
}

// e2e host-buffer call; offsets_host == nullptr: uniform batches of `batch`, else CSR offsets
// [n_iter + 1] of ragged batches whose largest is `batch`
static int assign_host_impl(const uint32_t* len_host, int n_iter, const uint32_t* offsets_host,
                            int batch, const hyd_scheme* schemes_host, int n_schemes, int k_pad,
                            const uint8_t* cand_host, const uint8_t* cand_np_host, int n_cand,
                            int cand_offset, int64_t* key_host, uint8_t* win_pipe_host,
                            uint16_t* win_mb_host, uint16_t* win_v_host, uint64_t* win_ptime_host,
                            uint32_t* status_host, hyd_collective_fn coll, void* coll_user,
                            void* ws, size_t ws_bytes, void* stream) {
  if (!len_host || !schemes_host || !cand_host || !cand_np_host || !key_host || !win_pipe_host ||
      !win_mb_host || !win_v_host || !win_ptime_host || !status_host ||
      !common_ok(n_iter, batch, n_schemes, k_pad) || cand_offset < 0 ||
      (long long)n_cand + cand_offset > (1ll << HYD_KEY_SHIFT) - 1)
    return HYD_E_INVALID;
  int max_np = 0;
  int rc = hyd_check_candidates(cand_host, cand_np_host, n_cand, schemes_host, n_schemes, &max_np);
  if (rc != HYD_OK) return rc;
  if (n_cand == 0) max_np = 1;
  size_t n_total = (size_t)n_iter * batch;
  if (offsets_host) {  // host-side CSR check: 0 = off[0] <= ... , 1 <= B_t <= batch
    if (offsets_host[0] != 0) return HYD_E_INVALID;
    for (int t = 0; t < n_iter; ++t) {
      const uint32_t d = offsets_host[t + 1] - offsets_host[t];
      if (offsets_host[t + 1] < offsets_host[t] || d < 1 || d > (uint32_t)batch) return HYD_E_INVALID;
    }
    n_total = offsets_host[n_iter];
  }
  const AssignLayout L = assign_layout(n_iter, n_total, batch, n_schemes, k_pad, n_cand, max_np);
  if (!ws || ws_bytes < L.total) return HYD_E_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  char* w = static_cast<char*>(ws);
  auto D = [&](size_t off) { return static_cast<void*>(w + off); };
  const size_t It = (size_t)n_iter, N = n_total, Cn = (size_t)n_cand;
  cudaError_t e;
#define HYD_CK(x)                                      \
  do {                                                 \
    e = (x);                                           \
    if (e != cudaSuccess) return record_cuda_error(e); \
  } while (0)
  HYD_CK(cudaMemsetAsync(D(L.status), 0, 4, s));
  HYD_CK(cudaMemcpyAsync(D(L.len), len_host, N * 4, cudaMemcpyHostToDevice, s));
  const uint32_t* off = nullptr;
  if (offsets_host) {
    HYD_CK(cudaMemcpyAsync(D(L.off), offsets_host, (It + 1) * 4, cudaMemcpyHostToDevice, s));
    off = static_cast<const uint32_t*>(D(L.off));
  }
  HYD_CK(cudaMemcpyAsync(D(L.schemes), schemes_host, (size_t)n_schemes * sizeof(hyd_scheme),
                         cudaMemcpyHostToDevice, s));
  if (Cn) {
    HYD_CK(cudaMemcpyAsync(D(L.cand), cand_host, Cn * HYD_MAX_PIPES, cudaMemcpyHostToDevice, s));
    HYD_CK(cudaMemcpyAsync(D(L.cand_np), cand_np_host, Cn, cudaMemcpyHostToDevice, s));
  }
  uint32_t* st = static_cast<uint32_t*>(D(L.status));
  auto* sorted = static_cast<uint32_t*>(D(L.sorted));
  auto* perm = static_cast<uint32_t*>(D(L.perm));
  auto* cost = static_cast<uint32_t*>(D(L.cost));
  auto* sch = static_cast<const hyd_scheme*>(D(L.schemes));
  auto* cand = static_cast<const uint8_t*>(D(L.cand));
  auto* cnp = static_cast<const uint8_t*>(D(L.cand_np));
  auto* pipe = static_cast<uint8_t*>(D(L.pipe));
  auto* mb = static_cast<uint16_t*>(D(L.mb));
  auto* vv = static_cast<uint16_t*>(D(L.v));
  auto* pt = static_cast<uint64_t*>(D(L.ptime));
  auto* ms = static_cast<uint64_t*>(D(L.makespan));
  auto* key = static_cast<int64_t*>(D(L.key));
  rc = launch_sort_cost(static_cast<const uint32_t*>(D(L.len)), n_iter, batch, off, sch, n_schemes,
                        k_pad, sorted, perm, cost, st, s);
  if (rc) return rc;
  auto* pst = static_cast<hyd_pipe_stats*>(D(L.stats));
  auto* mem = static_cast<uint32_t*>(D(L.members));
  if (batch <= HYD_SMALL_MAX_BATCH && max_np <= 16) {  // a3 + a4 in one kernel (hyd_dispatch_pack)
    rc = launch_small(sorted, cost, n_iter, batch, off, N, k_pad, sch, n_schemes, cand, cnp, n_cand, max_np, pipe,
                      static_cast<uint64_t*>(D(L.lb)), mb, vv, pt, ms, st, D(L.disp_ws), s);
    if (rc) return rc;
  } else {
    rc = launch_dispatch(sorted, cost, n_iter, batch, off, N, k_pad, sch, n_schemes, cand, cnp, n_cand, max_np,
                         pipe, static_cast<uint64_t*>(D(L.lb)), pst, mem, st, D(L.disp_ws), s);
    if (rc) return rc;
    rc = launch_pack(sorted, cost, n_iter, batch, off, N, k_pad, sch, n_schemes, cand, cnp, n_cand, max_np,
                     pipe, pst, mem, mb, vv, pt, ms, st, D(L.pack_ws), L.pack_bytes, s);
    if (rc) return rc;
  }
  rc = launch_select(ms, n_iter, n_cand, cand_offset, key, st, s);
  if (rc) return rc;
  if (coll && coll(key, It, HYD_COLL_MIN_I64, coll_user, stream) != 0) return HYD_E_REDUCE;
  // winner rows: zero-filled block, each rank writes the iterations its candidates won
  const size_t rows_bytes = L.disp_ws - L.win_pipe;  // win_pipe | win_mb | win_v | win_ptime (256-aligned)
  HYD_CK(cudaMemsetAsync(D(L.win_pipe), 0, rows_bytes, s));
  rc = launch_gather(key, perm, pipe, mb, vv, pt, n_iter, batch, off, N, n_cand, cand_offset,
                     static_cast<uint8_t*>(D(L.win_pipe)), static_cast<uint16_t*>(D(L.win_mb)),
                     static_cast<uint16_t*>(D(L.win_v)), static_cast<uint64_t*>(D(L.win_ptime)), s);
  if (rc) return rc;
  if (coll && coll(D(L.win_pipe), rows_bytes / 4, HYD_COLL_SUM_I32, coll_user, stream) != 0) return HYD_E_REDUCE;
  HYD_CK(cudaMemcpyAsync(key_host, key, It * 8, cudaMemcpyDeviceToHost, s));
  HYD_CK(cudaMemcpyAsync(win_pipe_host, D(L.win_pipe), N, cudaMemcpyDeviceToHost, s));
  HYD_CK(cudaMemcpyAsync(win_mb_host, D(L.win_mb), N * 2, cudaMemcpyDeviceToHost, s));
  HYD_CK(cudaMemcpyAsync(win_v_host, D(L.win_v), It * HYD_MAX_PIPES * 2, cudaMemcpyDeviceToHost, s));
  HYD_CK(cudaMemcpyAsync(win_ptime_host, D(L.win_ptime), It * HYD_MAX_PIPES * 8, cudaMemcpyDeviceToHost, s));
  HYD_CK(cudaMemcpyAsync(status_host, st, 4, cudaMemcpyDeviceToHost, s));
  HYD_CK(cudaStreamSynchronize(s));
#undef HYD_CK
  return HYD_OK;
}

int hyd_assign_host(const uint32_t* len_host, int n_iter, int batch, const hyd_scheme* schemes_host,
                    int n_schemes, int k_pad, const uint8_t* cand_host, const uint8_t* cand_np_host,
                    int n_cand, int cand_offset, int64_t* key_host, uint8_t* win_pipe_host,
                    uint16_t* win_mb_host, uint16_t* win_v_host, uint64_t* win_ptime_host,
                    uint32_t* status_host, hyd_collective_fn coll, void* coll_user, void* ws,
                    size_t ws_bytes, void* stream) {
  return assign_host_impl(len_host, n_iter, nullptr, batch, schemes_host, n_schemes, k_pad,
                          cand_host, cand_np_host, n_cand, cand_offset, key_host, win_pipe_host,
                          win_mb_host, win_v_host, win_ptime_host, status_host, coll, coll_user,
                          ws, ws_bytes, stream);
}

int hyd_assign_host_ragged(const uint32_t* len_host, int n_iter, const uint32_t* offsets_host,
                           int batch_max, const hyd_scheme* schemes_host, int n_schemes, int k_pad,
                           const uint8_t* cand_host, const uint8_t* cand_np_host, int n_cand,
                           int cand_offset, int64_t* key_host, uint8_t* win_pipe_host,
                           uint16_t* win_mb_host, uint16_t* win_v_host, uint64_t* win_ptime_host,
                           uint32_t* status_host, hyd_collective_fn coll, void* coll_user, void* ws,
                           size_t ws_bytes, void* stream) {
  if (!offsets_host) return HYD_E_INVALID;
  return assign_host_impl(len_host, n_iter, offsets_host, batch_max, schemes_host, n_schemes, k_pad,
                          cand_host, cand_np_host, n_cand, cand_offset, key_host, win_pipe_host,
                          win_mb_host, win_v_host, win_ptime_host, status_host, coll, coll_user,
                          ws, ws_bytes, stream);
}

}  // extern "C"
