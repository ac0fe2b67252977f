"""Per-iteration 64-bit digests of the assignment outputs, for full-size parity (no method
arithmetic: a hash of bytes in a fixed layout).  Both the golden writer
(tools/make_golden_digests.py, oracle outputs) and the GPU parity test (tests/test_digests_gpu.py,
C-ABI outputs) call ``iteration_digests`` on arrays in the include/hyd.h layouts:

  sorted_len, perm [It][B] u32; cost [It][B][k_pad] u32; pipe [C][It][B] u8; lb [C][It] u64;
  mb [C][It][B] u16; v [C][It][32] u16; ptime [C][It][32] u64; makespan [It][C] u64; key [It] i64
  (ragged batches: sorted_len / perm [N], cost [N][k_pad], pipe / mb [C][N], rows of t at
  offsets[t] .. offsets[t+1]).

Digest of (array, t) = the first 8 bytes (little-endian u64) of BLAKE2b over the bytes of
iteration t's slice taken over ALL candidates in candidate order (C-contiguous copy)."""
from __future__ import annotations

import hashlib

import numpy as np

ITER_MAJOR = ("sorted_len", "perm", "cost")  # [It][...]
CAND_MAJOR = ("pipe", "mb", "v", "ptime")  # [C][It][...]
NAMES = ITER_MAJOR + CAND_MAJOR + ("lb", "makespan", "key")


def _h(a) -> int:
    return int.from_bytes(hashlib.blake2b(np.ascontiguousarray(a).tobytes(), digest_size=8).digest(), "little")


def iteration_digests(out: dict, n_iter: int, offsets=None, t_lo: int = 0) -> dict:
    """{name: u64[n_iter]} for the iterations [t_lo, t_lo + n_iter) of ``out`` (whose arrays hold
    exactly those iterations)."""
    res = {k: np.zeros(n_iter, np.uint64) for k in NAMES if k in out}
    off = None if offsets is None else np.asarray(offsets, np.int64)
    for t in range(n_iter):
        rows = slice(off[t] - off[0], off[t + 1] - off[0]) if off is not None else None
        for k in res:
            a = out[k]
            if k in ITER_MAJOR:
                s = a[rows] if rows is not None else a[t]
            elif k in ("pipe", "mb"):
                s = a[:, rows] if rows is not None else a[:, t]
            elif k in ("v", "ptime", "lb"):
                s = a[:, t]
            elif k == "makespan":
                s = a[t]
            else:  # key
                s = a[t : t + 1]
            res[k][t] = _h(s)
    return res
