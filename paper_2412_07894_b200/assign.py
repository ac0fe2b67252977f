"""Host-side driver of the two-stage assignment: device buffers, the four C-ABI calls,
the cross-GPU argmin (a6) and shard planning.  No arithmetic of the method lives here;
every step runs in libhyd.so's sm_100a kernels (see include/hyd.h).

Multi-GPU: one process per GPU.  Candidates are split into contiguous
blocks [rank*C/G, (rank+1)*C/G); every rank sorts and costs all iterations itself
(redundant but tiny, avoids a broadcast); the only exchange is one
``all_reduce(key, MIN)`` of It int64 keys over NCCL -- key = makespan << 20 | c_global,
so the minimum key is the global argmin of (makespan, c).  With fewer candidates than
ranks, iterations are split instead and no collective is needed.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import hyd

KEY_MASK = (1 << hyd.KEY_SHIFT) - 1


@dataclass(frozen=True)
class Shard:
    cand_lo: int
    cand_hi: int
    iter_lo: int
    iter_hi: int
    by: str  # "cand" | "iter" | "none"

    @property
    def needs_reduce(self) -> bool:
        return self.by == "cand"


def plan_shard(n_cand: int, n_iter: int, world: int, rank: int) -> Shard:
    """Contiguous candidate blocks; iterations when candidates are fewer than ranks."""
    if world <= 1:
        return Shard(0, n_cand, 0, n_iter, "none")
    if n_cand >= world:
        return Shard(rank * n_cand // world, (rank + 1) * n_cand // world, 0, n_iter, "cand")
    return Shard(0, n_cand, rank * n_iter // world, (rank + 1) * n_iter // world, "iter")


def decode_key(key):
    """key -> (makespan, global candidate) ; (-1, -1) for an all-infeasible iteration."""
    key = np.asarray(key, dtype=np.int64)
    feas = key != hyd.INT64_MAX
    ms = np.where(feas, key >> hyd.KEY_SHIFT, -1)
    c = np.where(feas, key & KEY_MASK, -1)
    return ms, c


def reduce_keys(key, group=None):
    """a6: the cross-GPU argmin -- one allreduce(MIN) of the per-iteration int64 keys."""
    import torch.distributed as dist

    dist.all_reduce(key, op=dist.ReduceOp.MIN, group=group)
    return key


def share_rows(words, group=None):
    """Winner follow-up: allreduce(SUM) of the zero-filled winner-row block
    (int32 words); each iteration's rows are non-zero on the one rank that owns its winner,
    so the sum is that rank's rows and every rank receives every iteration's plan."""
    import torch.distributed as dist

    dist.all_reduce(words, op=dist.ReduceOp.SUM, group=group)
    return words


def schemes_bytes(schemes) -> np.ndarray:
    s = np.ascontiguousarray(schemes)
    assert s.dtype.itemsize == 48
    return s.view(np.uint8).reshape(-1)


class Assigner:
    """Device-resident buffers + the a1-a5 launch sequence for one (shard of a) workload.

    ``schemes``: structured array (48-byte hyd_scheme records); ``cand`` [C][32] u8;
    ``cand_np`` [C] u8 -- this rank's candidates, global index = cand_offset + local.
    ``trials`` > 0 replaces the HYD-H1 dispatch by Alg. 1 with that many random trials per
    (c,t) (NEXT-1, include/hyd.h hyd_dispatch_alg1), its permutations drawn from ``seed``.
    ``offsets`` (host CSR [It + 1], NEXT-2): ragged token-budget batches; ``batch`` is then the
    largest batch and every iteration-indexed array has ``offsets[-1]`` rows.
    """

    def __init__(self, schemes, cand, cand_np, n_iter, batch, k_pad, cand_offset=0, device=None, trials=0,
                 seed=0, offsets=None, fused=None):
        import torch

        self.torch = torch
        self.dev = torch.device(device if device is not None else "cuda")
        self.n_iter, self.batch, self.k_pad = int(n_iter), int(batch), int(k_pad)
        self.n_schemes = int(len(schemes))
        self.n_cand = int(cand.shape[0])
        self.cand_offset = int(cand_offset)
        self.max_np = hyd.check_candidates(cand, cand_np, schemes) if self.n_cand else 1
        ml = np.zeros((self.n_cand, hyd.MAX_PIPES), np.int64)
        for c in range(self.n_cand):
            ks = cand[c, : int(cand_np[c])]
            ml[c, : len(ks)] = schemes["max_len"][ks]
        self._ml = ml
        self._ml_k = schemes["max_len"].astype(np.int64)
        mult = np.zeros((self.n_cand, self.n_schemes), np.int64)
        for c in range(self.n_cand):
            for k in cand[c, : int(cand_np[c])]:
                mult[c, k] += 1
        self._mult = mult
        u8, dev = torch.uint8, self.dev
        self.schemes = torch.from_numpy(schemes_bytes(schemes).copy()).to(dev)
        self.cand = torch.from_numpy(np.ascontiguousarray(cand, dtype=np.uint8)).to(dev)
        self.cand_np = torch.from_numpy(np.ascontiguousarray(cand_np, dtype=np.uint8)).to(dev)
        It, B, Cn, kp = self.n_iter, self.batch, self.n_cand, self.k_pad
        i32 = torch.int32  # u32 buffers are carried as int32 storage
        self.ragged = offsets is not None
        if self.ragged:
            if trials:
                raise hyd.HydError("Alg. 1 (trials) runs on uniform batches only")
            off = np.ascontiguousarray(offsets, dtype=np.uint32)
            assert off.shape == (It + 1,) and off[0] == 0 and (np.diff(off.astype(np.int64)) >= 1).all()
            assert int(np.diff(off.astype(np.int64)).max()) <= B
            self.offsets_host = off
            self.off = torch.from_numpy(off.view(np.int32).copy()).to(dev)
            self.n_total = int(off[-1])
            rows = (self.n_total,)
        else:
            self.n_total = It * B
            rows = (It, B)
        N = self.n_total
        self.sorted_len = torch.empty(rows, dtype=i32, device=dev)
        self.perm = torch.empty(rows, dtype=i32, device=dev)
        self.cost = torch.empty(rows + (kp,), dtype=i32, device=dev)
        self.pipe = torch.empty((Cn, N) if self.ragged else (Cn, It, B), dtype=u8, device=dev)
        self.lb = torch.empty((Cn, It), dtype=torch.int64, device=dev)
        self.stats = torch.empty((Cn, It, self.max_np, hyd.PIPE_STATS_BYTES), dtype=u8, device=dev)
        self.members = torch.empty((It, Cn, (B + 31) // 32, self.max_np), dtype=i32, device=dev)
        self.mb = torch.empty((Cn, N) if self.ragged else (Cn, It, B), dtype=torch.int16, device=dev)
        self.v = torch.empty((Cn, It, hyd.MAX_PIPES), dtype=torch.int16, device=dev)
        self.ptime = torch.empty((Cn, It, hyd.MAX_PIPES), dtype=torch.int64, device=dev)
        self.makespan = torch.empty((It, Cn), dtype=torch.int64, device=dev)
        self.key = torch.empty((It,), dtype=torch.int64, device=dev)
        self.status = torch.zeros((1,), dtype=i32, device=dev)
        self.ws = torch.empty((max(hyd.pack_workspace(It, B, Cn, self.max_np), 1),), dtype=u8, device=dev)
        self.disp_ws = torch.empty((max(hyd.dispatch_workspace(It), 1),), dtype=u8, device=dev)
        self.trials, self.seed = int(trials), int(seed)
        # a3 + a4 in one kernel for small batches (include/hyd.h hyd_dispatch_pack); no stats/members
        small = B <= hyd.SMALL_MAX_BATCH and self.max_np <= 16 and not self.trials
        self.fused = small if fused is None else (bool(fused) and small)
        self.small_ws = torch.zeros((hyd.dispatch_pack_workspace(),), dtype=u8, device=dev)
        if self.trials:
            self.order = torch.empty((It, self.trials, B), dtype=torch.int16, device=dev)
            self.best = torch.empty((Cn, It), dtype=torch.int64, device=dev)
            self.alg1_ws = torch.empty((max(hyd.alg1_workspace(It), 1),), dtype=u8, device=dev)

    # a1-a5; ``len_dev`` int32/uint32-bit tensor [It][B] on the device
    def run(self, len_dev, stream=None):
        It, B, K, kp, Cn = self.n_iter, self.batch, self.n_schemes, self.k_pad, self.n_cand
        if self.ragged:  # NEXT-2: token-budget batches (CSR offsets)
            N = self.n_total
            hyd.cost_table_ragged(len_dev, It, self.off, N, B, self.schemes, K, kp, self.sorted_len, self.perm,
                                  self.cost, self.status, stream)
            if self.fused:
                hyd.dispatch_pack_ragged(self.sorted_len, self.cost, It, self.off, N, B, kp, self.schemes, K,
                                         self.cand, self.cand_np, Cn, self.max_np, self.pipe, self.lb, self.mb, self.v,
                                         self.ptime, self.makespan, self.status, self.small_ws, stream)
                hyd.select_best(self.makespan, It, Cn, self.cand_offset, self.key, self.status, stream)
                return self.key
            hyd.dispatch_ragged(self.sorted_len, self.cost, It, self.off, N, B, kp, self.schemes, K, self.cand,
                                self.cand_np, Cn, self.max_np, self.pipe, self.lb, self.stats, self.members,
                                self.status, self.disp_ws, stream)
            hyd.pack_ragged(self.sorted_len, self.cost, It, self.off, N, B, kp, self.schemes, K, self.cand,
                            self.cand_np, Cn, self.max_np, self.pipe, self.stats, self.members, self.mb, self.v,
                            self.ptime, self.makespan, self.status, self.ws, stream)
            hyd.select_best(self.makespan, It, Cn, self.cand_offset, self.key, self.status, stream)
            return self.key
        hyd.cost_table(len_dev, It, B, self.schemes, K, kp, self.sorted_len, self.perm, self.cost, self.status, stream)
        if self.fused:
            hyd.dispatch_pack(self.sorted_len, self.cost, It, B, kp, self.schemes, K, self.cand, self.cand_np, Cn,
                              self.max_np, self.pipe, self.lb, self.mb, self.v, self.ptime, self.makespan, self.status,
                              self.small_ws, stream)
            hyd.select_best(self.makespan, It, Cn, self.cand_offset, self.key, self.status, stream)
            return self.key
        if self.trials:
            hyd.alg1_permutations(self.seed, It, B, self.trials, self.order, stream)
            hyd.dispatch_alg1(self.sorted_len, self.cost, It, B, kp, self.schemes, K, self.cand, self.cand_np, Cn,
                              self.max_np, self.trials, self.order, self.best, self.pipe, self.lb, self.stats,
                              self.members, self.status, self.alg1_ws, stream)
        else:
            hyd.dispatch(self.sorted_len, self.cost, It, B, kp, self.schemes, K, self.cand, self.cand_np, Cn,
                         self.max_np, self.pipe, self.lb, self.stats, self.members, self.status, self.disp_ws,
                         stream)
        hyd.pack(self.sorted_len, self.cost, It, B, kp, self.schemes, K, self.cand, self.cand_np, Cn, self.max_np,
                 self.pipe, self.stats, self.members, self.mb, self.v, self.ptime, self.makespan, self.status, self.ws,
                 stream)
        hyd.select_best(self.makespan, It, Cn, self.cand_offset, self.key, self.status, stream)
        return self.key

    def eq3_exact(self, len_dev, pair_c, pair_t, node_limit=1 << 24, stream=None):
        """NEXT-4: exact Eq. 3 optimum of the listed (c, t) pairs (include/hyd.h hyd_eq3_exact),
        on this workload's sorted lengths / cost table.  Returns numpy (value, pipe, nodes, proved)."""
        torch = self.torch
        It, B, K, kp, Cn = self.n_iter, self.batch, self.n_schemes, self.k_pad, self.n_cand
        hyd.cost_table(len_dev, It, B, self.schemes, K, kp, self.sorted_len, self.perm, self.cost, self.status, stream)
        pc = torch.as_tensor(np.asarray(pair_c, np.int32), device=self.dev)
        pt = torch.as_tensor(np.asarray(pair_t, np.int32), device=self.dev)
        n = int(pc.numel())
        value = torch.empty((n,), dtype=torch.int64, device=self.dev)
        pipe = torch.empty((n, B), dtype=torch.uint8, device=self.dev)
        nodes = torch.empty((n,), dtype=torch.int64, device=self.dev)
        proved = torch.empty((n,), dtype=torch.uint8, device=self.dev)
        hyd.eq3_exact(self.sorted_len, self.cost, It, B, kp, self.schemes, K, self.cand, self.cand_np, Cn, pc, pt,
                      node_limit, value, pipe, nodes, proved, self.status, stream)
        torch.cuda.synchronize(self.dev)
        return (value.cpu().numpy().view(np.uint64), pipe.cpu().numpy(), nodes.cpu().numpy().view(np.uint64),
                proved.cpu().numpy().astype(bool))

    def eq1_exact(self, pair_c, pair_t, pair_j, node_limit=1 << 24, stream=None):
        """NEXT-4: exact Eq. 1 optimum of the listed pipelines of the LAST run() (its dispatch);
        include/hyd.h hyd_eq1_exact.  Returns numpy (v, obj, nodes, proved)."""
        if self.fused:
            raise hyd.HydError("eq1_exact reads the dispatch's members: build the Assigner with fused=False")
        torch = self.torch
        It, B, K, kp, Cn = self.n_iter, self.batch, self.n_schemes, self.k_pad, self.n_cand
        mk = lambda x: torch.as_tensor(np.asarray(x, np.int32), device=self.dev)
        pc, pt, pj = mk(pair_c), mk(pair_t), mk(pair_j)
        n = int(pc.numel())
        v = torch.empty((n,), dtype=torch.int32, device=self.dev)
        obj = torch.empty((n,), dtype=torch.int64, device=self.dev)
        nodes = torch.empty((n,), dtype=torch.int64, device=self.dev)
        proved = torch.empty((n,), dtype=torch.uint8, device=self.dev)
        hyd.eq1_exact(self.sorted_len, self.cost, It, B, kp, self.schemes, K, self.cand, Cn, self.max_np, self.members,
                      pc, pt, pj, node_limit, v, obj, nodes, proved, self.status, stream)
        torch.cuda.synchronize(self.dev)
        return (v.cpu().numpy().view(np.uint32), obj.cpu().numpy().view(np.uint64),
                nodes.cpu().numpy().view(np.uint64), proved.cpu().numpy().astype(bool))

    def pack_counters(self) -> dict:
        """Work counter written by the last hyd_pack (include/hyd.h: u64 at ws offset 16), or by
        the fused small-batch kernel (u64 at its ws offset 0)."""
        self.torch.cuda.synchronize(self.dev)
        if self.fused:
            return {"bin_evals": int(self.small_ws[0:8].cpu().numpy().view(np.uint64)[0]), "queued_tasks": 0,
                    "handoff": None}
        w = self.ws[0:256].cpu().numpy().view(np.uint64)
        names = ["sumt16", "va16", "bottom16", "cand16", "sumt32", "bottom32", "cand32", "overflow",
                 "clk_records", "clk_phase1", "clk_phase1b", "clk_walk", "clk_phase2", "clk_phase3",
                 "units_phase2", "tasks_lanes16"]
        return {"bin_evals": int(w[2]), "queued_tasks": int(w[0]),
                "handoff": {n: int(x) for n, x in zip(names, w[3:19])}}

    def dispatch_evals(self, lengths) -> int:
        """Sum over feasible (c,t) of sum_i J_i (feasible pipelines per sequence): the
        dispatch's algorithmic evaluation count, from the host tables (no method arithmetic)."""
        rows = [np.sort(np.asarray(r, dtype=np.int64)) for r in lengths]  # ascending per t (ragged ok)
        ml_k = self._ml_k  # MaxLen per scheme
        # cnt[k][t] = #{i : l_i <= MaxLen_k}
        cnt = np.stack([np.array([np.searchsorted(r, m, side="right") for r in rows]) for m in ml_k])
        per = self._mult @ cnt  # [C][It]
        longest = np.array([r[-1] for r in rows])
        feas = longest[None, :] <= self._ml[:, 0][:, None]
        return int(per[feas].sum())

    def status_bits(self) -> int:
        return int(self.status.item()) & 0xFFFFFFFF

    def numpy(self) -> dict:
        """All outputs as numpy arrays with the C ABI's unsigned dtypes."""
        self.torch.cuda.synchronize(self.dev)

        def u(t, dt):
            return t.cpu().numpy().view(dt)

        return dict(
            sorted_len=u(self.sorted_len, np.uint32),
            perm=u(self.perm, np.uint32),
            cost=u(self.cost, np.uint32),
            pipe=u(self.pipe, np.uint8),
            lb=u(self.lb, np.uint64),
            mb=u(self.mb, np.uint16),
            v=u(self.v, np.uint16),
            ptime=u(self.ptime, np.uint64),
            makespan=u(self.makespan, np.uint64),
            key=u(self.key, np.int64),
            status=self.status_bits(),
            **({"best_trial": np.where(u(self.best, np.uint64) == np.uint64(2**64 - 1), -1,
                                       (u(self.best, np.uint64) & np.uint64(0xFF)).astype(np.int64)).astype(np.int32),
                "best_obj": u(self.best, np.uint64) >> np.uint64(8)} if self.trials else {}),
        )


def lengths_to_device(lengths, device=None):
    import torch

    return torch.from_numpy(np.ascontiguousarray(lengths, dtype=np.uint32).view(np.int32)).to(
        device if device is not None else "cuda"
    )


class HostAssigner:
    """End-to-end path on HOST buffers through ``hyd_assign_host`` (the user-facing call).

    Per call: H2D of the lengths (and tables), a1-a5 on the device, and with ``reduce``
    (N > 1 ranks, candidates sharded) the two collectives of include/hyd.h -- allreduce-MIN of
    the keys (a6), then allreduce-SUM of the zero-filled winner rows so every rank holds every
    iteration's plan -- winner gather, D2H of keys + winners' plans in ORIGINAL sequence order,
    one stream synchronisation.  The collectives run ordered on the stream passed to the call.
    """

    def __init__(self, schemes, cand, cand_np, n_iter, batch, k_pad, cand_offset=0, group=None, reduce=False,
                 offsets=None):
        import torch

        self.torch = torch
        self.n_iter, self.batch, self.k_pad = int(n_iter), int(batch), int(k_pad)
        # NEXT-2: ragged batches -- host CSR offsets [It + 1]; ``batch`` is the largest batch
        self.offsets = None if offsets is None else np.ascontiguousarray(offsets, dtype=np.uint32)
        self.n_total = int(self.offsets[-1]) if self.offsets is not None else self.n_iter * self.batch
        self.schemes = np.ascontiguousarray(schemes)
        self.cand = np.ascontiguousarray(cand, dtype=np.uint8)
        self.cand_np = np.ascontiguousarray(cand_np, dtype=np.uint8)
        self.n_cand = int(self.cand.shape[0])
        self.cand_offset = int(cand_offset)
        self.max_np = hyd.check_candidates(self.cand, self.cand_np, self.schemes) if self.n_cand else 1
        if self.offsets is None:
            args = (self.n_iter, self.batch, len(self.schemes), self.k_pad, self.n_cand, self.max_np)
            wsz, koff = hyd.assign_workspace(*args), hyd.assign_key_offset(*args)
        else:
            args = (self.n_iter, self.n_total, self.batch, len(self.schemes), self.k_pad, self.n_cand, self.max_np)
            wsz, koff = hyd.assign_workspace_ragged(*args), hyd.assign_key_offset_ragged(*args)
        self.ws = torch.empty((wsz,), dtype=torch.uint8, device="cuda")
        self.key_view = self.ws[koff : koff + 8 * self.n_iter].view(torch.int64)
        pin = dict(pin_memory=True)
        It, B = self.n_iter, self.batch
        rows = (It, B) if self.offsets is None else (self.n_total,)
        self.key = torch.empty((It,), dtype=torch.int64, **pin)
        self.win_pipe = torch.empty(rows, dtype=torch.uint8, **pin)
        self.win_mb = torch.empty(rows, dtype=torch.int16, **pin)
        self.win_v = torch.empty((It, hyd.MAX_PIPES), dtype=torch.int16, **pin)
        self.win_ptime = torch.empty((It, hyd.MAX_PIPES), dtype=torch.int64, **pin)
        self.status = torch.zeros((1,), dtype=torch.int32, **pin)
        self.group = group
        self._cb = None
        if reduce:
            self._cb = hyd.COLL_FN(self._collective)
        # host copies of the (fixed) tables, pinned
        self._sch = torch.from_numpy(schemes_bytes(self.schemes).copy()).pin_memory()
        self._cand = torch.from_numpy(self.cand.copy()).pin_memory()
        self._cnp = torch.from_numpy(self.cand_np.copy()).pin_memory()
        self._off = (torch.from_numpy(self.offsets.view(np.int32).copy()).pin_memory()
                     if self.offsets is not None else None)

    def _collective(self, ptr, count, op, user, stream):
        """hyd_collective_fn: the buffer is a slice of this assigner's workspace; the collective
        runs ordered on the stream the library passes (include/hyd.h)."""
        torch = self.torch
        try:
            width = 8 if op == hyd.COLL_MIN_I64 else 4
            off, nbytes = int(ptr) - self.ws.data_ptr(), int(count) * width
            if op not in (hyd.COLL_MIN_I64, hyd.COLL_SUM_I32) or off < 0 or off + nbytes > self.ws.numel():
                return 1
            buf = self.ws[off : off + nbytes]
            s = torch.cuda.ExternalStream(int(stream)) if stream else torch.cuda.default_stream(self.ws.device)
            with torch.cuda.stream(s):
                if op == hyd.COLL_MIN_I64:
                    reduce_keys(buf.view(torch.int64), self.group)
                else:
                    share_rows(buf.view(torch.int32), self.group)
            return 0
        except Exception:  # reported as HYD_E_REDUCE
            return 1

    @property
    def h2d_bytes_fixed(self) -> int:
        return self._sch.numel() + self._cand.numel() + self._cnp.numel() + (
            self._off.numel() * 4 if self._off is not None else 0)

    @property
    def d2h_bytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in (self.key, self.win_pipe, self.win_mb, self.win_v,
                                                          self.win_ptime, self.status))

    def __call__(self, len_host, stream=None):
        """``len_host``: pinned int32 torch tensor [It][B] (u32 bit pattern), [N_total] if ragged."""
        It, B = self.n_iter, self.batch
        if self.offsets is not None:
            assert len_host.is_pinned() and tuple(len_host.shape) == (self.n_total,)
            hyd.assign_host_ragged(
                len_host.data_ptr(), It, self._off.data_ptr(), B, self._sch.data_ptr(), len(self.schemes),
                self.k_pad, self._cand.data_ptr(), self._cnp.data_ptr(), self.n_cand, self.cand_offset,
                self.key.data_ptr(), self.win_pipe.data_ptr(), self.win_mb.data_ptr(), self.win_v.data_ptr(),
                self.win_ptime.data_ptr(), self.status.data_ptr(), self._cb, self.ws, stream,
            )
            return self.key
        assert len_host.is_pinned() and tuple(len_host.shape) == (It, B)
        hyd.assign_host(
            len_host.data_ptr(), It, B, self._sch.data_ptr(), len(self.schemes), self.k_pad, self._cand.data_ptr(),
            self._cnp.data_ptr(), self.n_cand, self.cand_offset, self.key.data_ptr(), self.win_pipe.data_ptr(),
            self.win_mb.data_ptr(), self.win_v.data_ptr(), self.win_ptime.data_ptr(), self.status.data_ptr(),
            self._cb, self.ws, stream,
        )
        return self.key


class Proposer:
    """NEXT-3: the strategy-proposal DP (§5) on the device (include/hyd.h hyd_dp_propose).

    ``lengths``: a sample of the dataset's sequence lengths; ``step``/``J``: length grid
    (l = j step, context J step); ``scale``: 1 (integer DP) or 10 (0.1-step relaxation)."""

    def __init__(self, schemes, step, J, n_gpus, scale=10, device=None):
        import torch

        self.torch = torch
        self.dev = torch.device(device if device is not None else "cuda")
        self.schemes_np = np.ascontiguousarray(schemes)
        self.K, self.step, self.J, self.N, self.scale = len(schemes), int(step), int(J), int(n_gpus), int(scale)
        dev, K, J = self.dev, self.K, self.J
        NV = self.N * self.scale
        self.schemes = torch.from_numpy(schemes_bytes(self.schemes_np).copy()).to(dev)
        self.t_num = torch.empty((NV + 1, J + 1), dtype=torch.int64, device=dev)
        self.t_den = torch.empty((NV + 1, J + 1), dtype=torch.int64, device=dev)
        self.choice = torch.empty((NV + 1, J + 1), dtype=torch.int32, device=dev)
        self.counts = torch.empty((J + 1, K), dtype=torch.int16, device=dev)
        self.rows = torch.empty((J + 1, hyd.DP_MAX_ROUND, K), dtype=torch.uint8, device=dev)
        self.valid = torch.empty((J + 1, hyd.DP_MAX_ROUND), dtype=torch.uint8, device=dev)
        self.keep = torch.empty((J + 1, hyd.DP_MAX_ROUND), dtype=torch.uint8, device=dev)
        self.status = torch.zeros((1,), dtype=torch.int32, device=dev)
        self.ws = torch.empty((max(hyd.dp_workspace(K, J), 1),), dtype=torch.uint8, device=dev)

    def run(self, len_dev, stream=None):
        self.status.zero_()
        hyd.dp_propose(len_dev, int(len_dev.numel()), self.schemes, self.K, self.step, self.J, self.N, self.scale,
                       self.t_num, self.t_den, self.choice, self.counts, self.rows, self.valid, self.keep,
                       self.status, self.ws, stream)

    def candidates(self):
        """Proposed subset as per-scheme pipeline counts [M][K] (first-occurrence order) and as
        candidate tables (cand [M][32] u8 in canonical order, cand_np [M] u8), the tables made on
        the device by hyd_dp_candidates."""
        torch = self.torch
        M = (self.J + 1) * hyd.DP_MAX_ROUND
        cand = torch.empty((M, hyd.MAX_PIPES), dtype=torch.uint8, device=self.dev)
        cnp = torch.empty((M,), dtype=torch.uint8, device=self.dev)
        n_out = torch.zeros((1,), dtype=torch.int32, device=self.dev)
        hyd.dp_candidates(self.rows, self.keep, self.J, self.schemes, self.K, cand, cnp, n_out)
        torch.cuda.synchronize(self.dev)
        n = int(n_out.item())
        rows = self.rows.cpu().numpy().reshape(-1, self.K)
        keep = self.keep.cpu().numpy().reshape(-1).astype(bool)
        sel = rows[keep]
        cand, cnp = cand[:n].cpu().numpy(), cnp[:n].cpu().numpy()
        if (cnp == 0).any():
            raise hyd.HydError(f"a proposed candidate has more than {hyd.MAX_PIPES} pipelines")
        return sel, cand, cnp
