"""Seeded synthetic inputs for the Hydraulis two-stage assignment.

This module is the ONLY code shared by the CPU oracle (``oracle/``) and the CUDA
path (``paper_2412_07894_b200/``).  It holds none of the method's arithmetic:
it draws sequence lengths, builds the per-scheme profile (the paper's profiled
inputs: latency coefficients a,b,c of App. C.2, MaxLen of App. C.1
P:1055, UtilLen of App. D) and candidate strategy tables.  The Q32
fixed-point cost evaluation, sorting, dispatch, packing and selection live in
``oracle/`` and in the CUDA kernels, independently.

Input recipe:
  * lengths: numpy ``Generator(PCG64(seed))``; shapes follow SPEC.md's generator
    shapes because the paper's histograms (``fig:distribution``,
    P:124-130) are images absent from PAPER.md:
      cfg1 log-uniform floor(128*32^u) in [128,4096)
      cfg2/cfg4 lognormal(mu=6.9, sigma=1.2) clamped to [1, 32768]  (CommonCrawl-like)
      cfg3 Pareto(alpha=1.1, x_min=256) clamped to [1, 131072]      (GitHub-like)
      cfg5 mix 70% lognormal + 30% Pareto, clamped to [64, 262144]
  * latency model T(l,P)=a l^2 + b l + c (App. C.2), FLOP-based synthesis
    of per-stage forward+backward time in microseconds, frozen to Q32 integers
    ``round_half_even(x_us * 2^32)``; 1 tick = 1 us.
  * MaxLen from the App. C.1 linear memory model, exact rationals.
  * UtilLen (App. D): the smallest l <= MaxLen whose efficiency l/T(l)
    (real-valued profile) reaches 0.85 of the best efficiency on [1, MaxLen].
  * candidates: seeded distinct multisets of D schemes within the GPU budget,
    each in canonical order (MaxLen descending, then scheme index ascending;
    P:623), with candidate 0 a "safety" candidate whose first pipeline can hold
    the longest possible sequence.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

# 48-byte record, identical layout to ``hyd_scheme`` (include/hyd.h) and to the
# oracle's own struct.  A plain data layout, not shared code.
SCHEME_DTYPE = np.dtype(
    [
        ("tp", "<u4"),
        ("pp", "<u4"),
        ("cp", "<u4"),
        ("max_len", "<u4"),
        ("util_len", "<u4"),
        ("_pad", "<u4"),
        ("a_q32", "<u8"),
        ("b_q32", "<u8"),
        ("c_q32", "<u8"),
    ]
)
assert SCHEME_DTYPE.itemsize == 48

MAX_PIPES = 32  # candidate row width (D <= 32)
Q32 = float(2**32)


@dataclass(frozen=True)
class ModelShape:
    name: str
    hidden: int
    layers: int
    vocab: int
    per_layer_params_h2: float  # per-layer parameter count / h^2


@dataclass(frozen=True)
class Hardware:
    name: str
    mem_bytes: int
    margin_bytes: int
    flops_eff: float  # sustained dense bf16 FLOP/s per GPU used in T(l)
    intra_bw: float  # bytes/s per GPU for TP/CP collectives
    inter_bw: float  # bytes/s for PP activation send/recv


LLAMA2_7B = ModelShape("llama2-7b", 4096, 32, 32000, 12.0)
LLAMA2_13B = ModelShape("llama2-13b", 5120, 40, 32000, 12.0)
LLAMA_32B = ModelShape("llama-32b", 6656, 60, 32000, 12.0)
# 70B: GQA with 8 KV heads; attention 2h^2 + 2*h*(h/8); SwiGLU 3*h*28672 = 10.5 h^2
LLAMA_70B = ModelShape("llama-70b", 8192, 80, 32000, 12.75)

# The paper's testbed: A800 80 GB, NVLink 400 GB/s, IB 200 GB/s.
A800 = Hardware("A800-80GB", 80 * 10**9, 8 * 10**9, 0.5 * 312e12, 400e9, 25e9)
# A B200 cluster (this build's target box): 180 GB HBM3e, NVLink 5.
B200 = Hardware("B200-180GB", 180 * 10**9, 10 * 10**9, 0.45 * 2.25e15, 900e9, 50e9)

# App. C.1 constants: A = activation bytes per (token x hidden) per layer with
# TP sequence-parallel (Megatron's 34 sbh, no recompute, flash attention);
# B_const: bytes per parameter entry split by alpha = 3/4 (P:1055 example:
# 32-bit master+Adam states vs 16-bit params+grads).
ACT_A = 34
STATE_B_PER_PARAM = 16  # 12 B fp32 states + 4 B bf16 param/grad
ALPHA = Fraction(3, 4)
EMBED_BYTES = 16  # App. C.1 "x16" read as bytes per entry


def gpus(tp: int, pp: int, cp: int) -> int:
    return tp * pp * cp


def _latency_us(model: ModelShape, hw: Hardware, tp: int, pp: int, cp: int):
    """Real-valued (a, b, c) in microseconds of per-stage fwd+bwd T(l) (App. C.2)."""
    h = model.hidden
    lps = model.layers / pp  # layers per stage
    par = tp * cp
    f = hw.flops_eff
    # causal attention fwd 2*l^2*h, bwd 2x -> 6 l^2 h per layer, split over TP*CP
    a = 6.0 * h * lps / (par * f)
    # dense fwd+bwd 6 * params * l
    dense = 6.0 * model.per_layer_params_h2 * h * h * lps / (par * f)
    # TP: 4 collectives/layer (2 fwd, 2 bwd), ring volume 2(TP-1)/TP x 2h bytes/token
    tp_comm = 0.0 if tp == 1 else 4 * lps * (2.0 * (tp - 1) / tp) * 2 * h / hw.intra_bw / cp
    # CP ring attention: KV pass per layer, half assumed hidden behind compute
    cp_comm = 0.0 if cp == 1 else 0.5 * 3 * lps * ((cp - 1) / cp) * 2 * (h / 8) * 2 / hw.intra_bw / tp
    # PP: activation + gradient of one stage boundary
    pp_comm = 0.0 if pp == 1 else 2 * 2 * h / hw.inter_bw / (tp * cp)
    b = dense + tp_comm + cp_comm + pp_comm
    # constant: launch/sync overhead per stage, 2-5 ms
    c = 2.0e-3 + 0.4e-3 * math.log2(tp) + 0.4e-3 * math.log2(cp) + 0.2e-3 * (pp > 1)
    return a * 1e6, b * 1e6, c * 1e6


def _max_len(model: ModelShape, hw: Hardware, tp: int, pp: int, cp: int, n_cluster: int) -> int:
    """App. C.1: largest l with act(l) + states <= Mem - margin, exact rationals."""
    h, L, V = model.hidden, model.layers, model.vocab
    bc = Fraction(model.per_layer_params_h2) * STATE_B_PER_PARAM
    states = (
        Fraction(L * h * h, n_cluster) * bc * ALPHA
        + Fraction(L, pp) * Fraction(h * h, tp) * bc * (1 - ALPHA)
        + Fraction(h * V, n_cluster) * EMBED_BYTES * ALPHA
        + Fraction(h * V, tp) * EMBED_BYTES * (1 - ALPHA)
    )
    per_token = Fraction(L * h * ACT_A, tp * cp)
    budget = hw.mem_bytes - hw.margin_bytes - states
    if budget <= 0:
        return 0
    return int(budget // per_token)


def _util_len(a: float, b: float, c: float, max_len: int, thresh: float = 0.85) -> int:
    """App. D: smallest l <= MaxLen with eff(l) >= 0.85 * max eff, eff = l/T(l)."""
    if max_len <= 1:
        return max(max_len, 0)
    lstar = math.sqrt(c / a) if a > 0 else float(max_len)
    lstar = min(max(lstar, 1.0), float(max_len))
    eff_max = max(l / (a * l * l + b * l + c) for l in {math.floor(lstar), math.ceil(lstar)} if l >= 1)
    lo, hi = 1, int(min(max_len, math.ceil(lstar)))
    # efficiency is increasing on [1, lstar]: bisect for the first l meeting the threshold
    if hi / (a * hi * hi + b * hi + c) < thresh * eff_max:
        return int(max_len)
    while lo < hi:
        mid = (lo + hi) // 2
        if mid / (a * mid * mid + b * mid + c) >= thresh * eff_max:
            hi = mid
        else:
            lo = mid + 1
    return int(lo)


def _to_q32(x_us: float) -> int:
    v = np.rint(np.float64(x_us) * np.float64(Q32))  # round-half-even
    assert 0 <= v < 2.0**63
    return int(v)


def scheme_table(model, hw, shapes, n_cluster, max_len_override=None):
    """Profile table for schemes ``shapes`` = [(tp, pp, cp), ...]."""
    out = np.zeros(len(shapes), dtype=SCHEME_DTYPE)
    for k, (tp, pp, cp) in enumerate(shapes):
        a, b, c = _latency_us(model, hw, tp, pp, cp)
        ml = max_len_override if max_len_override is not None else _max_len(model, hw, tp, pp, cp, n_cluster)
        ml = int(min(ml, 2**24))
        out[k]["tp"], out[k]["pp"], out[k]["cp"] = tp, pp, cp
        out[k]["max_len"] = ml
        out[k]["util_len"] = _util_len(a, b, c, ml) if ml > 0 else 0
        out[k]["a_q32"], out[k]["b_q32"], out[k]["c_q32"] = _to_q32(a), _to_q32(b), _to_q32(c)
    return out


# ----------------------------------------------------------------------------- lengths
def lengths_loguniform(rng, n, lo=128, ratio=32):
    u = rng.random(n)
    return np.floor(lo * np.power(float(ratio), u)).astype(np.uint32)


def lengths_lognormal(rng, n, mu=6.9, sigma=1.2, lo=1, hi=32768):
    x = np.floor(rng.lognormal(mu, sigma, n))
    return np.clip(x, lo, hi).astype(np.uint32)


def sample_minibatches(rng, corpus, n_iter, token_budget, context):
    """Token-budget mini-batches: per iteration, draw lengths
    uniformly with replacement from ``corpus``, truncate each draw to ``context`` (the budget counts
    truncated tokens), stop at the first draw that brings the total to >= ``token_budget``.
    Returns (lengths u32 [N_total], offsets u32 [n_iter + 1])."""
    corpus = np.asarray(corpus, dtype=np.int64)
    out, offs, tot = [], [0], 0
    for _ in range(n_iter):
        got, acc = [], 0
        while acc < token_budget:
            x = min(int(corpus[int(rng.integers(0, corpus.size))]), context)
            got.append(x)
            acc += x
        out.extend(got)
        tot += len(got)
        offs.append(tot)
    return np.asarray(out, dtype=np.uint32), np.asarray(offs, dtype=np.uint32)


def lengths_pareto(rng, n, alpha=1.1, xmin=256, lo=1, hi=131072):
    x = np.floor(xmin * (1.0 + rng.pareto(alpha, n)))
    return np.clip(x, lo, hi).astype(np.uint32)


def lengths_mix(rng, n, p_pareto=0.3, lo=64, hi=262144):
    pick = rng.random(n) < p_pareto
    a = np.floor(rng.lognormal(6.9, 1.2, n))
    b = np.floor(256 * (1.0 + rng.pareto(1.1, n)))
    return np.clip(np.where(pick, b, a), lo, hi).astype(np.uint32)


# ----------------------------------------------------------------------------- candidates
def canonical(schemes, ks):
    """Order a pipeline list by (MaxLen desc, scheme index asc) -- P:623 ordering."""
    return sorted(ks, key=lambda k: (-int(schemes[k]["max_len"]), k))


def candidate_table(rng, schemes, n_cand, n_pipes, gpu_budget, safety, cover_len=None, p_cover=0.85):
    """Distinct multisets of ``n_pipes`` schemes with sum(GPUs) <= budget, canonical order.

    A fraction ``p_cover`` of the candidates can hold the context length ``cover_len``
    (their longest-MaxLen pipeline reaches it); the rest are "short-context" strategies,
    as the strategy proposal keeps optimal strategies for every length ceiling L <= L_max
    (§7 Problem 1).  Small spaces are enumerated and sampled without
    replacement; large ones are drawn pipeline by pipeline within the GPU budget.
    """
    import itertools

    K = len(schemes)
    g = [gpus(int(s["tp"]), int(s["pp"]), int(s["cp"])) for s in schemes]
    ml = [int(s["max_len"]) for s in schemes]
    gmin = min(g)
    cover_len = cover_len if cover_len is not None else 0
    seen = set()
    rows = []
    if safety is not None:
        row = tuple(canonical(schemes, safety))
        assert sum(g[k] for k in row) <= gpu_budget
        seen.add(tuple(sorted(row)))
        rows.append(row)
    need = n_cand - len(rows)
    if math.comb(K + n_pipes - 1, n_pipes) <= 2_000_000:
        pool = [
            m
            for m in itertools.combinations_with_replacement(range(K), n_pipes)
            if sum(g[k] for k in m) <= gpu_budget and m not in seen
        ]
        assert len(pool) >= need, f"only {len(pool)} distinct candidates for {need}"
        cov = [m for m in pool if max(ml[k] for k in m) >= cover_len]
        non = [m for m in pool if max(ml[k] for k in m) < cover_len]
        n_cov = min(len(cov), max(need - len(non), int(round(p_cover * need))))
        picks = [cov[i] for i in rng.permutation(len(cov))[:n_cov]]
        picks += [non[i] for i in rng.permutation(len(non))[: need - n_cov]]
        picks = [picks[i] for i in rng.permutation(len(picks))]
        rows += [tuple(canonical(schemes, list(m))) for m in picks]
    else:
        tries = 0
        while len(rows) < n_cand:
            tries += 1
            assert tries < 100 * n_cand + 100000, "candidate space too small"
            cover = rng.random() < p_cover
            ks, left = [], gpu_budget
            for r in range(n_pipes):
                room = left - gmin * (n_pipes - r - 1)
                ok = [k for k in range(K) if g[k] <= room and (r > 0 or not cover or ml[k] >= cover_len)]
                k = ok[int(rng.integers(0, len(ok)))]
                ks.append(k)
                left -= g[k]
            key = tuple(sorted(ks))
            if key in seen:
                continue
            seen.add(key)
            rows.append(tuple(canonical(schemes, ks)))
    cand = np.full((n_cand, MAX_PIPES), 0xFF, dtype=np.uint8)
    cand_np = np.zeros(n_cand, dtype=np.uint8)
    for c, row in enumerate(rows[:n_cand]):
        cand[c, : len(row)] = row
        cand_np[c] = len(row)
    return cand, cand_np


# ----------------------------------------------------------------------------- configs
@dataclass
class Workload:
    cfg: int
    name: str
    lengths: np.ndarray  # u32 [It][B], or [N_total] for ragged batches
    schemes: np.ndarray  # SCHEME_DTYPE [K]
    cand: np.ndarray  # u8 [C][32]
    cand_np: np.ndarray  # u8 [C]
    k_pad: int
    meta: dict = field(default_factory=dict)
    offsets: np.ndarray | None = None  # NEXT-2: u32 CSR [It + 1] of ragged (token-budget) batches

    @property
    def ragged(self):
        return self.offsets is not None

    @property
    def n_iter(self):
        return int(self.offsets.size - 1) if self.ragged else int(self.lengths.shape[0])

    @property
    def batch(self):
        """Sequences per iteration (the largest one for ragged batches)."""
        return int(np.diff(self.offsets.astype(np.int64)).max()) if self.ragged else int(self.lengths.shape[1])

    @property
    def n_total(self):
        return int(self.offsets[-1]) if self.ragged else self.n_iter * self.batch

    def iteration(self, t):
        """Lengths of iteration t (a view)."""
        return self.lengths[self.offsets[t]:self.offsets[t + 1]] if self.ragged else self.lengths[t]

    @property
    def n_cand(self):
        return int(self.cand.shape[0])

    @property
    def n_schemes(self):
        return int(self.schemes.shape[0])


# (B, D, C, It, gpu budget) per BASELINE.json configs; "(ours)" choices per SURVEY §8(d)
CONFIGS = {
    1: dict(name="cfg1-16seq-2homo-1cand", B=16, D=2, C=1, It=4096, budget=8, seed=101),
    2: dict(name="cfg2-cc32k-256seq-4pipe-64cand", B=256, D=4, C=64, It=1024, budget=32, seed=202),
    3: dict(name="cfg3-gh128k-512seq-8pipe-1024cand", B=512, D=8, C=1024, It=256, budget=64, seed=303),
    4: dict(name="cfg4-70b-512seq-8pipe-4096cand", B=512, D=8, C=4096, It=1024, budget=64, seed=404),
    5: dict(name="cfg5-stress-8192seq-16pipe-16384cand", B=8192, D=16, C=16384, It=16, budget=256, seed=505),
    # NEXT-2: the paper's workload shape -- 100K-token mini-batches, 32K context, ragged B
    6: dict(name="cfg6-70b-100ktok-32kctx-8pipe-4096cand", B=None, D=8, C=4096, It=1024, budget=64, seed=606,
            tokens=100_000, context=32768),
}

_SHAPES = {
    2: [(2, 1, 1), (4, 1, 1), (8, 1, 1), (16, 1, 1), (4, 2, 1), (8, 2, 1), (8, 1, 2)],
    3: [
        (2, 1, 1), (2, 2, 1), (2, 4, 1), (4, 1, 1), (4, 2, 1), (4, 4, 1), (8, 1, 1), (8, 2, 1),
        (8, 1, 2), (4, 1, 2), (8, 1, 4), (4, 2, 2),
    ],
    4: [
        (2, 2, 1), (2, 4, 1), (4, 1, 1), (4, 2, 1), (4, 4, 1), (8, 1, 1), (8, 2, 1), (8, 4, 1),
        (8, 1, 2), (4, 1, 2), (8, 2, 2), (4, 2, 2), (8, 1, 4), (2, 8, 1),
    ],
    5: [
        (2, 2, 1), (2, 4, 1), (4, 1, 1), (8, 1, 1), (4, 2, 1), (8, 2, 1), (8, 1, 2), (4, 1, 2),
        (8, 1, 4), (4, 1, 4), (8, 1, 8), (4, 2, 2), (8, 2, 2), (8, 2, 4), (4, 4, 1), (8, 4, 1),
        (2, 8, 1), (4, 2, 4), (8, 4, 2), (4, 4, 2),
    ],
}


def _kpad(K):
    return max(4, (K + 3) // 4 * 4)


def make_workload(cfg: int, n_cand: int | None = None, n_iter: int | None = None) -> Workload:
    """Config ``cfg`` (1-5).  ``n_cand``/``n_iter`` take a prefix (parity-test sizes)."""
    p = CONFIGS[cfg]
    if cfg == 6:
        return _make_ragged_workload(cfg, n_cand, n_iter)
    B, D, C, It = p["B"], p["D"], p["C"], p["It"]
    C = C if n_cand is None else n_cand
    It = It if n_iter is None else n_iter
    rng_len = np.random.Generator(np.random.PCG64(p["seed"]))
    rng_cand = np.random.Generator(np.random.PCG64(p["seed"] + 1))
    full_it = CONFIGS[cfg]["It"] if n_iter is None else max(n_iter, 1)
    if cfg == 1:
        lens = lengths_loguniform(rng_len, full_it * B)
        schemes = scheme_table(LLAMA2_7B, A800, [(2, 2, 1)], 8, max_len_override=8192)
        cand, cand_np = candidate_table(rng_cand, schemes, C, D, p["budget"], safety=[0, 0])
        hw, model, maxlen_cap = A800, LLAMA2_7B, 4096
    elif cfg == 2:
        lens = lengths_lognormal(rng_len, full_it * B, hi=32768)
        schemes = scheme_table(LLAMA2_13B, A800, _SHAPES[2], p["budget"])
        hw, model, maxlen_cap = A800, LLAMA2_13B, 32768
    elif cfg == 3:
        lens = lengths_pareto(rng_len, full_it * B, hi=131072)
        schemes = scheme_table(LLAMA_32B, B200, _SHAPES[3], p["budget"])
        hw, model, maxlen_cap = B200, LLAMA_32B, 131072
    elif cfg == 4:
        lens = lengths_lognormal(rng_len, full_it * B, hi=32768)
        schemes = scheme_table(LLAMA_70B, B200, _SHAPES[4], p["budget"])
        hw, model, maxlen_cap = B200, LLAMA_70B, 32768
    elif cfg == 5:
        lens = lengths_mix(rng_len, full_it * B)
        schemes = scheme_table(LLAMA_70B, B200, _SHAPES[5], p["budget"])
        hw, model, maxlen_cap = B200, LLAMA_70B, 262144
    else:
        raise ValueError(cfg)
    if cfg != 1:
        g = [gpus(int(s["tp"]), int(s["pp"]), int(s["cp"])) for s in schemes]
        ml = schemes["max_len"].astype(np.int64)
        longest = [k for k in range(len(schemes)) if ml[k] >= maxlen_cap]
        assert longest, f"cfg{cfg}: no scheme holds {maxlen_cap} tokens"
        k_long = min(longest, key=lambda k: (g[k], k))
        k_small = min(range(len(schemes)), key=lambda k: (g[k], -ml[k], k))
        safety = [k_long] + [k_small] * (D - 1)
        cand, cand_np = candidate_table(rng_cand, schemes, C, D, p["budget"], safety=safety, cover_len=maxlen_cap)
    lens = lens.reshape(full_it, B)[:It].copy()
    return Workload(
        cfg=cfg,
        name=p["name"],
        lengths=np.ascontiguousarray(lens, dtype=np.uint32),
        schemes=schemes,
        cand=cand,
        cand_np=cand_np,
        k_pad=_kpad(len(schemes)),
        meta=dict(model=model.name, hw=hw.name, gpu_budget=p["budget"], seed=p["seed"], D=D),
    )


def _make_ragged_workload(cfg, n_cand, n_iter):
    """Config 6 (NEXT-2): config 4's model, hardware, schemes and candidate recipe with
    token-budget batches drawn from a CommonCrawl-like corpus (lognormal mu 6.9, sigma 1.2)."""
    p = CONFIGS[cfg]
    D, C, It = p["D"], p["C"], p["It"]
    C = C if n_cand is None else n_cand
    It = It if n_iter is None else n_iter
    rng_len = np.random.Generator(np.random.PCG64(p["seed"]))
    rng_cand = np.random.Generator(np.random.PCG64(p["seed"] + 1))
    corpus = np.maximum(np.floor(rng_len.lognormal(6.9, 1.2, 1_000_000)), 1).astype(np.int64)
    lens, offs = sample_minibatches(rng_len, corpus, It, p["tokens"], p["context"])
    schemes = scheme_table(LLAMA_70B, B200, _SHAPES[4], p["budget"])
    maxlen_cap = p["context"]
    g = [gpus(int(s["tp"]), int(s["pp"]), int(s["cp"])) for s in schemes]
    ml = schemes["max_len"].astype(np.int64)
    longest = [k for k in range(len(schemes)) if ml[k] >= maxlen_cap]
    k_long = min(longest, key=lambda k: (g[k], k))
    k_small = min(range(len(schemes)), key=lambda k: (g[k], -ml[k], k))
    safety = [k_long] + [k_small] * (D - 1)
    cand, cand_np = candidate_table(rng_cand, schemes, C, D, p["budget"], safety=safety, cover_len=maxlen_cap)
    return Workload(
        cfg=cfg,
        name=p["name"],
        lengths=lens,
        schemes=schemes,
        cand=cand,
        cand_np=cand_np,
        k_pad=_kpad(len(schemes)),
        meta=dict(model=LLAMA_70B.name, hw=B200.name, gpu_budget=p["budget"], seed=p["seed"], D=D,
                  tokens_per_iteration=p["tokens"], context=p["context"]),
        offsets=offs,
    )


def custom_workload(lengths, schemes, cand_rows, k_pad=None, cfg=0, name="custom"):
    """Build a Workload from explicit arrays (tests).  ``cand_rows``: list of scheme-index lists."""
    lengths = np.ascontiguousarray(np.asarray(lengths, dtype=np.uint32))
    if lengths.ndim == 1:
        lengths = lengths[None, :]
    C = len(cand_rows)
    cand = np.full((C, MAX_PIPES), 0xFF, dtype=np.uint8)
    cand_np = np.zeros(C, dtype=np.uint8)
    for c, row in enumerate(cand_rows):
        cand[c, : len(row)] = row
        cand_np[c] = len(row)
    return Workload(cfg, name, lengths, schemes, cand, cand_np, k_pad or _kpad(len(schemes)))


def make_scheme(tp=1, pp=1, cp=1, max_len=8192, util_len=0, a_q32=0, b_q32=0, c_q32=0):
    s = np.zeros(1, dtype=SCHEME_DTYPE)
    s["tp"], s["pp"], s["cp"], s["max_len"], s["util_len"] = tp, pp, cp, max_len, util_len
    s["a_q32"], s["b_q32"], s["c_q32"] = a_q32, b_q32, c_q32
    return s


def random_small_instance(rng, B, D, K=3, max_pp=3, lmax=64):
    """Tiny heterogeneous instance for brute-force tests (integer coefficients)."""
    sch = np.zeros(K, dtype=SCHEME_DTYPE)
    for k in range(K):
        sch[k]["tp"] = 1
        sch[k]["pp"] = int(rng.integers(1, max_pp + 1))
        sch[k]["cp"] = 1
        sch[k]["max_len"] = int(rng.integers(lmax, 3 * lmax))
        sch[k]["util_len"] = int(rng.integers(0, lmax)) if rng.random() < 0.5 else 0
        sch[k]["a_q32"] = int(rng.integers(0, 4)) << 26  # a in [0, 3/64]
        sch[k]["b_q32"] = int(rng.integers(1, 5)) << 32
        sch[k]["c_q32"] = int(rng.integers(0, 20)) << 32
    ks = canonical(sch, [int(k) for k in rng.integers(0, K, D)])
    lens = rng.integers(1, lmax + 1, B).astype(np.uint32)
    ml0 = int(sch[ks[0]]["max_len"])
    lens = np.minimum(lens, ml0).astype(np.uint32)
    return custom_workload(lens, sch, [ks])


def load_config(path: str) -> Workload:
    """A configuration from its JSON (configs/cfgN.json, tools/export_configs.py): the scheme and
    candidate tables as stored; the lengths regenerated from the config's seeded generator and
    checked against the stored SHA-256."""
    import hashlib
    import json

    d = json.load(open(path))
    W = make_workload(int(d["config"]))
    lens = np.ascontiguousarray(W.lengths, np.uint32)
    if hashlib.sha256(lens.tobytes()).hexdigest() != d["lengths"]["sha256_lengths"]:
        raise ValueError(f"{path}: the regenerated lengths do not match the stored hash")
    sch = np.zeros(len(d["schemes"]), dtype=SCHEME_DTYPE)
    for i, s in enumerate(d["schemes"]):
        for k, v in s.items():
            sch[i][k] = v
    cand = np.full((len(d["candidates"]), 32), 0xFF, np.uint8)
    cnp = np.zeros(len(d["candidates"]), np.uint8)
    for c, row in enumerate(d["candidates"]):
        cand[c, : len(row)] = row
        cnp[c] = len(row)
    return Workload(W.cfg, d["workload"], lens, sch, cand, cnp, int(d["k_pad"]), meta=dict(d["meta"]),
                    offsets=W.offsets)
