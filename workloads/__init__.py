"""Seeded synthetic inputs for the five SAGA-NN layer configurations.

This module is shared by BOTH sides of every parity check (the CUDA path in
``paper_2009_00804_b200`` and the CPU oracle in ``oracle/``).  It therefore
holds NONE of the method's arithmetic: it only draws graphs, features and
weights.  Everything is produced by a counter-based generator (a splitmix64
finaliser over (stream key, counter)) written in plain int64 torch ops, so the
integer draws (graph topology, edge types, permutations) are bit-identical on
CPU and CUDA; float draws go through the same integer stream and are then
mapped with log/cos (Box-Muller), which may differ by one ulp between devices
before the bf16 rounding -- both sides always consume the same materialised
tensors, so this never affects a parity check.

Configurations follow BASELINE.json lines 7-11 (``configs``) with the readings
A2-A5, A10, A17 listed in DESIGN.md section "Readings".
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch

SEED_ROOT = 200900804  # arXiv id, SURVEY.md 8(d) "Seeds"

# ---------------------------------------------------------------- configs ----


@dataclass(frozen=True)
class Config:
    name: str
    model: str              # "gcn" | "sage" | "gat" | "gated" | "rgcn" | "sage_lstm" | "ggnn"
    graph: str              # "er" | "rmat"
    n: int                  # vertices
    m: int                  # generated edges (before appended self-loops)
    self_loops: bool
    dedup: bool             # distinct (src, dst) pairs (C1 ER, C2)
    dtype: str              # "f32" | "bf16"  (storage dtype of features/weights)
    dims: tuple             # feature widths, e.g. (64, 16) or (128, 128, 64)
    heads: int = 1
    num_etypes: int = 1
    rmat: tuple = (0.57, 0.19, 0.19, 0.05)
    index: int = 0
    extra: dict = field(default_factory=dict)

    @property
    def num_edges(self) -> int:
        return self.m + (self.n if self.self_loops else 0)

    @property
    def f_canon(self) -> int:
        """Row width Gather reduces in SAGA order (reading A20)."""
        return {"gcn": self.dims[0], "sage": self.dims[0], "gat": self.dims[-1],
                "gated": self.dims[0], "rgcn": self.dims[0], "sage_lstm": self.dims[0],
                "ggnn": self.dims[0]}[self.model]

    def updates_per_layer(self) -> int:
        """Edge-feature updates of one layer = E * F_canon (reading A20).

        For the 2-layer SAGE config every layer gathers a dims[layer]-wide row;
        this is the per-layer figure of the first layer; see layer_updates().
        """
        return self.num_edges * self.f_canon

    def layer_updates(self) -> int:
        """Edge-feature updates of the whole configured step (all layers)."""
        if self.model == "sage":
            return sum(self.num_edges * d for d in self.dims[:-1])
        return self.updates_per_layer()


CONFIGS = {
    # BJ:7  GCN fp32, ER N=2048, 10,240 edges + self-loops, 64 -> 16
    "C1": Config("C1", "gcn", "er", 2048, 10240, True, True, "f32", (64, 16), index=1),
    # BJ:8  SAGE-mean x2, R-MAT 2^16, 2^20 distinct edges, 128 -> 128 -> 64 (bf16)
    "C2": Config("C2", "sage", "rmat", 1 << 16, 1 << 20, False, True, "bf16", (128, 128, 64), index=2),
    # BJ:9  GAT 8 heads x 8, R-MAT 2^18, avg in-degree 16 + self-loops, 256 -> 64 (bf16)
    "C3": Config("C3", "gat", "rmat", 1 << 18, 1 << 22, True, False, "bf16", (256, 64), heads=8, index=3),
    # BJ:10 gated, 4 edge types, R-MAT 2^17, 2^21 edges, hidden 128 fp32
    "C4": Config("C4", "gated", "rmat", 1 << 17, 1 << 21, False, False, "f32", (128, 128), num_etypes=4, index=4),
    # BJ:11 GCN at scale, R-MAT 2^22, 2^26 edges + self-loops, 256 -> 256 (bf16)
    "C5": Config("C5", "gcn", "rmat", 1 << 22, 1 << 26, True, False, "bf16", (256, 256), index=5),
    # SURVEY 8(f) NEXT-3 (not a BASELINE config): R-GCN, C4's graph shape and widths,
    # 4 relation types, fp32, per-type mean + self connection + bias, ReLU
    "C6": Config("C6", "rgcn", "rmat", 1 << 17, 1 << 21, False, False, "f32", (128, 128), num_etypes=4, index=6),
    # SURVEY 8(f) NEXT-2 (not a BASELINE config): GraphSAGE-LSTM on C2's graph recipe,
    # bf16 128 -> 128, LSTM hidden 128, ReLU
    "C7": Config("C7", "sage_lstm", "rmat", 1 << 16, 1 << 20, False, True, "bf16", (128, 128), index=7),
    # SURVEY 8(f) NEXT-4 (not a BASELINE config): paper-form GGNN (edge MLP on
    # [h_src || h_dst] + ReLU, sum gather, GRU) on C4's graph shape, fp32 128
    "C8": Config("C8", "ggnn", "rmat", 1 << 17, 1 << 21, False, False, "f32", (128, 128), index=8,
                 extra={"agg": "sum"}),
}


def scaled(cfg: Config, n: int, m: int, name: str | None = None) -> Config:
    """Same model/dtype/dims/recipe on a smaller graph (parity-test sizes)."""
    return Config(name or f"{cfg.name}s", cfg.model, cfg.graph, n, m, cfg.self_loops, cfg.dedup,
                  cfg.dtype, cfg.dims, cfg.heads, cfg.num_etypes, cfg.rmat, cfg.index, dict(cfg.extra))


# ------------------------------------------------- counter-based generator ----

_M64 = (1 << 64) - 1


def _s64(x: int) -> int:
    """Reinterpret an unsigned 64-bit constant as torch int64."""
    x &= _M64
    return x - (1 << 64) if x >= (1 << 63) else x


_GOLDEN = _s64(0x9E3779B97F4A7C15)
_C1 = _s64(0xBF58476D1CE4E5B9)
_C2 = _s64(0x94D049BB133111EB)


def _lsr(x: torch.Tensor, s: int) -> torch.Tensor:
    """Logical right shift of an int64 tensor (torch's >> is arithmetic)."""
    return (x >> s) & ((1 << (64 - s)) - 1)


def mix64(x: torch.Tensor) -> torch.Tensor:
    """splitmix64 finaliser on int64 tensors (wrapping arithmetic)."""
    z = x + _GOLDEN
    z = (z ^ _lsr(z, 30)) * _C1
    z = (z ^ _lsr(z, 27)) * _C2
    return z ^ _lsr(z, 31)


def stream_key(cfg_index: int, stream: str) -> int:
    h = 1469598103934665603
    for ch in f"{SEED_ROOT}/{cfg_index}/{stream}":
        h = ((h ^ ord(ch)) * 1099511628211) & _M64
    return _s64(h)


def draw_u64(key: int, counter: torch.Tensor) -> torch.Tensor:
    """64 random bits per counter (int64 tensor)."""
    return mix64(mix64(counter ^ key) + key)


def draw_bits(key: int, counter: torch.Tensor, bits: int) -> torch.Tensor:
    """Top `bits` bits of the draw as a non-negative int64 (bits <= 62)."""
    return _lsr(draw_u64(key, counter), 64 - bits)


def draw_uniform(key: int, counter: torch.Tensor) -> torch.Tensor:
    """float64 uniform in [0, 1) with 53 random bits."""
    return draw_bits(key, counter, 53).to(torch.float64) * (1.0 / (1 << 53))


def draw_normal(key: int, counter: torch.Tensor) -> torch.Tensor:
    """float64 N(0,1) via Box-Muller on two sub-streams."""
    u1 = 1.0 - draw_uniform(key, counter * 2)         # (0, 1]
    u2 = draw_uniform(key, counter * 2 + 1)
    return torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(2.0 * math.pi * u2)


def _arange(a: int, b: int, device) -> torch.Tensor:
    return torch.arange(a, b, dtype=torch.int64, device=device)


# ------------------------------------------------------------------ graphs ----


def _rmat_edges(key: int, scale: int, lo: int, hi: int, abcd, device):
    """R-MAT (Graph500 style, no noise) edges for counters [lo, hi)."""
    a, b, c, _ = abcd
    t1 = int(round(a * (1 << 24)))
    t2 = int(round((a + b) * (1 << 24)))
    t3 = int(round((a + b + c) * (1 << 24)))
    e = _arange(lo, hi, device)
    src = torch.zeros_like(e)
    dst = torch.zeros_like(e)
    for lvl in range(scale):
        r = draw_bits(key, e * scale + lvl, 24)
        bit = 1 << (scale - 1 - lvl)
        src_bit = r >= t2                      # quadrants c, d
        dst_bit = ((r >= t1) & (r < t2)) | (r >= t3)  # quadrants b, d
        src += src_bit.to(torch.int64) * bit
        dst += dst_bit.to(torch.int64) * bit
    return src, dst


def _er_edges(key: int, n: int, lo: int, hi: int, device):
    e = _arange(lo, hi, device)
    bits = max(1, (n - 1).bit_length())
    r = draw_u64(key, e)
    if n & (n - 1) == 0:
        src = _lsr(r, 64 - bits)
        dst = _lsr(r, 64 - 2 * bits) & (n - 1)
    else:
        src = _lsr(r, 33) % n
        dst = (r & 0x7FFFFFFF) % n
    return src, dst


def _first_occurrence_unique(key64: torch.Tensor) -> torch.Tensor:
    """Mask keeping the first occurrence of every key (order preserved)."""
    uniq, inv = torch.unique(key64, return_inverse=True)
    first = torch.full((uniq.numel(),), key64.numel(), dtype=torch.int64, device=key64.device)
    first.scatter_reduce_(0, inv, torch.arange(key64.numel(), device=key64.device), reduce="amin")
    mask = torch.zeros(key64.numel(), dtype=torch.bool, device=key64.device)
    mask[first] = True
    return mask


def make_graph(cfg: Config, device="cpu"):
    """COO (src, dst, etype) int32 for `cfg` (readings A2-A5).

    Generated edges: self-loops dropped, duplicates dropped only if cfg.dedup,
    topped up from the same counter stream until exactly cfg.m remain; then a
    seeded vertex permutation; then N self-loops (v, v) appended in vertex
    order if cfg.self_loops.  etype ~ U{0..T-1} per edge (C4).
    """
    key = stream_key(cfg.index, f"graph/{cfg.n}/{cfg.m}")
    n, m = cfg.n, cfg.m
    srcs, dsts = [], []
    have = 0
    lo = 0
    seen = None
    while have < m:
        want = (m - have)
        hi = lo + int(want * 1.15) + 64
        if cfg.graph == "rmat":
            s, d = _rmat_edges(key, int(math.log2(n)), lo, hi, cfg.rmat, device)
        else:
            s, d = _er_edges(key, n, lo, hi, device)
        lo = hi
        keep = s != d
        s, d = s[keep], d[keep]
        if cfg.dedup:
            k64 = s * n + d
            allk = k64 if seen is None else torch.cat([seen, k64])
            mask = _first_occurrence_unique(allk)
            mask = mask[0 if seen is None else seen.numel():]
            s, d = s[mask], d[mask]
            k64 = k64[mask]
        take = min(m - have, s.numel())
        s, d = s[:take], d[:take]
        if cfg.dedup:
            k64 = k64[:take]
            seen = k64 if seen is None else torch.cat([seen, k64])
        srcs.append(s)
        dsts.append(d)
        have += take
    src = torch.cat(srcs) if srcs else torch.zeros(0, dtype=torch.int64, device=device)
    dst = torch.cat(dsts) if dsts else torch.zeros(0, dtype=torch.int64, device=device)
    if cfg.graph == "rmat":
        pkey = stream_key(cfg.index, f"perm/{n}")
        order = torch.argsort(draw_u64(pkey, _arange(0, n, device)))
        perm = torch.empty_like(order)
        perm[order] = _arange(0, n, device)
        src, dst = perm[src], perm[dst]
    if cfg.self_loops:
        v = _arange(0, n, device)
        src = torch.cat([src, v])
        dst = torch.cat([dst, v])
    etype = None
    if cfg.num_etypes > 1:
        tkey = stream_key(cfg.index, f"etype/{n}/{m}")
        etype = (draw_bits(tkey, _arange(0, src.numel(), device), 32) % cfg.num_etypes).to(torch.int32)
    return src.to(torch.int32), dst.to(torch.int32), etype


# ------------------------------------------------------- features/weights ----


def _chunked(fn, key, rows, cols, device, chunk_rows=1 << 16, out_dtype=torch.float32):
    out = torch.empty(rows, cols, dtype=out_dtype, device=device)
    for r0 in range(0, rows, chunk_rows):
        r1 = min(rows, r0 + chunk_rows)
        ctr = _arange(r0 * cols, r1 * cols, device)
        out[r0:r1] = fn(key, ctr).view(r1 - r0, cols).to(out_dtype)
    return out


def uniform(cfg_index: int, name: str, rows: int, cols: int, bound: float, device="cpu"):
    key = stream_key(cfg_index, name)
    return _chunked(lambda k, c: (draw_uniform(k, c) * 2.0 - 1.0) * bound, key, rows, cols, device)


def normal(cfg_index: int, name: str, rows: int, cols: int, std: float = 1.0, device="cpu"):
    key = stream_key(cfg_index, name)
    return _chunked(lambda k, c: draw_normal(k, c) * std, key, rows, cols, device)


def glorot(cfg_index: int, name: str, fan_in: int, fan_out: int, device="cpu"):
    return uniform(cfg_index, name, fan_in, fan_out, math.sqrt(6.0 / (fan_in + fan_out)), device)


def _store(t: torch.Tensor, dtype: str) -> torch.Tensor:
    """Round an fp32 draw to the storage dtype (RNE for bf16, reading A17)."""
    return t.to(torch.bfloat16) if dtype == "bf16" else t.contiguous()


def make_inputs(cfg: Config, device="cpu", graph=True):
    """All inputs of one configured step: graph + features + weights.

    Returns a dict; weights are stored [in][out] row-major (reading A8).
    """
    k = cfg.index
    d = {"cfg": cfg}
    if graph:
        d["src"], d["dst"], d["etype"] = make_graph(cfg, device)
    n = cfg.n
    if cfg.model == "gcn":
        fi, fo = cfg.dims
        if cfg.dtype == "f32":
            x = uniform(k, f"X/{n}", n, fi, 1.0, device)          # BJ:7 U[-1,1]
        else:
            x = normal(k, f"X/{n}", n, fi, 1.0, device)           # BJ:11 N(0,1)
        d["X"] = _store(x, cfg.dtype)
        d["W"] = _store(glorot(k, "W", fi, fo, device), cfg.dtype)
        d["b"] = torch.zeros(fo, dtype=torch.float32, device=device)   # BJ:7 bias zero
    elif cfg.model == "sage":
        f0, f1, f2 = cfg.dims
        d["X"] = _store(normal(k, f"X/{n}", n, f0, 1.0, device), cfg.dtype)
        d["W1"] = _store(glorot(k, "W1", 2 * f0, f1, device), cfg.dtype)   # [self; neigh] x out
        d["W2"] = _store(glorot(k, "W2", 2 * f1, f2, device), cfg.dtype)
    elif cfg.model == "gat":
        fi, fo = cfg.dims
        hd = fo // cfg.heads
        d["X"] = _store(normal(k, f"X/{n}", n, fi, 1.0, device), cfg.dtype)
        d["W"] = _store(glorot(k, "W", fi, fo, device), cfg.dtype)
        d["a_src"] = normal(k, "a_src", cfg.heads, hd, 0.1, device)          # fp32
        d["a_dst"] = normal(k, "a_dst", cfg.heads, hd, 0.1, device)
    elif cfg.model == "gated":
        f, hdim = cfg.dims
        T = cfg.num_etypes
        bnd = 1.0 / math.sqrt(hdim)
        d["H"] = normal(k, f"H/{n}", n, f, 1.0, device)
        d["W_type"] = uniform(k, "W_type", T * f, f, bnd, device).view(T, f, f)
        d["W_ih"] = uniform(k, "W_ih", 3 * f, hdim, bnd, device).view(3, f, hdim)
        d["W_hh"] = uniform(k, "W_hh", 3 * hdim, hdim, bnd, device).view(3, hdim, hdim)
        d["b_ih"] = uniform(k, "b_ih", 3, hdim, bnd, device)
        d["b_hh"] = uniform(k, "b_hh", 3, hdim, bnd, device)
    elif cfg.model == "sage_lstm":
        f, fo = cfg.dims
        bnd = 1.0 / math.sqrt(f)
        d["X"] = _store(normal(k, f"X/{n}", n, f, 1.0, device), cfg.dtype)
        d["W_ih"] = _store(uniform(k, "W_ih", 4 * f, f, bnd, device), cfg.dtype).view(4, f, f)
        d["W_hh"] = _store(uniform(k, "W_hh", 4 * f, f, bnd, device), cfg.dtype).view(4, f, f)
        d["b_ih"] = uniform(k, "b_ih", 4, f, bnd, device)
        d["b_hh"] = uniform(k, "b_hh", 4, f, bnd, device)
        d["W"] = _store(glorot(k, "W", 2 * f, fo, device), cfg.dtype)
        d["b"] = torch.zeros(fo, dtype=torch.float32, device=device)
    elif cfg.model == "rgcn":
        f, fo = cfg.dims
        T = cfg.num_etypes
        bnd = 1.0 / math.sqrt(f)
        d["H"] = normal(k, f"H/{n}", n, f, 1.0, device)
        d["W_type"] = uniform(k, "W_type", T * f, fo, bnd, device).view(T, f, fo)
        d["W_self"] = uniform(k, "W_self", f, fo, bnd, device)
        d["b"] = uniform(k, "b", 1, fo, bnd, device).view(fo)
    elif cfg.model == "ggnn":
        f, _ = cfg.dims
        bnd_e, bnd = 1.0 / math.sqrt(2 * f), 1.0 / math.sqrt(f)
        d["H"] = normal(k, f"H/{n}", n, f, 1.0, device)
        d["W_e"] = uniform(k, "W_e", 2 * f, f, bnd_e, device)          # [src rows; dst rows] x out
        d["b_e"] = uniform(k, "b_e", 1, f, bnd_e, device).view(f)
        d["W_ih"] = uniform(k, "W_ih", 3 * f, f, bnd, device).view(3, f, f)
        d["W_hh"] = uniform(k, "W_hh", 3 * f, f, bnd, device).view(3, f, f)
        d["b_ih"] = uniform(k, "b_ih", 3, f, bnd, device)
        d["b_hh"] = uniform(k, "b_hh", 3, f, bnd, device)
    else:
        raise ValueError(cfg.model)
    return d
