"""Tiny-graph zoo for pins and GPU edge cases (SURVEY.md 8(c) "Tiny-graph zoo").

Each entry is (name, n, src, dst) with int32 numpy arrays.  Shared by the
oracle pin tests and the GPU parity tests; holds no layer arithmetic.
"""
import numpy as np


def _g(name, n, edges):
    e = np.asarray(edges, dtype=np.int32).reshape(-1, 2)
    return name, n, np.ascontiguousarray(e[:, 0]), np.ascontiguousarray(e[:, 1])


def with_self_loops(n, src, dst):
    v = np.arange(n, dtype=np.int32)
    return np.concatenate([src, v]), np.concatenate([dst, v])


def circulant(n, d):
    """Directed d-regular circulant: v <- v-1, ..., v-d (mod n)."""
    src, dst = [], []
    for v in range(n):
        for k in range(1, d + 1):
            src.append((v - k) % n)
            dst.append(v)
    return np.asarray(src, np.int32), np.asarray(dst, np.int32)


def random_multigraph(n, e, seed):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, e, dtype=np.int64).astype(np.int32)
    dst = rng.integers(0, n // 2 + 1, e, dtype=np.int64).astype(np.int32)  # leaves zero-degree rows
    dup = rng.integers(0, e, e // 5)
    src[: e // 5] = src[dup]
    dst[: e // 5] = dst[dup]
    return src, dst


def hub_graph(n, hub_deg, seed):
    """One vertex (0) with in-degree `hub_deg` plus a sparse random remainder."""
    rng = np.random.default_rng(seed)
    s1 = rng.integers(0, n, hub_deg).astype(np.int32)
    d1 = np.zeros(hub_deg, np.int32)
    s2 = rng.integers(0, n, 4 * n).astype(np.int32)
    d2 = rng.integers(0, n, 4 * n).astype(np.int32)
    return np.concatenate([s1, s2]), np.concatenate([d1, d2])


def zoo(include_big=False):
    out = [
        _g("empty", 3, []),
        _g("single_selfloop", 1, [(0, 0)]),
        _g("two_cycle", 2, [(0, 1), (1, 0)]),
        _g("star_in", 6, [(i, 0) for i in range(1, 6)]),
        _g("star_out", 6, [(0, i) for i in range(1, 6)]),
        _g("path", 3, [(0, 1), (1, 2)]),
        _g("k8", 8, [(u, v) for u in range(8) for v in range(8) if u != v]),
    ]
    s, d = circulant(16, 3)
    out.append(("circulant16_3", 16, s, d))
    s, d = random_multigraph(64, 300, 7)
    out.append(("multigraph64", 64, s, d))
    s, d = random_multigraph(333, 2500, 11)      # N not a multiple of 128 (GEMM tails)
    out.append(("multigraph333", 333, s, d))
    if include_big:
        s, d = hub_graph(5000, 70000, 3)         # exercises hub splitting
        out.append(("hub70k", 5000, s, d))
    return out
