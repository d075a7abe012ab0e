"""Pins for oracle.rgcn (Table 1,
lines 327-328; reading A24), against things other than the oracle:

* dense brute force in NumPy with per-type, row-normalised adjacency
  matrices A_t / c_{v,t} (the matrix form of Gather, PAPER.md 350-354),
* the same layer written with torch.sparse (a library SpMM) in fp64,
* reductions: T = 1 gives GraphSAGE-mean with W = [W_self; W_1]
  (torch matmul on [H || mean]); all W_t = 0 gives ReLU(H W_self + b); a
  vertex with no in-edges of type t gets no contribution from W_t.
"""
import numpy as np
import pytest
import torch

import oracle
from tests import zoo

RNG = np.random.default_rng(179)


def dense_adj(n, src, dst):
    A = np.zeros((n, n))
    np.add.at(A, (dst, src), 1.0)
    return A


def rgcn_dense(n, s, d, et, T, H, Wt, Ws, b, act=True):
    out = H @ Ws + b
    for t in range(T):
        sel = et == t
        A = dense_adj(n, s[sel], d[sel])
        c = A.sum(1)
        An = np.where(c[:, None] > 0, A / np.maximum(c, 1)[:, None], 0.0)
        out = out + An @ H @ Wt[t]
    return np.maximum(out, 0) if act else out


GRAPHS = [z for z in zoo.zoo() if z[1] > 0]


@pytest.mark.parametrize("name,n,s,d", GRAPHS, ids=[g[0] for g in GRAPHS])
def test_rgcn_dense_bruteforce(name, n, s, d):
    T, f, fo = 3, 6, 5
    et = (np.arange(s.shape[0]) * 5 % T).astype(np.int32)
    H = RNG.standard_normal((n, f))
    Wt = RNG.standard_normal((T, f, fo))
    Ws = RNG.standard_normal((f, fo))
    b = RNG.standard_normal(fo)
    g = oracle.csr_build(n, s, d, et, T)
    for act in (0, 1):
        np.testing.assert_allclose(oracle.rgcn(g, H, Wt, Ws, b, act=act),
                                   rgcn_dense(n, s, d, et, T, H, Wt, Ws, b, act == 1), rtol=1e-11, atol=1e-12)


def test_rgcn_torch_sparse_library():
    n, e, T, f = 300, 2500, 4, 8
    s, d = zoo.random_multigraph(n, e, 21)
    et = RNG.integers(0, T, e).astype(np.int32)
    H = torch.randn(n, f, dtype=torch.float64, generator=torch.Generator().manual_seed(5))
    Wt = torch.randn(T, f, f, dtype=torch.float64, generator=torch.Generator().manual_seed(6))
    Ws = torch.randn(f, f, dtype=torch.float64, generator=torch.Generator().manual_seed(7))
    ref = H @ Ws
    for t in range(T):
        sel = torch.from_numpy(et == t)
        dst_t, src_t = torch.from_numpy(d)[sel].long(), torch.from_numpy(s)[sel].long()
        cnt = torch.bincount(dst_t, minlength=n).double()
        w = 1.0 / cnt[dst_t]
        A = torch.sparse_coo_tensor(torch.stack([dst_t, src_t]), w, (n, n))
        ref = ref + torch.sparse.mm(A, H) @ Wt[t]
    y = oracle.rgcn(oracle.csr_build(n, s, d, et, T), H.numpy(), Wt.numpy(), Ws.numpy(), act=0)
    np.testing.assert_allclose(y, ref.numpy(), rtol=1e-11, atol=1e-12)


def test_rgcn_reductions():
    n, e, f, fo = 64, 300, 7, 4
    s, d = zoo.random_multigraph(n, e, 3)
    H = RNG.standard_normal((n, f))
    Ws = RNG.standard_normal((f, fo))
    W1 = RNG.standard_normal((f, fo))
    g1 = oracle.csr_build(n, s, d)
    # T = 1 is GraphSAGE-mean on [H || mean] with W = [W_self; W_1] (a second oracle
    # function, itself pinned by dense brute force) and the torch formula
    y = oracle.rgcn(g1, H, W1[None], Ws, act=1)
    np.testing.assert_allclose(y, oracle.sage_mean(g1, H, np.concatenate([Ws, W1]), act=1), rtol=1e-12)
    A = dense_adj(n, s, d)
    c = A.sum(1)
    M = np.where(c[:, None] > 0, (A @ H) / np.maximum(c, 1)[:, None], 0.0)
    ref = torch.relu(torch.from_numpy(np.concatenate([H, M], 1)) @ torch.from_numpy(np.concatenate([Ws, W1])))
    np.testing.assert_allclose(y, ref.numpy(), rtol=1e-12)
    # all type weights zero -> only the self connection
    T = 3
    et = (np.arange(e) % T).astype(np.int32)
    g = oracle.csr_build(n, s, d, et, T)
    b = RNG.standard_normal(fo)
    np.testing.assert_allclose(oracle.rgcn(g, H, np.zeros((T, f, fo)), Ws, b), np.maximum(H @ Ws + b, 0),
                               rtol=1e-14)
    # a type a vertex never receives contributes nothing (no 0/0)
    et2 = np.zeros(e, np.int32)
    g2 = oracle.csr_build(n, s, d, et2, T)
    Wt = RNG.standard_normal((T, f, fo))
    Wt_only0 = Wt.copy()
    Wt_only0[1:] = 1e300   # would overflow if types 1, 2 were touched
    y2 = oracle.rgcn(g2, H, Wt_only0, Ws, act=0)
    assert np.all(np.isfinite(y2))
    np.testing.assert_allclose(y2, oracle.rgcn(g1, H, Wt[:1], Ws, act=0), rtol=1e-12)
