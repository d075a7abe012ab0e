"""Pins for oracle.sage_lstm (Table 1,
lines 357-360; reading A25), against things other than the oracle:

* torch.nn.LSTMCell in fp64 run over each vertex's in-edges in ascending COO
  index order, then torch matmul for the GraphSAGE concat-GEMM,
* all-zero LSTM parameters give h = 0; a length-1
  sequence is one cell step from the zero state (closed form below),
* the sequence semantics: swapping the COO order of a vertex's in-edges
  changes its output exactly as swapping the LSTMCell inputs does,
* a vertex without in-edges aggregates to 0.
"""
import numpy as np
import pytest
import torch

import oracle
from tests import zoo

RNG = np.random.default_rng(180)


def lstm_params(f, scale=0.4):
    return (RNG.uniform(-scale, scale, (4, f, f)), RNG.uniform(-scale, scale, (4, f, f)),
            RNG.uniform(-scale, scale, (4, f)), RNG.uniform(-scale, scale, (4, f)))


def torch_ref(n, s, d, X, Wi, Wh, bi, bh, W, b, act=True):
    """Per-vertex torch.nn.LSTMCell over in-edges sorted by COO index."""
    f = X.shape[1]
    cell = torch.nn.LSTMCell(f, f, dtype=torch.float64)
    with torch.no_grad():
        # torch weight layout: weight_ih [4f][f] with rows (gate, out), x . W_ih[g] -> W_ih[g].T rows
        cell.weight_ih.copy_(torch.from_numpy(np.concatenate([Wi[g].T for g in range(4)])))
        cell.weight_hh.copy_(torch.from_numpy(np.concatenate([Wh[g].T for g in range(4)])))
        cell.bias_ih.copy_(torch.from_numpy(bi.reshape(-1)))
        cell.bias_hh.copy_(torch.from_numpy(bh.reshape(-1)))
    Xt = torch.from_numpy(X)
    H = torch.zeros(n, f, dtype=torch.float64)
    order = np.argsort(d, kind="stable")
    with torch.no_grad():
        for v in range(n):
            eids = [e for e in order if d[e] == v]
            h = torch.zeros(1, f, dtype=torch.float64)
            c = torch.zeros(1, f, dtype=torch.float64)
            for e in eids:
                h, c = cell(Xt[s[e]][None], (h, c))
            H[v] = h[0]
        out = torch.cat([Xt, H], 1) @ torch.from_numpy(W) + torch.from_numpy(b)
    out = out.numpy()
    return np.maximum(out, 0) if act else out


GRAPHS = [z for z in zoo.zoo() if 0 < z[1] <= 64]


@pytest.mark.parametrize("name,n,s,d", GRAPHS, ids=[g[0] for g in GRAPHS])
def test_sage_lstm_vs_torch_lstmcell(name, n, s, d):
    f, fo = 5, 4
    X = RNG.standard_normal((n, f))
    Wi, Wh, bi, bh = lstm_params(f)
    W = RNG.standard_normal((2 * f, fo))
    b = RNG.standard_normal(fo)
    g = oracle.csr_build(n, s, d)
    for act in (0, 1):
        np.testing.assert_allclose(oracle.sage_lstm(g, X, Wi, Wh, bi, bh, W, b, act=act),
                                   torch_ref(n, s, d, X, Wi, Wh, bi, bh, W, b, act == 1), rtol=1e-11, atol=1e-12)


def test_sage_lstm_closed_forms():
    n, f, fo = 6, 4, 3
    # star_in: vertex 0 receives 1..5 in order; 1..5 receive nothing
    s = np.array([1, 2, 3, 4, 5], np.int32)
    d = np.zeros(5, np.int32)
    g = oracle.csr_build(n, s, d)
    X = RNG.standard_normal((n, f))
    W = RNG.standard_normal((2 * f, fo))
    b = RNG.standard_normal(fo)
    z4, zb = np.zeros((4, f, f)), np.zeros((4, f))
    # all LSTM parameters zero -> h = 0 -> out = act(x W_self + b)
    np.testing.assert_allclose(oracle.sage_lstm(g, X, z4, z4, zb, zb, W, b, act=0), X @ W[:f] + b, rtol=1e-14)
    # length-1 sequence: one step from the zero state
    Wi, Wh, bi, bh = lstm_params(f)
    g1 = oracle.csr_build(n, np.array([3], np.int32), np.array([0], np.int32))
    zz = np.stack([X[3] @ Wi[k] + bi[k] + bh[k] for k in range(4)])
    sig = lambda t: 1 / (1 + np.exp(-t))
    h = sig(zz[3]) * np.tanh(sig(zz[0]) * np.tanh(zz[2]))
    y = oracle.sage_lstm(g1, X, Wi, Wh, bi, bh, W, b, act=0)
    np.testing.assert_allclose(y[0], X[0] @ W[:f] + h @ W[f:] + b, rtol=1e-13)
    # vertices without in-edges aggregate to zero
    np.testing.assert_allclose(y[1:], X[1:] @ W[:f] + b, rtol=1e-14)


def test_sage_lstm_is_order_sensitive_in_coo_order():
    n, f, fo = 3, 4, 4
    X = RNG.standard_normal((n, f))
    Wi, Wh, bi, bh = lstm_params(f, 0.8)
    W = np.eye(2 * f)[:, :fo * 2]
    ga = oracle.csr_build(n, np.array([1, 2], np.int32), np.array([0, 0], np.int32))
    gb = oracle.csr_build(n, np.array([2, 1], np.int32), np.array([0, 0], np.int32))
    ya = oracle.sage_lstm(ga, X, Wi, Wh, bi, bh, W, act=0)
    yb = oracle.sage_lstm(gb, X, Wi, Wh, bi, bh, W, act=0)
    assert np.max(np.abs(ya[0] - yb[0])) > 1e-3      # a sequence, not a set
    np.testing.assert_allclose(yb, torch_ref(n, np.array([2, 1]), np.array([0, 0]), X, Wi, Wh, bi, bh, W,
                                             np.zeros(W.shape[1]), act=False), rtol=1e-12)
