"""Pins for oracle.ggnn (Table 1
line 178, line 218; reading A26), against things other than the oracle:

* per-edge brute force in NumPy written edge-list-first (COO order, no CSR):
  concatenate [H[u] || H[v]], one matrix product per edge, ReLU, scatter-add
  (or scatter-max with np.maximum.at) into the destination, then
  torch.nn.GRUCell in fp64 (a library cell),
* the linear case (no activation) in closed matrix form:
  m = A H W_a + diag(deg) (H W_b + 1 b^T) with the dense adjacency A,
* reductions: W_b = 0, b_e = 0, no activation, sum gives the gated layer with
  one edge type and W_type = W_a (oracle.gated, itself pinned);
  all-zero GRU weights and biases give h' = h / 2;
  a vertex without in-edges gets m = 0 for both aggregators.
"""
import numpy as np
import pytest
import torch

import oracle
from tests import zoo

RNG = np.random.default_rng(178)
GRAPHS = [z for z in zoo.zoo() if z[1] > 0]


def gru_torch(m, h, W_ih, W_hh, b_ih, b_hh):
    f = W_ih.shape[1]
    cell = torch.nn.GRUCell(f, f).double()
    with torch.no_grad():
        cell.weight_ih.copy_(torch.from_numpy(np.concatenate([W_ih[g].T for g in range(3)], 0)))
        cell.weight_hh.copy_(torch.from_numpy(np.concatenate([W_hh[g].T for g in range(3)], 0)))
        cell.bias_ih.copy_(torch.from_numpy(b_ih.reshape(-1)))
        cell.bias_hh.copy_(torch.from_numpy(b_hh.reshape(-1)))
        return cell(torch.from_numpy(m), torch.from_numpy(h)).numpy()


def params(f, scale=0.3):
    return (RNG.uniform(-scale, scale, (2 * f, f)), RNG.uniform(-scale, scale, f),
            RNG.uniform(-scale, scale, (3, f, f)), RNG.uniform(-scale, scale, (3, f, f)),
            RNG.uniform(-scale, scale, (3, f)), RNG.uniform(-scale, scale, (3, f)))


def ggnn_edges(n, s, d, H, We, be, Wih, Whh, bih, bhh, relu=True, agg="sum"):
    f = H.shape[1]
    x = np.concatenate([H[s], H[d]], axis=1)          # Scatter, edge by edge (COO order)
    y = x @ We + be                                    # ApplyEdge
    if relu:
        y = np.maximum(y, 0.0)
    if agg == "sum":
        m = np.zeros((n, f))
        np.add.at(m, d, y)
    else:
        m = np.full((n, f), -np.inf)
        np.maximum.at(m, d, y)
        m[np.isinf(m)] = 0.0                           # no in-edges -> 0
    return gru_torch(m, H, Wih, Whh, bih, bhh)


@pytest.mark.parametrize("name,n,s,d", GRAPHS, ids=[g[0] for g in GRAPHS])
@pytest.mark.parametrize("agg", ["sum", "max"])
def test_ggnn_edge_bruteforce(name, n, s, d, agg):
    f = 5
    H = RNG.standard_normal((n, f))
    We, be, Wih, Whh, bih, bhh = params(f)
    g = oracle.csr_build(n, s, d)
    for relu in (True, False):
        y = oracle.ggnn(g, H, We, be, Wih, Whh, bih, bhh, act=1 if relu else 0, agg=agg)
        ref = ggnn_edges(n, s, d, H, We, be, Wih, Whh, bih, bhh, relu, agg)
        np.testing.assert_allclose(y, ref, rtol=1e-11, atol=1e-12)


def test_ggnn_linear_closed_form():
    n, e, f = 120, 900, 6
    s, d = zoo.random_multigraph(n, e, 17)
    H = RNG.standard_normal((n, f))
    We, be, Wih, Whh, bih, bhh = params(f)
    A = np.zeros((n, n))
    np.add.at(A, (d, s), 1.0)
    deg = A.sum(1)
    m = A @ H @ We[:f] + deg[:, None] * (H @ We[f:] + be)
    ref = gru_torch(m, H, Wih, Whh, bih, bhh)
    y = oracle.ggnn(oracle.csr_build(n, s, d), H, We, be, Wih, Whh, bih, bhh, act=0)
    np.testing.assert_allclose(y, ref, rtol=1e-11, atol=1e-12)


def test_ggnn_reduces_to_gated():
    n, e, f = 80, 500, 7
    s, d = zoo.random_multigraph(n, e, 4)
    H = RNG.standard_normal((n, f))
    We, be, Wih, Whh, bih, bhh = params(f)
    We[f:] = 0.0
    g = oracle.csr_build(n, s, d)
    y = oracle.ggnn(g, H, We, np.zeros(f), Wih, Whh, bih, bhh, act=0)
    ref = oracle.gated(g, H, We[:f][None], Wih, Whh, bih, bhh)
    np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-13)


def test_ggnn_zero_gru_and_empty_rows():
    n, f = 6, 4
    s = np.array([0, 1, 1], np.int32)
    d = np.array([2, 2, 3], np.int32)               # vertices 0, 1, 4, 5 have no in-edges
    H = RNG.standard_normal((n, f))
    We, be, _, _, _, _ = params(f)
    z3 = np.zeros((3, f, f))
    zb = np.zeros((3, f))
    g = oracle.csr_build(n, s, d)
    for agg in ("sum", "max"):
        np.testing.assert_allclose(oracle.ggnn(g, H, We, be, z3, z3, zb, zb, agg=agg), 0.5 * H, rtol=1e-14)
    # m = 0 for the empty rows: their GRU sees only h
    _, _, Wih, Whh, bih, bhh = params(f)
    y = oracle.ggnn(g, H, We, be, Wih, Whh, bih, bhh, agg="max")
    ref = gru_torch(np.zeros((n, f)), H, Wih, Whh, bih, bhh)
    np.testing.assert_allclose(y[[0, 1, 4, 5]], ref[[0, 1, 4, 5]], rtol=1e-12, atol=1e-13)


def test_ggnn_rows_sampling_matches_full():
    n, e, f = 200, 1500, 4
    s, d = zoo.random_multigraph(n, e, 9)
    H = RNG.standard_normal((n, f))
    We, be, Wih, Whh, bih, bhh = params(f)
    g = oracle.csr_build(n, s, d)
    full = oracle.ggnn(g, H, We, be, Wih, Whh, bih, bhh, agg="max")
    rows = np.array([3, 150, 0, 199], np.int64)
    np.testing.assert_array_equal(oracle.ggnn(g, H, We, be, Wih, Whh, bih, bhh, agg="max", rows=rows), full[rows])
