"""Pins for the oracle's layer functions, against things other than the oracle.

* dense-adjacency brute force in NumPy and torch fp64 (matrix formulation of
  PAPER.md lines 350-354: fused Gather = adjacency x embedding matrix),
* closed forms (d-regular GCN, BASELINE.json north_star; GAT with zero
  attention; GRU with zero weights),
* a library cell (torch.nn.GRUCell in fp64),
* a hand-computed golden fixture (tests/golden/gcn_path.txt),
* invariants: attention weights sum to 1, relabelling equivariance,
  COO-order independence, determinism.
"""
import math
import os

import numpy as np
import pytest
import torch

import oracle
from tests import zoo

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
RNG = np.random.default_rng(2009_00804)


def dense_adj(n, src, dst):
    """A[v, u] = multiplicity of edge u -> v (row = destination)."""
    A = np.zeros((n, n))
    np.add.at(A, (dst, src), 1.0)
    return A


def graphs():
    out = []
    for name, n, s, d in zoo.zoo():
        if n == 0:
            continue
        out.append((name, n, s, d))
        s2, d2 = zoo.with_self_loops(n, s, d)
        out.append((name + "+I", n, s2, d2))
    return out


GRAPHS = graphs()
IDS = [g[0] for g in GRAPHS]


# ------------------------------------------------------------------- GCN ----

def gcn_dense(n, s, d, X, Wm, b, act=True):
    A = dense_adj(n, s, d)
    deg = A.sum(1)
    dinv = np.where(deg > 0, 1.0 / np.sqrt(np.maximum(deg, 1)), 0.0)
    Y = (dinv[:, None] * A * dinv[None, :]) @ X @ Wm + b
    return np.maximum(Y, 0) if act else Y


@pytest.mark.parametrize("name,n,s,d", GRAPHS, ids=IDS)
def test_gcn_dense_bruteforce(name, n, s, d):
    X = RNG.standard_normal((n, 12))
    Wm = RNG.standard_normal((12, 5))
    b = RNG.standard_normal(5)
    g = oracle.csr_build(n, s, d)
    for act in (0, 1):
        y = oracle.gcn(g, X, Wm, b, act=act)
        np.testing.assert_allclose(y, gcn_dense(n, s, d, X, Wm, b, bool(act)), rtol=1e-12, atol=1e-12)


def test_gcn_torch_sparse_library():
    """torch.sparse.mm in fp64 (a library SpMM) on a random multigraph + I."""
    s, d = zoo.random_multigraph(300, 2000, 1)
    s, d = zoo.with_self_loops(300, s, d)
    X = torch.randn(300, 16, dtype=torch.float64)
    Wm = torch.randn(16, 8, dtype=torch.float64)
    deg = torch.bincount(torch.from_numpy(d).long(), minlength=300).double()
    w = deg[torch.from_numpy(s).long()].rsqrt() * deg[torch.from_numpy(d).long()].rsqrt()
    A = torch.sparse_coo_tensor(torch.stack([torch.from_numpy(d).long(), torch.from_numpy(s).long()]), w, (300, 300))
    ref = torch.relu(torch.sparse.mm(A, X) @ Wm).numpy()
    y = oracle.gcn(oracle.csr_build(300, s, d), X, Wm)
    np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("deg_d", [1, 3, 7])
def test_gcn_regular_closed_form(deg_d):
    """BASELINE.json north_star: on a d-regular graph with self-loops, W = I,
    X >= 0, the GCN layer is (x_v + sum_{u in N(v)} x_u) / (d+1)."""
    n = 40
    s, d = zoo.circulant(n, deg_d)
    s, d = zoo.with_self_loops(n, s, d)
    X = RNG.uniform(0, 1, (n, 6))
    y = oracle.gcn(oracle.csr_build(n, s, d), X, np.eye(6))
    ref = np.empty_like(X)
    for v in range(n):
        ref[v] = (X[v] + sum(X[(v - k) % n] for k in range(1, deg_d + 1))) / (deg_d + 1)
    np.testing.assert_allclose(y, ref, rtol=1e-13)
    # neighbour mean scaled by d/(d+1) plus x_v/(d+1)
    nb = np.stack([np.mean([X[(v - k) % n] for k in range(1, deg_d + 1)], axis=0) for v in range(n)])
    np.testing.assert_allclose(y, deg_d / (deg_d + 1) * nb + X / (deg_d + 1), rtol=1e-13)


def test_gcn_path_golden():
    """Reading A1 (in-degree of A+I on both sides) on the non-regular path
    0->1->2 + self-loops: hand-computed values in tests/golden/gcn_path.txt."""
    vals = {}
    for line in open(os.path.join(GOLDEN, "gcn_path.txt")):
        line = line.split("#")[0].strip()
        if ":" in line:
            k, v = line.split(":", 1)
            vals[k.strip()] = [float(t) for t in v.split()]
    s, d = zoo.with_self_loops(3, np.array([0, 1], np.int32), np.array([1, 2], np.int32))
    X = np.array(vals["x"])[:, None]
    y = oracle.gcn(oracle.csr_build(3, s, d), X, np.eye(1), act=0)
    np.testing.assert_allclose(y[:, 0], vals["out"], rtol=1e-12)


# ------------------------------------------------------------------ SAGE ----

def sage_dense(n, s, d, X, Wm, act=True):
    A = dense_adj(n, s, d)
    deg = A.sum(1)
    M = np.where(deg[:, None] > 0, (A @ X) / np.maximum(deg, 1)[:, None], 0.0)
    Y = np.concatenate([X, M], 1) @ Wm
    return np.maximum(Y, 0) if act else Y


@pytest.mark.parametrize("name,n,s,d", GRAPHS, ids=IDS)
def test_sage_dense_bruteforce(name, n, s, d):
    X = RNG.standard_normal((n, 10))
    Wm = RNG.standard_normal((20, 7))
    g = oracle.csr_build(n, s, d)
    for act in (0, 1):
        np.testing.assert_allclose(oracle.sage_mean(g, X, Wm, act=act), sage_dense(n, s, d, X, Wm, bool(act)),
                                   rtol=1e-12, atol=1e-12)


def test_sage_star_and_zero_neighbour_weight():
    n = 6
    s = np.arange(1, 6, dtype=np.int32)
    d = np.zeros(5, np.int32)
    X = RNG.standard_normal((n, 4))
    Wm = RNG.standard_normal((8, 3))
    y = oracle.sage_mean(oracle.csr_build(n, s, d), X, Wm, act=0)
    np.testing.assert_allclose(y[0], X[0] @ Wm[:4] + X[1:].mean(0) @ Wm[4:], rtol=1e-12)
    np.testing.assert_allclose(y[1:], X[1:] @ Wm[:4], rtol=1e-12)   # leaves: empty mean = 0 (A12)
    W0 = Wm.copy()
    W0[4:] = 0.0                                                     # W_neigh = 0 -> plain GEMM
    s2, d2 = zoo.random_multigraph(50, 400, 2)
    X2 = RNG.standard_normal((50, 4))
    y2 = oracle.sage_mean(oracle.csr_build(50, s2, d2), X2, W0, act=1)
    np.testing.assert_allclose(y2, np.maximum(np.matmul(X2, W0[:4]), 0), rtol=1e-12, atol=1e-14)


# ------------------------------------------------------------------- GAT ----

def gat_dense(n, s, d, X, Wm, a_s, a_d, slope):
    A = dense_adj(n, s, d)
    H, D = a_s.shape
    z = X @ Wm
    out = np.zeros((n, H * D))
    for h in range(H):
        zh = z[:, h * D:(h + 1) * D]
        el = zh @ a_s[h]
        er = zh @ a_d[h]
        S = er[:, None] + el[None, :]
        S = np.where(S > 0, S, slope * S)
        S = np.where(A > 0, S, -np.inf)
        mx = S.max(1, keepdims=True)
        mx = np.where(np.isfinite(mx), mx, 0.0)
        P = A * np.exp(S - mx)                      # multiplicity-weighted terms
        den = P.sum(1, keepdims=True)
        alpha = np.where(den > 0, P / np.where(den > 0, den, 1), 0.0)
        out[:, h * D:(h + 1) * D] = alpha @ zh
    return np.where(out > 0, out, np.expm1(out))


@pytest.mark.parametrize("name,n,s,d", GRAPHS, ids=IDS)
def test_gat_dense_bruteforce(name, n, s, d):
    X = RNG.standard_normal((n, 9))
    Wm = RNG.standard_normal((9, 12))
    a_s = RNG.standard_normal((3, 4))
    a_d = RNG.standard_normal((3, 4))
    y = oracle.gat(oracle.csr_build(n, s, d), X, Wm, a_s, a_d, 0.2)
    np.testing.assert_allclose(y, gat_dense(n, s, d, X, Wm, a_s, a_d, 0.2), rtol=1e-11, atol=1e-12)


def test_gat_alpha_sums_to_one_and_special_cases():
    s, d = zoo.random_multigraph(120, 900, 4)
    s, d = zoo.with_self_loops(120, s, d)
    g = oracle.csr_build(120, s, d)
    X = RNG.standard_normal((120, 8))
    Wm = RNG.standard_normal((8, 8))
    a_s = RNG.standard_normal((2, 4))
    a_d = RNG.standard_normal((2, 4))
    y, alpha = oracle.gat(g, X, Wm, a_s, a_d, 0.2, want_alpha=True)
    seg = np.repeat(np.arange(120), np.diff(g.row_ptr))
    sums = np.zeros((120, 2))
    np.add.at(sums, seg, alpha)
    np.testing.assert_allclose(sums, 1.0, atol=1e-12)           # north_star: sum alpha = 1
    # a_src = a_dst = 0: uniform weights -> ELU(mean over the in-edge multiset)
    z = X @ Wm
    y0 = oracle.gat(g, X, Wm, np.zeros((2, 4)), np.zeros((2, 4)), 0.2)
    mean = np.zeros((120, 8))
    np.add.at(mean, seg, z[g.col_src])
    mean /= np.diff(g.row_ptr)[:, None]
    np.testing.assert_allclose(y0, np.where(mean > 0, mean, np.expm1(mean)), rtol=1e-12, atol=1e-14)
    # self-loop-only graph: out = ELU(z); single in-edge: alpha = 1
    v = np.arange(10, dtype=np.int32)
    y1, a1 = oracle.gat(oracle.csr_build(10, v, v), X[:10], Wm, a_s, a_d, 0.2, want_alpha=True)
    np.testing.assert_allclose(a1, 1.0)
    np.testing.assert_allclose(y1, np.where(z[:10] > 0, z[:10], np.expm1(z[:10])), rtol=1e-12)


# ----------------------------------------------------------------- Gated ----

def gru_torch(m, h, W_ih, W_hh, b_ih, b_hh):
    f, hid = W_ih.shape[1], W_ih.shape[2]
    cell = torch.nn.GRUCell(f, hid).double()
    with torch.no_grad():
        cell.weight_ih.copy_(torch.from_numpy(np.concatenate([W_ih[g].T for g in range(3)], 0)))
        cell.weight_hh.copy_(torch.from_numpy(np.concatenate([W_hh[g].T for g in range(3)], 0)))
        cell.bias_ih.copy_(torch.from_numpy(b_ih.reshape(-1)))
        cell.bias_hh.copy_(torch.from_numpy(b_hh.reshape(-1)))
        return cell(torch.from_numpy(m), torch.from_numpy(h)).numpy()


def gated_params(f, T, scale=0.3):
    return (RNG.uniform(-scale, scale, (T, f, f)), RNG.uniform(-scale, scale, (3, f, f)),
            RNG.uniform(-scale, scale, (3, f, f)), RNG.uniform(-scale, scale, (3, f)),
            RNG.uniform(-scale, scale, (3, f)))


@pytest.mark.parametrize("name,n,s,d", GRAPHS, ids=IDS)
def test_gated_dense_and_grucell(name, n, s, d):
    T, f = 3, 6
    et = (np.arange(s.shape[0]) * 7 % T).astype(np.int32)
    H = RNG.standard_normal((n, f))
    Wt, Wih, Whh, bih, bhh = gated_params(f, T)
    g = oracle.csr_build(n, s, d, et, T)
    y = oracle.gated(g, H, Wt, Wih, Whh, bih, bhh)
    m = np.zeros((n, f))
    for t in range(T):
        sel = et == t
        m += (dense_adj(n, s[sel], d[sel]) @ H) @ Wt[t]
    np.testing.assert_allclose(y, gru_torch(m, H, Wih, Whh, bih, bhh), rtol=1e-11, atol=1e-12)


def test_gated_messages_per_edge():
    """ApplyEdge is per edge: m[v] = sum over in-edges
    e = (u -> v) of H[u] . W_type(e), summed edge by edge with np.add.at and
    no per-type grouping, against the oracle's GRU of it (a wrong type index
    or a transposed W_t fails here)."""
    n, T, f = 30, 3, 5
    s, d = zoo.random_multigraph(n, 150, 21)
    et = (np.arange(150) * 5 % T).astype(np.int32)
    H = RNG.standard_normal((n, f))
    Wt, Wih, Whh, bih, bhh = gated_params(f, T)
    msgs = np.einsum("ek,ekj->ej", H[s], Wt[et])
    m = np.zeros((n, f))
    np.add.at(m, d, msgs)
    y = oracle.gated(oracle.csr_build(n, s, d, et, T), H, Wt, Wih, Whh, bih, bhh)
    np.testing.assert_allclose(y, gru_torch(m, H, Wih, Whh, bih, bhh), rtol=1e-11, atol=1e-12)


def test_rgcn_messages_per_edge():
    """R-GCN (reading A24): out[v] = act(sum_e H[u] W_type(e) / c_{v,type(e)} +
    H[v] W_self + b), accumulated edge by edge."""
    n, T, f, fo = 25, 4, 4, 3
    s, d = zoo.random_multigraph(n, 120, 22)
    et = (np.arange(120) * 3 % T).astype(np.int32)
    X = RNG.standard_normal((n, f))
    Wt, Ws, b = RNG.standard_normal((T, f, fo)), RNG.standard_normal((f, fo)), RNG.standard_normal(fo)
    c = np.zeros((n, T))
    np.add.at(c, (d, et), 1.0)
    msgs = np.einsum("ek,ekj->ej", X[s], Wt[et]) / c[d, et][:, None]
    ref = X @ Ws + b
    np.add.at(ref, d, msgs)
    y = oracle.rgcn(oracle.csr_build(n, s, d, et, T), X, Wt, Ws, b, act=0)
    np.testing.assert_allclose(y, ref, rtol=1e-11, atol=1e-12)


def test_gated_gru_closed_forms():
    s, d = zoo.random_multigraph(40, 200, 9)
    et = (np.arange(200) % 4).astype(np.int32)
    g = oracle.csr_build(40, s, d, et, 4)
    H = RNG.standard_normal((40, 5))
    Wt = RNG.standard_normal((4, 5, 5))
    z3 = np.zeros((3, 5, 5))
    zb = np.zeros((3, 5))
    # all GRU weights and biases zero -> h' = 0.5 h
    np.testing.assert_allclose(oracle.gated(g, H, Wt, z3, z3, zb, zb), 0.5 * H, rtol=1e-15)
    # zero weights, nonzero biases -> PyTorch-form closed form (reading A15);
    # the Cho/GGNN variant of SPEC.md line 253 would give a different value.
    bih = RNG.standard_normal((3, 5))
    bhh = RNG.standard_normal((3, 5))
    sig = lambda x: 1 / (1 + np.exp(-x))
    zg = sig(bih[1] + bhh[1])
    ng = np.tanh(bih[2] + sig(bih[0] + bhh[0]) * bhh[2])
    np.testing.assert_allclose(oracle.gated(g, H, Wt, z3, z3, bih, bhh), (1 - zg) * ng + zg * H, rtol=1e-13)
    # T = 1, W = I: m is the plain in-neighbour sum
    g1 = oracle.csr_build(40, s, d)
    Wih, Whh = RNG.standard_normal((3, 5, 5)), RNG.standard_normal((3, 5, 5))
    y = oracle.gated(g1, H, np.eye(5)[None], Wih, Whh, bih, bhh)
    m = dense_adj(40, s, d) @ H
    np.testing.assert_allclose(y, gru_torch(m, H, Wih, Whh, bih, bhh), rtol=1e-11)
    # all W_t equal -> result independent of the edge types
    Weq = np.repeat(Wt[:1], 4, 0)
    np.testing.assert_allclose(oracle.gated(g, H, Weq, Wih, Whh, bih, bhh),
                               oracle.gated(g1, H, Wt[:1], Wih, Whh, bih, bhh), rtol=1e-12)


# ------------------------------------------------------------ invariants ----

def _all_models(g, n, X, et=None):
    Wg = np.linspace(-1, 1, X.shape[1] * 4).reshape(X.shape[1], 4)
    Ws = np.linspace(-1, 1, 2 * X.shape[1] * 3).reshape(2 * X.shape[1], 3)
    a = np.linspace(-0.5, 0.5, 4).reshape(2, 2)
    f = X.shape[1]
    P = [np.sin(np.arange(k)).reshape(sh) for k, sh in
         [(2 * f * f, (2, f, f)), (3 * f * f, (3, f, f)), (3 * f * f, (3, f, f)), (3 * f, (3, f)), (3 * f, (3, f))]]
    return [oracle.gcn(g, X, Wg), oracle.sage_mean(g, X, Ws), oracle.gat(g, X, Wg, a, a[::-1]),
            oracle.gated(g, X, *P), oracle.rgcn(g, X, np.stack([Wg, Wg[::-1]]), Wg[:, ::-1].copy())]


def test_relabel_equivariance_bitexact():
    n = 90
    s, d = zoo.random_multigraph(n, 700, 12)
    s, d = zoo.with_self_loops(n, s, d)
    et = (np.arange(s.shape[0]) % 2).astype(np.int32)
    X = RNG.standard_normal((n, 6))
    perm = RNG.permutation(n).astype(np.int32)          # new id of old vertex v is perm[v]
    Xp = np.empty_like(X)
    Xp[perm] = X
    base = _all_models(oracle.csr_build(n, s, d, et, 2), n, X)
    relab = _all_models(oracle.csr_build(n, perm[s], perm[d], et, 2), n, Xp)
    for y, yp in zip(base, relab):
        np.testing.assert_array_equal(yp[perm], y)      # same per-row order -> bit-exact


def test_coo_order_shuffle_and_determinism():
    n = 90
    s, d = zoo.random_multigraph(n, 700, 13)
    et = (np.arange(700) % 2).astype(np.int32)
    X = RNG.standard_normal((n, 6))
    sh = RNG.permutation(700)
    a = _all_models(oracle.csr_build(n, s, d, et, 2), n, X)
    b = _all_models(oracle.csr_build(n, s[sh], d[sh], et[sh], 2), n, X)
    c = _all_models(oracle.csr_build(n, s, d, et, 2), n, X)
    for y, yb, yc in zip(a, b, c):
        assert oracle.rel_err(yb, y) < 1e-12
        np.testing.assert_array_equal(y, yc)


def test_row_subset_matches_full():
    s, d = zoo.random_multigraph(80, 500, 3)
    g = oracle.csr_build(80, s, d, (np.arange(500) % 2).astype(np.int32), 2)
    X = RNG.standard_normal((80, 6))
    rows = np.array([79, 0, 5, 5, 33], np.int64)
    Wg = RNG.standard_normal((6, 4))
    np.testing.assert_array_equal(oracle.gcn(g, X, Wg, rows=rows), oracle.gcn(g, X, Wg)[rows])
    Ws = RNG.standard_normal((12, 4))
    np.testing.assert_array_equal(oracle.sage_mean(g, X, Ws, rows=rows), oracle.sage_mean(g, X, Ws)[rows])
    a = RNG.standard_normal((2, 2))
    np.testing.assert_array_equal(oracle.gat(g, X, Wg, a, a, rows=rows), oracle.gat(g, X, Wg, a, a)[rows])
    P = gated_params(6, 2)
    np.testing.assert_array_equal(oracle.gated(g, X, *P, rows=rows), oracle.gated(g, X, *P)[rows])


def test_bf16_and_f32_feature_upcast_exact():
    s, d = zoo.random_multigraph(50, 300, 8)
    g = oracle.csr_build(50, s, d)
    Xb = torch.randn(50, 8).to(torch.bfloat16)
    Wg = RNG.standard_normal((8, 3))
    y_b = oracle.gcn(g, Xb, Wg)
    y_d = oracle.gcn(g, Xb.double().numpy(), Wg)
    np.testing.assert_array_equal(y_b, y_d)
    Xf = torch.randn(50, 8)
    np.testing.assert_array_equal(oracle.gcn(g, Xf, Wg), oracle.gcn(g, Xf.double().numpy(), Wg))
