"""ctypes front-end of the fp64 CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` leg may import this package.  The product
path (paper_2009_00804_b200) never imports it and shares no code with it.

Each wrapper takes torch CPU tensors / numpy arrays and returns numpy fp64
results.  Citations for every definition live in oracle.c.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

X_F32, X_BF16, X_F64 = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (baseline x86-64, no -march=native, no FMA
    contraction, OpenMP over destination rows)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
                               "-std=c11", _SRC, "-o", _SO, "-lm"])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        i32, i64, dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        L.oracle_csr_build.restype = i64
        L.oracle_csr_build.argtypes = [i32, i64, P, P, P, i32, P, P, P, P, P, P]
        L.oracle_gcn.restype = None
        L.oracle_gcn.argtypes = [i32, P, P, P, P, ctypes.c_int, i32, P, i32, P, ctypes.c_int, P, i64, P]
        L.oracle_sage_mean.restype = None
        L.oracle_sage_mean.argtypes = [i32, P, P, P, P, ctypes.c_int, i32, P, i32, P, ctypes.c_int, P, i64, P]
        L.oracle_gat.restype = None
        L.oracle_gat.argtypes = [i32, P, P, P, ctypes.c_int, i32, P, i32, i32, P, P, dbl, P, i64, P, P]
        L.oracle_gated.restype = None
        L.oracle_gated.argtypes = [i32, P, P, P, i32, P, ctypes.c_int, i32, P, P, P, P, P, P, i64, P]
        L.oracle_sage_lstm.restype = None
        L.oracle_sage_lstm.argtypes = [i32, P, P, P, ctypes.c_int, i32, P, P, P, P, P, i32, P, ctypes.c_int, P, i64, P]
        L.oracle_ggnn.restype = None
        L.oracle_ggnn.argtypes = [i32, P, P, P, ctypes.c_int, i32, P, P, ctypes.c_int, ctypes.c_int,
                                  P, P, P, P, P, i64, P]
        L.oracle_rgcn.restype = None
        L.oracle_rgcn.argtypes = [i32, P, P, P, i32, P, ctypes.c_int, i32, P, P, i32, P, ctypes.c_int, P, i64, P]
        _lib = L
    return _lib


def _np(t, dtype=None):
    """torch tensor / array -> contiguous numpy (no copy when possible)."""
    try:
        import torch
        if isinstance(t, torch.Tensor):
            t = t.detach().cpu()
            if t.dtype == torch.bfloat16:
                t = t.view(torch.int16)
            t = t.contiguous().numpy()
    except ImportError:  # pragma: no cover
        pass
    a = np.ascontiguousarray(t)
    if dtype is not None:
        a = np.ascontiguousarray(a.astype(dtype, copy=False))
    return a


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _features(x):
    """Return (numpy array, dtype code) keeping the exact stored values."""
    import torch
    if isinstance(x, torch.Tensor):
        if x.dtype == torch.bfloat16:
            return _np(x), X_BF16
        if x.dtype == torch.float32:
            return _np(x), X_F32
        return _np(x, np.float64), X_F64
    x = np.ascontiguousarray(x)
    if x.dtype == np.float32:
        return x, X_F32
    return np.ascontiguousarray(x, dtype=np.float64), X_F64


def _f64(t):
    import torch
    if isinstance(t, torch.Tensor):
        return np.ascontiguousarray(t.detach().cpu().to(torch.float64).numpy())
    return np.ascontiguousarray(np.asarray(t, dtype=np.float64))


class CSR:
    """The oracle's own destination-sorted CSR (reading A7)."""

    def __init__(self, n, row_ptr, col_src, edge_id, etype, in_deg, out_deg):
        self.n = n
        self.row_ptr, self.col_src, self.edge_id = row_ptr, col_src, edge_id
        self.etype, self.in_deg, self.out_deg = etype, in_deg, out_deg


class OracleRangeError(ValueError):
    def __init__(self, index):
        super().__init__(f"COO entry {index} out of range")
        self.index = index


def csr_build(n, src, dst, etype=None, num_etypes=1) -> CSR:
    src = _np(src, np.int32)
    dst = _np(dst, np.int32)
    et = None if etype is None else _np(etype, np.int32)
    e = src.shape[0]
    row_ptr = np.zeros(n + 1, np.int64)
    col_src = np.zeros(e, np.int32)
    edge_id = np.zeros(e, np.int32)
    etc = np.zeros(e, np.int32)
    ind = np.zeros(max(n, 1), np.int32)[:n]
    outd = np.zeros(max(n, 1), np.int32)[:n]
    bad = lib().oracle_csr_build(n, e, _ptr(src), _ptr(dst), _ptr(et), num_etypes,
                                 _ptr(row_ptr), _ptr(col_src), _ptr(edge_id), _ptr(etc),
                                 _ptr(ind), _ptr(outd))
    if bad >= 0:
        raise OracleRangeError(int(bad))
    return CSR(n, row_ptr, col_src, edge_id, etc, ind, outd)


def _rows(rows, n):
    if rows is None:
        return None, n
    r = _np(rows, np.int64)
    return r, r.shape[0]


def gcn(g: CSR, X, W, b=None, act=1, rows=None):
    x, xd = _features(X)
    W = _f64(W)
    f_in, f_out = W.shape
    bb = None if b is None else _f64(b)
    r, nr = _rows(rows, g.n)
    out = np.zeros((nr, f_out), np.float64)
    lib().oracle_gcn(g.n, _ptr(g.row_ptr), _ptr(g.col_src), _ptr(g.in_deg), _ptr(x), xd, f_in,
                     _ptr(W), f_out, _ptr(bb), act, _ptr(r), nr, _ptr(out))
    return out


def sage_mean(g: CSR, X, W, b=None, act=1, rows=None):
    x, xd = _features(X)
    W = _f64(W)
    f_out = W.shape[1]
    f_in = W.shape[0] // 2
    bb = None if b is None else _f64(b)
    r, nr = _rows(rows, g.n)
    out = np.zeros((nr, f_out), np.float64)
    lib().oracle_sage_mean(g.n, _ptr(g.row_ptr), _ptr(g.col_src), _ptr(g.in_deg), _ptr(x), xd, f_in,
                           _ptr(W), f_out, _ptr(bb), act, _ptr(r), nr, _ptr(out))
    return out


def gat(g: CSR, X, W, a_src, a_dst, slope=0.2, rows=None, want_alpha=False):
    x, xd = _features(X)
    W = _f64(W)
    f_in, f_out = W.shape
    a_s, a_d = _f64(a_src), _f64(a_dst)
    heads, hd = a_s.shape
    assert heads * hd == f_out
    r, nr = _rows(rows, g.n)
    out = np.zeros((nr, f_out), np.float64)
    alpha = np.zeros((g.col_src.shape[0], heads), np.float64) if (want_alpha and rows is None) else None
    lib().oracle_gat(g.n, _ptr(g.row_ptr), _ptr(g.col_src), _ptr(x), xd, f_in, _ptr(W), heads, hd,
                     _ptr(a_s), _ptr(a_d), float(slope), _ptr(r), nr, _ptr(out), _ptr(alpha))
    return (out, alpha) if want_alpha else out


def gated(g: CSR, H, W_type, W_ih, W_hh, b_ih, b_hh, num_etypes=None, rows=None):
    x, xd = _features(H)
    Wt = _f64(W_type)
    T, f, _ = Wt.shape
    if g.etype.size and int(g.etype.max()) >= T:
        raise ValueError(f"graph has edge types >= T = {T}")
    r, nr = _rows(rows, g.n)
    out = np.zeros((nr, f), np.float64)
    lib().oracle_gated(g.n, _ptr(g.row_ptr), _ptr(g.col_src), _ptr(g.etype), T, _ptr(x), xd, f,
                       _ptr(Wt), _ptr(_f64(W_ih)), _ptr(_f64(W_hh)), _ptr(_f64(b_ih)), _ptr(_f64(b_hh)),
                       _ptr(r), nr, _ptr(out))
    return out


def rgcn(g: CSR, H, W_type, W_self, b=None, act=1, rows=None):
    """R-GCN layer (oracle.c oracle_rgcn; reading A24)."""
    x, xd = _features(H)
    Wt = _f64(W_type)
    T, f, f_out = Wt.shape
    if g.etype.size and int(g.etype.max()) >= T:
        raise ValueError(f"graph has edge types >= T = {T}")
    Ws = _f64(W_self)
    bb = None if b is None else _f64(b)
    r, nr = _rows(rows, g.n)
    out = np.zeros((nr, f_out), np.float64)
    lib().oracle_rgcn(g.n, _ptr(g.row_ptr), _ptr(g.col_src), _ptr(g.etype), T, _ptr(x), xd, f, _ptr(Wt),
                      _ptr(Ws), f_out, _ptr(bb), act, _ptr(r), nr, _ptr(out))
    return out


def sage_lstm(g: CSR, X, W_ih, W_hh, b_ih, b_hh, W, b=None, act=1, rows=None):
    """GraphSAGE-LSTM layer (oracle.c oracle_sage_lstm; reading A25)."""
    x, xd = _features(X)
    Wi, Wh = _f64(W_ih), _f64(W_hh)
    f = Wi.shape[1]
    Wm = _f64(W)
    f_out = Wm.shape[1]
    assert Wi.shape == (4, f, f) and Wh.shape == (4, f, f) and Wm.shape[0] == 2 * f
    bb = None if b is None else _f64(b)
    r, nr = _rows(rows, g.n)
    out = np.zeros((nr, f_out), np.float64)
    lib().oracle_sage_lstm(g.n, _ptr(g.row_ptr), _ptr(g.col_src), _ptr(x), xd, f, _ptr(Wi), _ptr(Wh),
                           _ptr(_f64(b_ih)), _ptr(_f64(b_hh)), _ptr(Wm), f_out, _ptr(bb), act, _ptr(r), nr, _ptr(out))
    return out


def ggnn(g: CSR, H, W_e, b_e, W_ih, W_hh, b_ih, b_hh, act=1, agg="sum", rows=None):
    """Paper-form GGNN layer (oracle.c oracle_ggnn; reading A26): per-edge
    MLP on [H[u] || H[v]], sum (or max) over in-edges, GRUCell."""
    x, xd = _features(H)
    We = _f64(W_e)
    f = We.shape[1]
    assert We.shape == (2 * f, f)
    be = None if b_e is None else _f64(b_e)
    r, nr = _rows(rows, g.n)
    out = np.zeros((nr, f), np.float64)
    lib().oracle_ggnn(g.n, _ptr(g.row_ptr), _ptr(g.col_src), _ptr(x), xd, f, _ptr(We), _ptr(be), act,
                      1 if agg == "max" else 0, _ptr(_f64(W_ih)), _ptr(_f64(W_hh)), _ptr(_f64(b_ih)),
                      _ptr(_f64(b_hh)), _ptr(r), nr, _ptr(out))
    return out


def rel_err(y, y_ref) -> float:
    """Normwise inf-relative error max|y - y_ref| / max|y_ref| (reading A18).

    NaN/Inf anywhere -> inf.  If y_ref is all zero, the absolute error."""
    y = np.asarray(y, dtype=np.float64)
    y_ref = np.asarray(y_ref, dtype=np.float64)
    if not np.all(np.isfinite(y)):
        return float("inf")
    den = float(np.max(np.abs(y_ref))) if y_ref.size else 0.0
    num = float(np.max(np.abs(y - y_ref))) if y.size else 0.0
    return num / den if den > 0 else num


def row_err(y, y_ref, floor=1e-3):
    """Per-row diagnostic of SURVEY.md 8(c) (the "Error metric" row):
    max over rows v of ||y_v - yref_v||_inf / max(||yref_v||_inf, floor * ||yref||_inf).

    Returns (worst value, index of the worst row).  A row that is badly wrong
    but small next to the tensor's largest row shows up here and not in
    rel_err.  NaN/Inf anywhere -> (inf, -1); an empty tensor -> (0, -1)."""
    y = np.asarray(y, dtype=np.float64)
    y_ref = np.asarray(y_ref, dtype=np.float64)
    if not np.all(np.isfinite(y)):
        return float("inf"), -1
    if y_ref.size == 0:
        return 0.0, -1
    y2, r2 = y.reshape(y.shape[0], -1), y_ref.reshape(y_ref.shape[0], -1)
    glob = float(np.max(np.abs(r2)))
    if glob == 0.0:
        num = np.max(np.abs(y2 - r2), axis=1)
        return float(num.max()), int(num.argmax())
    den = np.maximum(np.max(np.abs(r2), axis=1), floor * glob)
    e = np.max(np.abs(y2 - r2), axis=1) / den
    return float(e.max()), int(e.argmax())
