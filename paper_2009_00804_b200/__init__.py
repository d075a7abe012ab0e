"""Python binding of libsaga.so -- the C ABI declared in include/saga.h.

Argument marshalling only: every step of the layer runs in the library's CUDA
kernels.  PyTorch is used for device memory and streams.  There is no CPU or
PyTorch fallback: importing this package raises if libsaga.so is missing, and
every call raises SagaError when the library reports a failure.

Entry points keep the C names: saga_graph_build, saga_graph_copy_csr,
saga_layer_workspace_bytes, saga_layer, saga_free (plus saga_abi_version and
saga_last_error).  ``layer()`` is a convenience wrapper that allocates the
output and workspace with torch and calls saga_layer.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsaga.so")

SAGA_OK, SAGA_EINVAL, SAGA_ERANGE, SAGA_ESHAPE, SAGA_EDTYPE, SAGA_ENOMEM, SAGA_ECUDA, SAGA_EUNSUPPORTED, \
    SAGA_EINTERNAL = range(9)
SAGA_F32, SAGA_BF16 = 0, 1
SAGA_GCN, SAGA_SAGE, SAGA_GAT, SAGA_GATED, SAGA_RGCN, SAGA_SAGE_LSTM, SAGA_GGNN = 0, 1, 2, 3, 4, 5, 6
SAGA_AGG_SUM, SAGA_AGG_MAX = 0, 1
SAGA_ACT_NONE, SAGA_ACT_RELU, SAGA_ACT_ELU = 0, 1, 2
MODELS = {"gcn": SAGA_GCN, "sage": SAGA_SAGE, "gat": SAGA_GAT, "gated": SAGA_GATED, "rgcn": SAGA_RGCN,
          "sage_lstm": SAGA_SAGE_LSTM, "ggnn": SAGA_GGNN}

# Every symbol include/saga.h declares (checked by tests/test_abi.py).
EXPORTS = ["saga_abi_version", "saga_graph_build", "saga_graph_info", "saga_graph_copy_csr",
           "saga_layer_workspace_bytes", "saga_layer", "saga_free", "saga_last_error",
           "saga_profile_enable", "saga_profile_filter", "saga_profile_count", "saga_profile_get",
           "saga_profile_trace_count", "saga_profile_trace_get"]


class SagaError(RuntimeError):
    def __init__(self, status, msg, first_bad_edge=-1):
        super().__init__(f"saga status {status}: {msg}")
        self.status = status
        self.first_bad_edge = first_bad_edge


class saga_tensor(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("dtype", ctypes.c_int32),
                ("rows", ctypes.c_int64), ("cols", ctypes.c_int64)]


class saga_layer_opts(ctypes.Structure):
    _fields_ = [("in_dim", ctypes.c_int32), ("out_dim", ctypes.c_int32), ("heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("act", ctypes.c_int32), ("leaky_slope", ctypes.c_float),
                ("aggregator", ctypes.c_int32), ("fused", ctypes.c_int32), ("workspace_zeroed", ctypes.c_int32)]


class saga_weights(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in
                ("W", "bias", "attn_src", "attn_dst", "W_type", "W_ih", "W_hh", "b_ih", "b_hh")]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(nvcc, sm_100a). There is no fallback path.")
    L = ctypes.CDLL(LIB_PATH)
    P, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    L.saga_abi_version.restype = ctypes.c_int
    L.saga_abi_version.argtypes = []
    L.saga_graph_build.restype = ctypes.c_int
    L.saga_graph_build.argtypes = [i32, i64, P, P, P, i32, P, ctypes.POINTER(P), ctypes.POINTER(i64)]
    L.saga_graph_info.restype = ctypes.c_int
    L.saga_graph_info.argtypes = [P, ctypes.POINTER(i32), ctypes.POINTER(i64), ctypes.POINTER(i32)]
    L.saga_graph_copy_csr.restype = ctypes.c_int
    L.saga_graph_copy_csr.argtypes = [P, P, P, P, P, P, P, P]
    L.saga_layer_workspace_bytes.restype = ctypes.c_int
    L.saga_layer_workspace_bytes.argtypes = [ctypes.c_int, P, ctypes.POINTER(saga_layer_opts),
                                             ctypes.POINTER(ctypes.c_size_t)]
    L.saga_layer.restype = ctypes.c_int
    L.saga_layer.argtypes = [ctypes.c_int, P, ctypes.POINTER(saga_tensor), ctypes.POINTER(saga_weights),
                             ctypes.POINTER(saga_tensor), ctypes.POINTER(saga_layer_opts), P, ctypes.c_size_t, P]
    L.saga_free.restype = None
    L.saga_free.argtypes = [P]
    L.saga_last_error.restype = ctypes.c_char_p
    L.saga_last_error.argtypes = []
    L.saga_profile_enable.restype = ctypes.c_int
    L.saga_profile_enable.argtypes = [ctypes.c_int]
    L.saga_profile_filter.restype = ctypes.c_int
    L.saga_profile_filter.argtypes = [ctypes.c_char_p]
    L.saga_profile_count.restype = ctypes.c_int32
    L.saga_profile_count.argtypes = []
    L.saga_profile_get.restype = ctypes.c_int
    L.saga_profile_get.argtypes = [i32, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(i64),
                                   ctypes.POINTER(ctypes.c_double)]
    L.saga_profile_trace_count.restype = ctypes.c_int32
    L.saga_profile_trace_count.argtypes = []
    L.saga_profile_trace_get.restype = ctypes.c_int
    L.saga_profile_trace_get.argtypes = [i32, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_double),
                                         ctypes.POINTER(ctypes.c_double)]
    return L


_lib = _load()


def saga_abi_version() -> int:
    return _lib.saga_abi_version()


def saga_profile_enable(enable: bool = True):
    """Per-kernel CUDA-event timing inside saga_layer (resets the counters)."""
    _check(_lib.saga_profile_enable(1 if enable else 0))


def saga_profile_filter(label=None):
    """Bracket only the launches labelled `label` (None: all); the others keep PDL."""
    _check(_lib.saga_profile_filter(label.encode() if label else None))


def saga_profile_read() -> dict:
    """{kernel name: (launches, total device ms)} since the last enable."""
    out = {}
    for i in range(_lib.saga_profile_count()):
        name, n, ms = ctypes.c_char_p(), ctypes.c_int64(), ctypes.c_double()
        _check(_lib.saga_profile_get(i, ctypes.byref(name), ctypes.byref(n), ctypes.byref(ms)))
        out[name.value.decode()] = (n.value, ms.value)
    return out


def saga_profile_trace() -> list:
    """[(label, start ms, end ms)] of every bracketed launch since the last
    enable, in launch order (times from the first bracket's start)."""
    out = []
    for i in range(_lib.saga_profile_trace_count()):
        name, t0, t1 = ctypes.c_char_p(), ctypes.c_double(), ctypes.c_double()
        _check(_lib.saga_profile_trace_get(i, ctypes.byref(name), ctypes.byref(t0), ctypes.byref(t1)))
        out.append((name.value.decode(), t0.value, t1.value))
    return out


def saga_last_error() -> str:
    return _lib.saga_last_error().decode()


def _check(status, first_bad=-1):
    if status != SAGA_OK:
        raise SagaError(status, saga_last_error(), first_bad)


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _dptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("device tensors required (the ABI takes device pointers)")
    if not t.is_contiguous():
        raise ValueError("contiguous tensors required")
    return ctypes.c_void_p(t.data_ptr())


def _dtype_code(t):
    if t.dtype == torch.float32:
        return SAGA_F32
    if t.dtype == torch.bfloat16:
        return SAGA_BF16
    raise ValueError(f"unsupported dtype {t.dtype}")


class Graph:
    """Owning handle of a built graph (freed by saga_free / close())."""

    def __init__(self, handle, n, e, t):
        self.handle = handle
        self.num_vertices, self.num_edges, self.num_etypes = n, e, t

    def close(self, sync=True):
        """saga_free is stream-ordered on the BUILD stream only (saga.h): layers
        may have used the graph on other streams, so wait for the device first.
        sync=False skips that wait: for a graph used only on its build stream
        (a serving loop on one stream), the stream-ordered free already follows
        every use, and the host does not block."""
        if self.handle:
            if sync:
                torch.cuda.synchronize()
            saga_free(self)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def csr(self, stream=None):
        return saga_graph_copy_csr(self, stream)


def saga_graph_build(num_vertices, src, dst, etype=None, num_etypes=1, stream=None) -> Graph:
    """COO (int32 device tensors) -> destination-sorted CSR (saga.h)."""
    e = src.numel()
    if dst.numel() != e or (etype is not None and etype.numel() != e):
        raise ValueError("src/dst/etype lengths differ")
    for t in (src, dst) + ((etype,) if etype is not None else ()):
        if t.dtype != torch.int32:
            raise ValueError("COO arrays must be int32")
    h = ctypes.c_void_p()
    bad = ctypes.c_int64(-1)
    st = _lib.saga_graph_build(int(num_vertices), e, _dptr(src), _dptr(dst), _dptr(etype),
                               int(num_etypes if etype is not None else 1), _stream(stream),
                               ctypes.byref(h), ctypes.byref(bad))
    _check(st, bad.value)
    n, ee, t = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int32()
    _check(_lib.saga_graph_info(h, ctypes.byref(n), ctypes.byref(ee), ctypes.byref(t)))
    return Graph(h, n.value, ee.value, t.value)


def saga_graph_copy_csr(g: Graph, stream=None) -> dict:
    dev = torch.device("cuda", torch.cuda.current_device())
    n, e = g.num_vertices, g.num_edges
    out = {"row_ptr": torch.empty(n + 1, dtype=torch.int64, device=dev),
           "col_src": torch.empty(e, dtype=torch.int32, device=dev),
           "edge_id": torch.empty(e, dtype=torch.int32, device=dev),
           "etype": torch.empty(e, dtype=torch.int32, device=dev),
           "in_deg": torch.empty(n, dtype=torch.int32, device=dev),
           "out_deg": torch.empty(n, dtype=torch.int32, device=dev)}
    _check(_lib.saga_graph_copy_csr(g.handle, *[_dptr(out[k]) for k in
                                                ("row_ptr", "col_src", "edge_id", "etype", "in_deg", "out_deg")],
                                    _stream(stream)))
    return out


def saga_free(g: Graph):
    _lib.saga_free(g.handle)


def make_opts(in_dim, out_dim, act, heads=0, head_dim=0, leaky_slope=0.2, aggregator=0,
              fused=0, workspace_zeroed=0) -> saga_layer_opts:
    return saga_layer_opts(int(in_dim), int(out_dim), int(heads), int(head_dim), int(act), float(leaky_slope),
                           int(aggregator), int(fused), int(workspace_zeroed))


def saga_layer_workspace_bytes(kind, g: Graph, opts: saga_layer_opts) -> int:
    b = ctypes.c_size_t()
    _check(_lib.saga_layer_workspace_bytes(int(kind), g.handle, ctypes.byref(opts), ctypes.byref(b)))
    return b.value


def _tensor(t):
    return saga_tensor(_dptr(t), _dtype_code(t), t.shape[0], t.shape[1] if t.dim() > 1 else 1)


def saga_layer(kind, g: Graph, features, weights: dict, out, opts: saga_layer_opts, workspace, stream=None):
    """One SAGA-NN layer on device tensors (saga.h); returns `out`."""
    w = saga_weights(**{k: _dptr(v) for k, v in weights.items() if v is not None})
    x_t, o_t = _tensor(features), _tensor(out)
    ws_ptr = _dptr(workspace) if workspace is not None and workspace.numel() else None
    ws_bytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
    _check(_lib.saga_layer(int(kind), g.handle, ctypes.byref(x_t), ctypes.byref(w), ctypes.byref(o_t),
                           ctypes.byref(opts), ws_ptr, ws_bytes, _stream(stream)))
    return out


class Layer:
    """Plans one layer once (opts, workspace) and runs it many times."""

    def __init__(self, kind, g: Graph, in_dim, out_dim, act, dtype, heads=0, head_dim=0, leaky_slope=0.2,
                 aggregator=0, fused=False):
        self.kind, self.g = MODELS.get(kind, kind), g
        self.opts = make_opts(in_dim, out_dim, act, heads, head_dim, leaky_slope,
                              {"sum": 0, "max": 1}.get(aggregator, aggregator), int(fused))
        nbytes = saga_layer_workspace_bytes(self.kind, g, self.opts)
        # zero-filled once and owned by this Layer: every completed call leaves
        # its ticket counters zero, so calls skip re-zeroing them
        self.workspace = torch.zeros(max(nbytes, 16), dtype=torch.uint8, device="cuda")
        self._filled = torch.cuda.Event()          # the first call's stream waits for the fill
        self._filled.record()
        self.opts.workspace_zeroed = 1
        self.out_shape = (g.num_vertices, out_dim)
        self.dtype = dtype

    def __call__(self, features, weights: dict, out=None, stream=None):
        if out is None:
            out = torch.empty(self.out_shape, dtype=self.dtype, device=features.device)
        if self._filled is not None:
            (stream or torch.cuda.current_stream()).wait_event(self._filled)
            self._filled = None
        return saga_layer(self.kind, self.g, features, weights, out, self.opts, self.workspace, stream)
