"""Error behaviour of the C ABI (include/saga.h "Errors").

CPU tests exercise the argument checks that run before any CUDA call; the
`gpu` tests exercise shape / dtype / alignment / workspace / unsupported
checks on real device buffers and the degenerate sizes (N = 0, E = 0)."""
import ctypes

import numpy as np
import pytest
import torch


@pytest.fixture(scope="module")
def saga():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2009_00804_b200 as s
    return s


def test_graph_build_argument_checks_cpu(saga):
    L = saga._lib
    h, bad = ctypes.c_void_p(), ctypes.c_int64(7)
    # E >= 2^31 is rejected before any device access
    assert L.saga_graph_build(5, 1 << 31, None, None, None, 1, None, ctypes.byref(h), ctypes.byref(bad)) == \
        saga.SAGA_EINVAL
    assert bad.value == -1 and not h.value
    # NULL src/dst with E > 0
    assert L.saga_graph_build(5, 3, None, None, None, 1, None, ctypes.byref(h), None) == saga.SAGA_EINVAL
    # negative sizes
    assert L.saga_graph_build(-1, 0, None, None, None, 1, None, ctypes.byref(h), None) == saga.SAGA_EINVAL
    # NULL out handle
    assert L.saga_graph_build(5, 0, None, None, None, 1, None, None, None) == saga.SAGA_EINVAL
    # N = 0 with E > 0: the lowest COO index (0) is out of range
    fake = ctypes.c_void_p(16)
    assert L.saga_graph_build(0, 4, fake, fake, None, 1, None, ctypes.byref(h), ctypes.byref(bad)) == \
        saga.SAGA_ERANGE
    assert bad.value == 0
    assert "range" in saga.saga_last_error()


def test_layer_argument_checks_cpu(saga):
    L = saga._lib
    opts = saga.make_opts(64, 16, saga.SAGA_ACT_RELU)
    n = ctypes.c_size_t()
    assert L.saga_layer(saga.SAGA_GCN, None, None, None, None, ctypes.byref(opts), None, 0, None) == saga.SAGA_EINVAL
    assert L.saga_layer_workspace_bytes(saga.SAGA_GCN, None, ctypes.byref(opts), ctypes.byref(n)) == saga.SAGA_EINVAL
    assert L.saga_graph_info(None, None, None, None) == saga.SAGA_EINVAL
    L.saga_free(None)  # NULL-safe
    assert saga.saga_last_error() != ""


# ---------------------------------------------------------------- GPU ----

def _graph(saga, n, src, dst, etype=None, T=1):
    dev = "cuda"
    s = torch.tensor(src, dtype=torch.int32, device=dev)
    d = torch.tensor(dst, dtype=torch.int32, device=dev)
    et = None if etype is None else torch.tensor(etype, dtype=torch.int32, device=dev)
    return saga.saga_graph_build(n, s, d, et, T)


@pytest.mark.gpu
def test_empty_vertex_set(saga):
    g = _graph(saga, 0, [], [])
    assert (g.num_vertices, g.num_edges) == (0, 0)
    lay = saga.Layer("gcn", g, 64, 64, saga.SAGA_ACT_RELU, torch.bfloat16)
    x = torch.empty(0, 64, dtype=torch.bfloat16, device="cuda")
    w = torch.zeros(64, 64, dtype=torch.bfloat16, device="cuda")
    y = lay(x, {"W": w})
    torch.cuda.synchronize()
    assert y.shape == (0, 64)


@pytest.mark.gpu
def test_no_edges_gives_bias_only(saga):
    """E = 0: every gather is empty (reading A12), so GCN = act(0 . W + b)."""
    g = _graph(saga, 5, [], [])
    b = torch.linspace(-1, 1, 64, device="cuda")
    lay = saga.Layer("gcn", g, 64, 64, saga.SAGA_ACT_RELU, torch.bfloat16)
    y = lay(torch.randn(5, 64, device="cuda").bfloat16(), {"W": torch.randn(64, 64, device="cuda").bfloat16(),
                                                            "bias": b})
    torch.cuda.synchronize()
    ref = torch.relu(b).bfloat16().expand(5, 64)
    assert torch.equal(y.cpu(), ref.cpu())


@pytest.mark.gpu
def test_layer_rejects_bad_arguments(saga):
    g = _graph(saga, 4, [0, 1, 2, 3], [1, 2, 3, 0])
    dev = "cuda"
    x = torch.randn(4, 64, device=dev).bfloat16()
    w = torch.randn(64, 64, device=dev).bfloat16()
    opts = saga.make_opts(64, 64, saga.SAGA_ACT_RELU)
    nbytes = saga.saga_layer_workspace_bytes(saga.SAGA_GCN, g, opts)
    ws = torch.empty(nbytes + 64, dtype=torch.uint8, device=dev)
    out = torch.empty(4, 64, dtype=torch.bfloat16, device=dev)

    def status(fn):
        with pytest.raises(saga.SagaError) as ei:
            fn()
        return ei.value.status

    # shape: features rows != N
    assert status(lambda: saga.saga_layer(saga.SAGA_GCN, g, x[:3], {"W": w}, out, opts, ws)) == saga.SAGA_ESHAPE
    # shape: out columns != out_dim
    assert status(lambda: saga.saga_layer(saga.SAGA_GCN, g, x, {"W": w}, out[:, :32].contiguous(), opts, ws)) == \
        saga.SAGA_ESHAPE
    # dtype: out dtype != features dtype
    assert status(lambda: saga.saga_layer(saga.SAGA_GCN, g, x, {"W": w}, out.float(), opts, ws)) == saga.SAGA_EDTYPE
    # workspace too small
    assert status(lambda: saga.saga_layer(saga.SAGA_GCN, g, x, {"W": w}, out, opts, ws[: nbytes - 256])) == \
        saga.SAGA_EINVAL
    # misaligned features pointer (2-byte offset)
    xb = torch.empty(4 * 64 + 1, dtype=torch.bfloat16, device=dev)
    xm = xb[1:].view(4, 64)
    assert status(lambda: saga.saga_layer(saga.SAGA_GCN, g, xm, {"W": w}, out, opts, ws)) == saga.SAGA_EINVAL
    # missing weight
    assert status(lambda: saga.saga_layer(saga.SAGA_GCN, g, x, {}, out, opts, ws)) == saga.SAGA_EINVAL
    # unsupported width
    o2 = saga.make_opts(64, 96, saga.SAGA_ACT_RELU)
    out96 = torch.empty(4, 96, dtype=torch.bfloat16, device=dev)
    ws96 = torch.empty(saga.saga_layer_workspace_bytes(saga.SAGA_GCN, g, o2), dtype=torch.uint8, device=dev)
    assert status(lambda: saga.saga_layer(saga.SAGA_GCN, g, x, {"W": w}, out96, o2, ws96)) == saga.SAGA_EUNSUPPORTED
    # GAT: heads must be 8 x 8, slope in [0, 1]
    x256 = torch.randn(4, 256, device=dev).bfloat16()
    wg = torch.randn(256, 64, device=dev).bfloat16()
    a = torch.randn(8, 8, device=dev)
    og = saga.make_opts(256, 64, saga.SAGA_ACT_ELU, heads=4, head_dim=16)
    ws4 = torch.empty(saga.saga_layer_workspace_bytes(saga.SAGA_GAT, g, og), dtype=torch.uint8, device=dev)
    assert status(lambda: saga.saga_layer(saga.SAGA_GAT, g, x256, {"W": wg, "attn_src": a, "attn_dst": a},
                                          out, og, ws4)) == saga.SAGA_EUNSUPPORTED
    og = saga.make_opts(256, 64, saga.SAGA_ACT_ELU, heads=8, head_dim=8, leaky_slope=1.5)
    wsg = torch.empty(saga.saga_layer_workspace_bytes(saga.SAGA_GAT, g, og), dtype=torch.uint8, device=dev)
    assert status(lambda: saga.saga_layer(saga.SAGA_GAT, g, x256, {"W": wg, "attn_src": a, "attn_dst": a},
                                          out, og, wsg)) == saga.SAGA_EUNSUPPORTED
    # nothing was enqueued by the failing calls: a valid call still works
    saga.saga_layer(saga.SAGA_GCN, g, x, {"W": w}, out, opts, ws)
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()


@pytest.mark.gpu
def test_gated_etype_out_of_range(saga):
    with pytest.raises(saga.SagaError) as ei:
        _graph(saga, 4, [0, 1, 2, 3], [1, 2, 3, 0], [0, 3, 4, 1], 4)
    assert ei.value.status == saga.SAGA_ERANGE and ei.value.first_bad_edge == 2


@pytest.mark.gpu
def test_ggnn_rejects_bad_arguments(saga):
    g = _graph(saga, 4, [0, 1, 2, 3], [1, 2, 3, 0])
    dev = "cuda"
    h = torch.randn(4, 128, device=dev)
    w = {"W": torch.randn(256, 128, device=dev), "W_ih": torch.randn(3, 128, 128, device=dev),
         "W_hh": torch.randn(3, 128, 128, device=dev), "b_ih": torch.randn(3, 128, device=dev),
         "b_hh": torch.randn(3, 128, device=dev)}
    out = torch.empty(4, 128, device=dev)

    def status(opts, ww=w, x=h, o=out):
        ws = torch.empty(saga.saga_layer_workspace_bytes(saga.SAGA_GGNN, g, opts), dtype=torch.uint8, device=dev)
        with pytest.raises(saga.SagaError) as ei:
            saga.saga_layer(saga.SAGA_GGNN, g, x, ww, o, opts, ws)
        return ei.value.status

    assert status(saga.make_opts(128, 128, saga.SAGA_ACT_RELU, aggregator=7)) == saga.SAGA_EUNSUPPORTED
    assert status(saga.make_opts(128, 128, saga.SAGA_ACT_ELU)) == saga.SAGA_EUNSUPPORTED
    assert status(saga.make_opts(128, 128, saga.SAGA_ACT_RELU), ww={k: v for k, v in w.items() if k != "W"}) == \
        saga.SAGA_EINVAL
    assert status(saga.make_opts(128, 128, saga.SAGA_ACT_RELU), x=h.bfloat16(), o=out.bfloat16()) == \
        saga.SAGA_EDTYPE
    # a valid call (bias omitted = 0) still works afterwards
    opts = saga.make_opts(128, 128, saga.SAGA_ACT_RELU, aggregator=saga.SAGA_AGG_MAX)
    ws = torch.empty(saga.saga_layer_workspace_bytes(saga.SAGA_GGNN, g, opts), dtype=torch.uint8, device=dev)
    saga.saga_layer(saga.SAGA_GGNN, g, h, w, out, opts, ws)
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()



@pytest.mark.gpu
def test_sage_fused_rejects_unsupported_widths(saga):
    g = _graph(saga, 4, [0, 1, 2, 3], [1, 2, 3, 0])
    x = torch.randn(4, 64, device="cuda").bfloat16()
    w = torch.randn(128, 64, device="cuda").bfloat16()
    out = torch.empty(4, 64, dtype=torch.bfloat16, device="cuda")
    opts = saga.make_opts(64, 64, saga.SAGA_ACT_RELU, fused=1)
    ws = torch.empty(saga.saga_layer_workspace_bytes(saga.SAGA_SAGE, g, opts), dtype=torch.uint8, device="cuda")
    with pytest.raises(saga.SagaError) as ei:
        saga.saga_layer(saga.SAGA_SAGE, g, x, {"W": w}, out, opts, ws)
    assert ei.value.status == saga.SAGA_EUNSUPPORTED


@pytest.mark.gpu
def test_gcn_fused_rejects_unsupported_widths(saga):
    g = _graph(saga, 4, [0, 1, 2, 3], [1, 2, 3, 0])
    x = torch.randn(4, 128, device="cuda").bfloat16()
    w = torch.randn(128, 64, device="cuda").bfloat16()
    out = torch.empty(4, 64, dtype=torch.bfloat16, device="cuda")
    opts = saga.make_opts(128, 64, saga.SAGA_ACT_RELU, fused=1)
    ws = torch.empty(saga.saga_layer_workspace_bytes(saga.SAGA_GCN, g, opts), dtype=torch.uint8, device="cuda")
    with pytest.raises(saga.SagaError) as ei:
        saga.saga_layer(saga.SAGA_GCN, g, x, {"W": w}, out, opts, ws)
    assert ei.value.status == saga.SAGA_EUNSUPPORTED
