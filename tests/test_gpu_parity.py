"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Bars (BASELINE.json north_star): CSR and degrees bit-exact; layer outputs
within normwise inf-relative error 1e-4 (fp32 configs) / 2e-2 (bf16 configs)
of the fp64 oracle (reading A18).
"""
import numpy as np
import pytest
import torch

import oracle
import workloads as W
from tests import harness as H
from tests import zoo

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def saga():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2009_00804_b200 as s
    return s


DEV = "cuda"


def _csr_check(saga, n, s, d, et=None, T=1):
    st, dt = torch.from_numpy(np.ascontiguousarray(s)), torch.from_numpy(np.ascontiguousarray(d))
    ett = None if et is None else torch.from_numpy(np.ascontiguousarray(et))
    g = saga.saga_graph_build(n, st.to(DEV), dt.to(DEV), None if ett is None else ett.to(DEV), T)
    got = {k: v.cpu().numpy() for k, v in g.csr().items()}
    og = oracle.csr_build(n, s, d, et, T)
    np.testing.assert_array_equal(got["row_ptr"], og.row_ptr)
    np.testing.assert_array_equal(got["col_src"], og.col_src)
    np.testing.assert_array_equal(got["edge_id"], og.edge_id)
    np.testing.assert_array_equal(got["etype"], og.etype)
    np.testing.assert_array_equal(got["in_deg"], og.in_deg)
    np.testing.assert_array_equal(got["out_deg"], og.out_deg)


@pytest.mark.parametrize("name,n,s,d", zoo.zoo(include_big=True), ids=lambda x: x if isinstance(x, str) else "")
def test_csr_bitexact_zoo(saga, name, n, s, d):
    _csr_check(saga, n, s, d)
    et = (np.arange(s.shape[0]) % 3).astype(np.int32)
    _csr_check(saga, n, s, d, et, 3)


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4", "C5"])
def test_csr_bitexact_configs(saga, cfg):
    c = W.CONFIGS[cfg]
    s, d, et = W.make_graph(c, DEV)
    g = saga.saga_graph_build(c.n, s, d, et, c.num_etypes)
    got = g.csr()
    og = oracle.csr_build(c.n, s.cpu(), d.cpu(), None if et is None else et.cpu(), c.num_etypes)
    assert torch.equal(got["row_ptr"].cpu(), torch.from_numpy(og.row_ptr))
    assert torch.equal(got["col_src"].cpu(), torch.from_numpy(og.col_src))
    assert torch.equal(got["edge_id"].cpu(), torch.from_numpy(og.edge_id))
    assert torch.equal(got["in_deg"].cpu(), torch.from_numpy(og.in_deg))
    assert torch.equal(got["out_deg"].cpu(), torch.from_numpy(og.out_deg))
    if et is not None:
        assert torch.equal(got["etype"].cpu(), torch.from_numpy(og.etype))


def test_range_error_reports_lowest_index(saga):
    s = torch.tensor([0, 1, 2, 9, 1, -1], dtype=torch.int32, device=DEV)
    d = torch.tensor([1, 2, 0, 0, 7, 0], dtype=torch.int32, device=DEV)
    with pytest.raises(saga.SagaError) as ei:
        saga.saga_graph_build(3, s, d)
    assert ei.value.status == saga.SAGA_ERANGE and ei.value.first_bad_edge == 3
    et = torch.tensor([0, 0, 5], dtype=torch.int32, device=DEV)
    with pytest.raises(saga.SagaError) as ei:
        saga.saga_graph_build(3, s[:3], d[:3], et, 2)
    assert ei.value.first_bad_edge == 2


# ------------------------------------------------------------ layer zoo ----

def _zoo_inputs(model, n, s, d, seed):
    """Small-graph inputs for each model at supported widths."""
    gen = torch.Generator().manual_seed(seed)
    r = lambda *sh, sc=1.0: torch.randn(*sh, generator=gen) * sc
    if model == "gcn_bf16":
        return {"X": r(n, 64).bfloat16(), "W": r(64, 64, sc=0.2).bfloat16(), "b": r(64, sc=0.1)}
    if model == "gcn_f32":
        return {"X": r(n, 64), "W": r(64, 16, sc=0.2), "b": r(16, sc=0.1)}
    if model == "sage":
        return {"X": r(n, 128).bfloat16(), "W1": r(256, 128, sc=0.1).bfloat16(), "W2": r(256, 64, sc=0.1).bfloat16()}
    if model == "gat":
        return {"X": r(n, 256).bfloat16(), "W": r(256, 64, sc=0.1).bfloat16(), "a_src": r(8, 8, sc=0.5),
                "a_dst": r(8, 8, sc=0.5)}
    if model == "gated":
        b = 1 / np.sqrt(128)
        u = lambda *sh: (torch.rand(*sh, generator=gen) * 2 - 1) * b
        return {"H": r(n, 128), "W_type": u(4, 128, 128), "W_ih": u(3, 128, 128), "W_hh": u(3, 128, 128),
                "b_ih": u(3, 128), "b_hh": u(3, 128)}
    if model == "sage_lstm":
        b = 1 / np.sqrt(128)
        u = lambda *sh: (torch.rand(*sh, generator=gen) * 2 - 1) * b
        return {"X": r(n, 128).bfloat16(), "W_ih": u(4, 128, 128).bfloat16(), "W_hh": u(4, 128, 128).bfloat16(),
                "b_ih": u(4, 128), "b_hh": u(4, 128), "W": r(256, 128, sc=0.1).bfloat16(), "b": u(128)}
    if model == "rgcn":
        b = 1 / np.sqrt(128)
        u = lambda *sh: (torch.rand(*sh, generator=gen) * 2 - 1) * b
        return {"H": r(n, 128), "W_type": u(4, 128, 128), "W_self": u(128, 128), "b": u(128)}
    if model in ("ggnn", "ggnn_max"):
        b = 1 / np.sqrt(128)
        u = lambda *sh: (torch.rand(*sh, generator=gen) * 2 - 1) * b
        return {"H": r(n, 128), "W_e": u(256, 128), "b_e": u(128), "W_ih": u(3, 128, 128), "W_hh": u(3, 128, 128),
                "b_ih": u(3, 128), "b_hh": u(3, 128)}


def _zoo_cfg(model, n, e):
    base = {"gcn_bf16": W.Config("z", "gcn", "er", n, e, False, False, "bf16", (64, 64)),
            "gcn_f32": W.Config("z", "gcn", "er", n, e, False, False, "f32", (64, 16)),
            "sage": W.Config("z", "sage", "er", n, e, False, False, "bf16", (128, 128, 64)),
            "gat": W.Config("z", "gat", "er", n, e, False, False, "bf16", (256, 64), heads=8),
            "gated": W.Config("z", "gated", "er", n, e, False, False, "f32", (128, 128), num_etypes=4),
            "rgcn": W.Config("z", "rgcn", "er", n, e, False, False, "f32", (128, 128), num_etypes=4),
            "sage_lstm": W.Config("z", "sage_lstm", "er", n, e, False, False, "bf16", (128, 128)),
            "ggnn": W.Config("z", "ggnn", "er", n, e, False, False, "f32", (128, 128), extra={"agg": "sum"}),
            "ggnn_max": W.Config("z", "ggnn", "er", n, e, False, False, "f32", (128, 128), extra={"agg": "max"})}
    return base[model]


ZOO = [z for z in zoo.zoo(include_big=True) if z[1] > 0]
MODELS = ["gcn_bf16", "gcn_f32", "sage", "gat", "gated", "rgcn", "sage_lstm", "ggnn", "ggnn_max"]


@pytest.mark.parametrize("model", MODELS)
@pytest.mark.parametrize("name,n,s,d", ZOO, ids=lambda x: x if isinstance(x, str) else "")
@pytest.mark.parametrize("loops", [False, True])
def test_layer_zoo(saga, model, name, n, s, d, loops):
    if loops:
        s, d = zoo.with_self_loops(n, s, d)
    cfg = _zoo_cfg(model, n, s.shape[0])
    x = _zoo_inputs(model, n, s, d, 7)
    x["src"], x["dst"] = torch.from_numpy(s), torch.from_numpy(d)
    if model in ("gated", "rgcn"):
        x["etype"] = torch.from_numpy((np.arange(s.shape[0]) * 7 % 4).astype(np.int32))
    dx = H.dev_inputs(x, DEV)
    g = H.gpu_graph(saga, cfg, dx)
    outs, _ = H.gpu_step(saga, cfg, g, dx)
    torch.cuda.synchronize()
    og = H.oracle_graph(oracle, cfg, x)
    refs = H.oracle_step(oracle, cfg, og, x, layer_inputs=[None, outs[0].cpu()] if model == "sage" else None)
    tol = H.TOL[cfg.dtype]
    for i, (y, ref) in enumerate(zip(outs, refs)):
        H.check(y, ref, tol, f"{model}/{name}/loops={loops}/layer{i}")


# ----------------------------------------------------- configured steps ----

def _config_check(saga, cfg, rows_k=None):
    d = W.make_inputs(cfg, DEV)
    g = H.gpu_graph(saga, cfg, d)
    outs, layers = H.gpu_step(saga, cfg, g, d)
    outs2, _ = H.gpu_step(saga, cfg, g, d, layers)           # determinism: bitwise equal
    torch.cuda.synchronize()
    for a, b in zip(outs, outs2):
        assert torch.equal(a, b)
    og = H.oracle_graph(oracle, cfg, d)
    rows = None if rows_k is None else H.sample_rows(og, rows_k)
    tol = H.TOL[cfg.dtype]
    li = [None, outs[0].cpu()] if cfg.model == "sage" else None
    refs = H.oracle_step(oracle, cfg, og, d, rows=rows, layer_inputs=li)
    for i, (y, ref) in enumerate(zip(outs, refs)):
        yy = H.to_np(y if rows is None else y[torch.from_numpy(rows).to(y.device)])
        H.check(yy, ref, tol, f"{cfg.name}/layer{i}")
    if cfg.model == "sage":   # end to end: the oracle chains its own fp64 H1 (A19)
        ref_e2e = H.oracle_step(oracle, cfg, og, d, rows=rows)[1]
        yy = H.to_np(outs[1] if rows is None else outs[1][torch.from_numpy(rows).to(DEV)])
        H.check(yy, ref_e2e, tol, f"{cfg.name}/end-to-end")


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4", "C6", "C8"])
def test_config_full(saga, cfg):
    _config_check(saga, W.CONFIGS[cfg])


@pytest.mark.parametrize("cfg", ["C2", "C3", "C4", "C5", "C6", "C7", "C8"])
def test_config_scaled_ragged(saga, cfg):
    """Same recipe at a size that is not a multiple of any tile (ragged tails)."""
    c = W.CONFIGS[cfg]
    _config_check(saga, W.scaled(c, 3000 if cfg != "C5" else 5000, 40000, cfg + "r"))


def test_c5_full_sampled(saga):
    """C5 at full size (launch config the bench times), sampled rows incl. hubs."""
    _config_check(saga, W.CONFIGS["C5"], rows_k=3000)


def test_c7_full_sampled(saga):
    """C7 (GraphSAGE-LSTM, NEXT-2) at full size, sampled rows incl. the 16 longest sequences."""
    _config_check(saga, W.CONFIGS["C7"], rows_k=2000)


def test_relabel_invariance_gpu(saga):
    cfg = W.scaled(W.CONFIGS["C3"], 2000, 30000, "rl")
    d = W.make_inputs(cfg, "cpu")
    perm = torch.randperm(cfg.n, generator=torch.Generator().manual_seed(1)).to(torch.int32)
    d2 = dict(d)
    d2["src"], d2["dst"] = perm[d["src"].long()], perm[d["dst"].long()]
    X2 = torch.empty_like(d["X"])
    X2[perm.long()] = d["X"]
    d2["X"] = X2
    a, b = H.dev_inputs(d, DEV), H.dev_inputs(d2, DEV)
    ya = H.gpu_step(__import__("paper_2009_00804_b200"), cfg, H.gpu_graph(saga, cfg, a), a)[0][0]
    yb = H.gpu_step(saga, cfg, H.gpu_graph(saga, cfg, b), b)[0][0]
    err = oracle.rel_err(H.to_np(yb[perm.long().to(DEV)]), H.to_np(ya))
    assert err <= 2e-2


@pytest.mark.parametrize("model", ["gated", "rgcn"])
@pytest.mark.parametrize("T,types", [(1, "none"), (1, "zeros"), (2, "mod"), (3, "skew"), (4, "one_hot_hub")])
def test_typed_view(saga, model, T, types):
    """The typed gathers run over the graph's (destination, type) view: every
    T <= 4, graphs without edge types (T = 1, plain CSR), a type that only a
    few vertices receive, and a hub whose in-edges are all of one type."""
    n = 3001
    rng = np.random.default_rng(5)
    s = rng.integers(0, n, 40000).astype(np.int32)
    d = np.minimum(rng.zipf(1.6, 40000) - 1, n - 1).astype(np.int32)  # power-law in-degree
    d[:5000] = 17                                                        # one hub
    e = s.shape[0]
    if types == "none":
        et = None
    elif types == "zeros":
        et = np.zeros(e, np.int32)
    elif types == "mod":
        et = (np.arange(e) % 2).astype(np.int32)
    elif types == "skew":
        et = np.where(np.arange(e) % 97 == 0, 2, np.arange(e) % 2).astype(np.int32)
    else:
        et = (np.arange(e) % 4).astype(np.int32)
        et[d == 17] = 3
    cfg = W.Config("tv", model, "er", n, e, False, False, "f32", (128, 128), num_etypes=T)
    x = _zoo_inputs(model, n, s, d, 11)
    x["W_type"] = x["W_type"][:T].contiguous()
    x["src"], x["dst"] = torch.from_numpy(s), torch.from_numpy(d)
    if et is not None:
        x["etype"] = torch.from_numpy(et)
    dx = H.dev_inputs(x, DEV)
    g = H.gpu_graph(saga, cfg, dx)
    outs, _ = H.gpu_step(saga, cfg, g, dx)
    torch.cuda.synchronize()
    og = H.oracle_graph(oracle, cfg, x)
    refs = H.oracle_step(oracle, cfg, og, x)
    H.check(outs[0], refs[0], H.TOL["f32"], f"{model} T={T} {types}")


@pytest.mark.parametrize("hub", [1500, 6000, 20000])
@pytest.mark.parametrize("agg", ["sum", "max"])
@pytest.mark.parametrize("relu", [True, False])
def test_ggnn_aggregators(saga, agg, relu, hub):
    """NEXT-4 paper-form GGNN: both Gather reductions, with and without the
    edge-MLP ReLU, on a power-law graph (zipf in-degrees: vertex 0 already
    receives ~14K edges) with one more hub of `hub` in-edges, split across
    tasks.  With ReLU and sum the hubs' messages grow linearly with their
    in-degree (every term >= 0; |m| ~ 1.5e4 at 6K in-edges): rows with
    in-degree >= 256 run ApplyVertex in fp64 (gru_f64.cu), whose error is set
    by the fp32 storage of m (~4e-6); the split-TF32 tensor-core GEMM
    (fp32 accumulator) misses the fp32 bar on such rows (1.35e-4 at 6K,
    scripts/tc_accum_probe.py)."""
    n = 2500
    rng = np.random.default_rng(7)
    s = rng.integers(0, n, 30000).astype(np.int32)
    d = np.minimum(rng.zipf(1.7, 30000) - 1, n - 1).astype(np.int32)
    d[:hub] = 11
    x = _zoo_inputs("ggnn", n, s, d, 3)
    dx = H.dev_inputs(dict(x, src=torch.from_numpy(s), dst=torch.from_numpy(d)), DEV)
    g = saga.saga_graph_build(n, dx["src"], dx["dst"])
    lay = saga.Layer("ggnn", g, 128, 128, saga.SAGA_ACT_RELU if relu else saga.SAGA_ACT_NONE, torch.float32,
                     aggregator=agg)
    w = {"W": dx["W_e"], "bias": dx["b_e"], "W_ih": dx["W_ih"], "W_hh": dx["W_hh"], "b_ih": dx["b_ih"],
         "b_hh": dx["b_hh"]}
    y = lay(dx["H"], w)
    y2 = lay(dx["H"], w)
    torch.cuda.synchronize()
    assert torch.equal(y, y2)
    og = oracle.csr_build(n, s, d)
    ref = oracle.ggnn(og, x["H"], x["W_e"], x["b_e"], x["W_ih"], x["W_hh"], x["b_ih"], x["b_hh"],
                      act=1 if relu else 0, agg=agg)
    err, _ = H.check(y, ref, H.TOL["f32"], f"ggnn {agg} relu={relu} hub={hub}")
    # heavy rows (fp64 ApplyVertex) are as accurate as fp32 storage of m allows
    assert err <= 2e-5, f"ggnn {agg} relu={relu} hub={hub}: {err:.3e} above the fp64-path level"


def test_gated_hub70k_fp64_level(saga):
    """The gated layer's worst zoo case (a 70K-in-edge hub whose per-type sums
    reach |S| ~ 130): the hub runs ApplyVertex in fp64, so the layer error is
    below the fp32 FFMA level measured in round 1 (2.0e-5)."""
    name, n, s, d = [z for z in zoo.zoo(include_big=True) if z[0] == "hub70k"][0]
    cfg = _zoo_cfg("gated", n, s.shape[0])
    x = _zoo_inputs("gated", n, s, d, 7)
    x["src"], x["dst"] = torch.from_numpy(s), torch.from_numpy(d)
    x["etype"] = torch.from_numpy((np.arange(s.shape[0]) * 7 % 4).astype(np.int32))
    dx = H.dev_inputs(x, DEV)
    g = H.gpu_graph(saga, cfg, dx)
    outs, _ = H.gpu_step(saga, cfg, g, dx)
    torch.cuda.synchronize()
    og = H.oracle_graph(oracle, cfg, x)
    ref = H.oracle_step(oracle, cfg, og, x)[0]
    err, _ = H.check(outs[0], ref, H.TOL["f32"], "gated hub70k")
    assert err <= 2e-5, f"gated hub70k: {err:.3e}"


def _fused(cfg, n=None, m=None, name=None):
    c = W.scaled(cfg, n or cfg.n, m or cfg.m, name or cfg.name + "f")
    c.extra["fused"] = True
    return c


@pytest.mark.parametrize("size", ["full", "ragged", "tiny"])
def test_sage_fused_next1(saga, size):
    """NEXT-1: GraphSAGE-mean Gather fused with the tcgen05 concat-GEMM (one
    kernel per layer) at C2 full size, a ragged size (last tile partial,
    hubs split across warps) and a graph smaller than one tile."""
    c = W.CONFIGS["C2"]
    cfg = {"full": _fused(c), "ragged": _fused(c, 3001, 40000), "tiny": _fused(c, 77, 300)}[size]
    _config_check(saga, cfg)


@pytest.mark.parametrize("name,n,s,d", ZOO, ids=lambda x: x if isinstance(x, str) else "")
def test_sage_fused_zoo(saga, name, n, s, d):
    cfg = W.Config("zf", "sage", "er", n, s.shape[0], False, False, "bf16", (128, 128, 64), extra={"fused": True})
    x = _zoo_inputs("sage", n, s, d, 7)
    x["src"], x["dst"] = torch.from_numpy(s), torch.from_numpy(d)
    dx = H.dev_inputs(x, DEV)
    g = H.gpu_graph(saga, cfg, dx)
    outs, _ = H.gpu_step(saga, cfg, g, dx)
    torch.cuda.synchronize()
    og = H.oracle_graph(oracle, cfg, x)
    refs = H.oracle_step(oracle, cfg, og, x, layer_inputs=[None, outs[0].cpu()])
    for i, (y, ref) in enumerate(zip(outs, refs)):
        H.check(y, ref, H.TOL["bf16"], f"fused sage/{name}/layer{i}")


def _random_graph(seed):
    """Random multigraph with a mix of degree shapes: uniform, power-law with
    a hub, many empty rows, duplicates and self-loops."""
    rng = np.random.default_rng(seed)
    n = int(rng.choice([1, 2, 17, 63, 64, 65, 129, 700, 2500]))
    e = int(rng.integers(0, 12 * n + 1))
    kind = seed % 3
    s = rng.integers(0, n, e).astype(np.int32)
    if kind == 0:
        d = rng.integers(0, n, e).astype(np.int32)
    elif kind == 1:
        d = np.minimum(rng.zipf(1.5, e) - 1, n - 1).astype(np.int32)
    else:
        d = rng.integers(0, max(1, n // 4), e).astype(np.int32)   # 3/4 of the rows empty
    return n, s, d


@pytest.mark.parametrize("size", ["full_sampled", "ragged", "tiny"])
def test_gcn_fused_next1(saga, size):
    """NEXT-1 for C5: the GCN aggregation fused with its tcgen05 GEMM in SAGA
    order (one kernel), at C5 full size on sampled rows
    (hubs included; the launch configuration the bench times), a ragged size
    (last tile partial, hubs split across warps, dynamic tiles) and a graph
    smaller than one tile."""
    c = W.CONFIGS["C5"]
    if size == "full_sampled":
        _config_check(saga, _fused(c), rows_k=3000)
    else:
        _config_check(saga, {"ragged": _fused(c, 5000, 40000), "tiny": _fused(c, 77, 300)}[size])


@pytest.mark.parametrize("fo", [64, 128, 256])
@pytest.mark.parametrize("name,n,s,d", ZOO, ids=lambda x: x if isinstance(x, str) else "")
@pytest.mark.parametrize("loops", [False, True])
def test_gcn_fused_zoo(saga, name, n, s, d, loops, fo):
    """The zoo (empty rows, stars, the 70K-edge hub, non-multiples of the tile)
    through the fused GCN at every supported output width."""
    if fo != 256 and name not in ("hub70k", "multigraph333"):
        pytest.skip("narrow outputs: two zoo graphs")
    if loops:
        s, d = zoo.with_self_loops(n, s, d)
    _gcn_fused_case(saga, n, s, d, fo, 7, f"fused gcn/{name}/loops={loops}/fo={fo}")


def _gcn_fused_case(saga, n, s, d, fo, seed, label):
    gen = torch.Generator().manual_seed(seed)
    r = lambda *sh, sc=1.0: torch.randn(*sh, generator=gen) * sc
    x = {"X": r(n, 256).bfloat16(), "W": r(256, fo, sc=0.1).bfloat16(), "b": r(fo, sc=0.1)}
    x["src"], x["dst"] = torch.from_numpy(s), torch.from_numpy(d)
    cfg = W.Config("zg", "gcn", "er", n, s.shape[0], False, False, "bf16", (256, fo), extra={"fused": True})
    dx = H.dev_inputs(x, DEV)
    g = H.gpu_graph(saga, cfg, dx)
    outs, _ = H.gpu_step(saga, cfg, g, dx)
    torch.cuda.synchronize()
    og = H.oracle_graph(oracle, cfg, x)
    ref = H.oracle_step(oracle, cfg, og, x)[0]
    H.check(outs[0], ref, H.TOL["bf16"], label)


def test_gcn_fused_no_edges(saga):
    """Vertices without any in-edge (dinv = 0): every output row is act(bias);
    three tiles, the last one partial, no source chunk is ever loaded."""
    n = 300
    e = np.zeros(0, dtype=np.int32)
    _gcn_fused_case(saga, n, e, e, 256, 3, "fused gcn/no edges")


@pytest.mark.parametrize("seed", range(40))
def test_gcn_fused_random_graphs(saga, seed):
    n, s, d = _random_graph(1000 * seed + 7)
    _gcn_fused_case(saga, n, s, d, [256, 128, 64][seed % 3], seed, f"fused gcn/seed {seed} (n={n}, e={s.shape[0]})")


@pytest.mark.parametrize("seed", range(40))
@pytest.mark.parametrize("model", ["gcn_bf16", "gcn_f32", "sage", "sage_fused", "gat", "gated", "rgcn", "ggnn",
                                   "ggnn_max", "sage_lstm"])
def test_random_graphs(saga, model, seed):
    """Randomised sweep over graph shapes (1..2500 vertices, 0..12 N edges,
    uniform / power-law / mostly-empty) for every model, against the oracle;
    covers the row-per-warp and merge-path paths, task boundaries at every
    offset, and the typed view with types that some vertices never see."""
    if model == "sage_lstm" and seed >= 10:
        pytest.skip("the fp64 LSTM oracle is slow; 10 seeds")
    n, s, d = _random_graph(1000 * seed + 7)
    fused = model == "sage_fused"
    if fused:
        model = "sage"
    cfg = _zoo_cfg(model, n, s.shape[0])
    if fused:
        cfg.extra["fused"] = True
    x = _zoo_inputs(model, n, s, d, seed)
    x["src"], x["dst"] = torch.from_numpy(s), torch.from_numpy(d)
    if model in ("gated", "rgcn"):
        x["etype"] = torch.from_numpy((np.random.default_rng(seed).integers(0, 4, s.shape[0])).astype(np.int32))
    dx = H.dev_inputs(x, DEV)
    g = H.gpu_graph(saga, cfg, dx)
    outs, _ = H.gpu_step(saga, cfg, g, dx)
    torch.cuda.synchronize()
    og = H.oracle_graph(oracle, cfg, x)
    refs = H.oracle_step(oracle, cfg, og, x, layer_inputs=[None, outs[0].cpu()] if model == "sage" else None)
    tol = H.TOL[cfg.dtype]
    for i, (y, ref) in enumerate(zip(outs, refs)):
        H.check(y, ref, tol, f"{model}/seed {seed} (n={n}, e={s.shape[0]})/layer{i}")


def _named(cfg):
    """A BASELINE config by name; "C5f" / "C2f": the same through the NEXT-1 fused kernels."""
    if cfg.endswith("f"):
        return _fused(W.CONFIGS[cfg[:-1]])
    return W.CONFIGS[cfg]


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4", "C5f", "C6", "C7", "C8"])
def test_cuda_graph_replay_matches_eager(saga, cfg):
    """bench.py times the step captured in a CUDA graph: the replayed step is
    bit-identical to the eagerly launched one (same kernels, deterministic;
    C7 also forks its batches onto the library stream inside the capture)."""
    c = _named(cfg)
    if c.n > 200000:
        c = W.scaled(c, 20000, 200000, cfg + "g")
    d = W.make_inputs(c, DEV)
    g = H.gpu_graph(saga, c, d)
    outs, layers = H.gpu_step(saga, c, g, d)
    torch.cuda.synchronize()
    ref = [o.clone() for o in outs]
    for o in outs:
        o.zero_()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        H.gpu_step(saga, c, g, d, layers, outs)
    graph.replay()
    torch.cuda.synchronize()
    for a, b in zip(outs, ref):
        assert torch.equal(a, b)


@pytest.mark.parametrize("cfg", ["C2", "C3", "C4", "C5", "C5f", "C6", "C7", "C8"])
def test_programmatic_launch_matches_serialised(saga, cfg):
    """Inside a layer call every kernel after the first is a programmatic
    dependent launch (internal.cuh); with per-kernel profiling on, the library
    launches them fully serialised.  Both give bit-identical outputs (each
    kernel waits for its predecessor before reading its output)."""
    c = _named(cfg)
    if c.n > 200000:
        c = W.scaled(c, 30000, 400000, cfg + "p")
    d = W.make_inputs(c, DEV)
    g = H.gpu_graph(saga, c, d)
    outs, layers = H.gpu_step(saga, c, g, d)          # programmatic
    torch.cuda.synchronize()
    ref = [o.clone() for o in outs]
    for o in outs:
        o.zero_()
    saga.saga_profile_enable(True)                    # serialised (event pairs between kernels)
    try:
        H.gpu_step(saga, c, g, d, layers, outs)
        torch.cuda.synchronize()
    finally:
        saga.saga_profile_enable(False)
    for a, b in zip(outs, ref):
        assert torch.equal(a, b)
    for _ in range(3):                                # back-to-back programmatic steps
        H.gpu_step(saga, c, g, d, layers, outs)
    torch.cuda.synchronize()
    for a, b in zip(outs, ref):
        assert torch.equal(a, b)


@pytest.mark.parametrize("cfg", ["C2", "C3", "C4", "C5", "C5f", "C6", "C7", "C8"])
def test_workspace_zeroed_contract(saga, cfg):
    """opts.workspace_zeroed (include/saga.h): with 0 the library zeroes the
    ticket counters itself (a garbage-filled workspace gives the same output);
    every completed call leaves them zero, so the next call may pass 1."""
    c = _named(cfg)
    if c.n > 200000:
        c = W.scaled(c, 30000, 400000, cfg + "w")
    d = W.make_inputs(c, DEV)
    g = H.gpu_graph(saga, c, d)
    outs, layers = H.gpu_step(saga, c, g, d)          # Layer: zero-filled workspace, flag 1
    torch.cuda.synchronize()
    ref = [o.clone() for o in outs]
    for lay in layers:
        lay.workspace.fill_(0xAB)
        lay.opts.workspace_zeroed = 0
    H.gpu_step(saga, c, g, d, layers, outs)
    torch.cuda.synchronize()
    for a, b in zip(outs, ref):
        assert torch.equal(a, b)
    for lay in layers:
        lay.opts.workspace_zeroed = 1                 # left zero by the call above
    for o in outs:
        o.zero_()
    H.gpu_step(saga, c, g, d, layers, outs)
    torch.cuda.synchronize()
    for a, b in zip(outs, ref):
        assert torch.equal(a, b)


@pytest.mark.parametrize("model", MODELS)
def test_workspace_reuse_across_graphs(saga, model):
    """saga.h: every completed call leaves the workspace's ticket counters
    zero, so a workspace may be reused with workspace_zeroed = 1 for ANOTHER
    graph with more tasks (round-1 advisor: the LSTM queue head used to sit
    in a counter slot that a larger graph uses as a ticket)."""
    n = 3000
    rng = np.random.default_rng(21)
    small_s, small_d = rng.integers(0, n, 40).astype(np.int32), rng.integers(0, n, 40).astype(np.int32)
    big_s = rng.integers(0, n, 60000).astype(np.int32)
    big_d = np.minimum(rng.zipf(1.6, 60000) - 1, n - 1).astype(np.int32)
    cfg = _zoo_cfg(model, n, big_s.shape[0])
    x = _zoo_inputs(model, n, big_s, big_d, 5)
    et = lambda e: torch.from_numpy((np.arange(e) % 4).astype(np.int32)).to(DEV)
    typed = model in ("gated", "rgcn")
    gs = saga.saga_graph_build(n, torch.from_numpy(small_s).to(DEV), torch.from_numpy(small_d).to(DEV),
                               et(40) if typed else None, 4 if typed else 1)
    gb = saga.saga_graph_build(n, torch.from_numpy(big_s).to(DEV), torch.from_numpy(big_d).to(DEV),
                               et(60000) if typed else None, 4 if typed else 1)
    dx = H.dev_inputs(dict(x, src=torch.from_numpy(big_s), dst=torch.from_numpy(big_d)), DEV)
    if typed:
        dx["etype"] = et(60000)
    fresh, layers = H.gpu_step(saga, cfg, gb, dx)                 # reference: own zero-filled workspace
    torch.cuda.synchronize()
    ref = [o.clone() for o in fresh]
    ws = torch.zeros(max(l.workspace.numel() for l in layers), dtype=torch.uint8, device=DEV)
    small_layers = H.gpu_step(saga, cfg, gs, dx)[1]
    for lay_s, lay_b in zip(small_layers, layers):
        lay_s.workspace, lay_b.workspace = ws, ws
    H.gpu_step(saga, cfg, gs, dx, small_layers)                   # small graph on the shared workspace
    for o in fresh:
        o.zero_()
    H.gpu_step(saga, cfg, gb, dx, layers, fresh)                  # then the big graph, workspace_zeroed = 1
    torch.cuda.synchronize()
    for a, b in zip(fresh, ref):
        assert torch.equal(a, b)
    assert int(ws[:64].count_nonzero()) == 0 or model in ("gcn_f32",)  # first ticket counters left zero


@pytest.mark.parametrize("scale", [1.0, 8.0, 40.0, 400.0])
@pytest.mark.parametrize("hub", [0, 20000])
def test_gat_score_range(saga, scale, hub):
    """GAT's softmax shift per row is the bound LeakyReLU(max_u el[u] + er[v])
    (reading A29): attention vectors scaled so the scores span a few units up
    to thousands -- every row's weights then underflow against the bound
    except those that reach max el, and the rows whose weight sum falls below
    kGatTiny are recomputed by the online-softmax fallback -- on a power-law
    graph with self-loops, optionally with a hub split across tasks."""
    n = 3001
    rng = np.random.default_rng(13)
    s = rng.integers(0, n, 30000).astype(np.int32)
    d = np.minimum(rng.zipf(1.7, 30000) - 1, n - 1).astype(np.int32)
    if hub:
        s = np.concatenate([s, rng.integers(0, n, hub).astype(np.int32)])
        d = np.concatenate([d, np.full(hub, 29, np.int32)])
    s, d = zoo.with_self_loops(n, s, d)
    cfg = _zoo_cfg("gat", n, s.shape[0])
    x = _zoo_inputs("gat", n, s, d, 17)
    x["a_src"] = (x["a_src"] * scale).contiguous()
    x["a_dst"] = (x["a_dst"] * scale).contiguous()
    x["src"], x["dst"] = torch.from_numpy(s), torch.from_numpy(d)
    dx = H.dev_inputs(x, DEV)
    g = H.gpu_graph(saga, cfg, dx)
    outs, layers = H.gpu_step(saga, cfg, g, dx)
    outs2, _ = H.gpu_step(saga, cfg, g, dx, layers)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs2[0])
    og = H.oracle_graph(oracle, cfg, x)
    refs = H.oracle_step(oracle, cfg, og, x)
    H.check(outs[0], refs[0], H.TOL["bf16"], f"gat scale={scale} hub={hub}")


def test_graph_close_stream_ordered(saga):
    """Graph.close(sync=False): the stream-ordered free of a graph used only on
    its build stream (bench.py's serving loop) -- graphs built, used and
    freed back to back on one stream without a host wait give the same
    outputs as the first one."""
    cfg = W.scaled(W.CONFIGS["C3"], 3000, 40000, "close")
    d = W.make_inputs(cfg, DEV)
    outs = []
    for _ in range(4):
        g = H.gpu_graph(saga, cfg, d)
        y = H.gpu_step(saga, cfg, g, d)[0][0]
        g.close(sync=False)
        outs.append(y)
    torch.cuda.synchronize()
    for y in outs[1:]:
        assert torch.equal(y, outs[0])
