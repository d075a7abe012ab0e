"""Test/bench glue: run a configured step on the GPU path and on the oracle.

The GPU side goes only through paper_2009_00804_b200 (the C ABI); the oracle
side only through oracle/.  Both consume the same tensors from workloads/.
"""
from __future__ import annotations

import numpy as np
import torch

import workloads as W

TOL = {"f32": 1e-4, "bf16": 2e-2}   # BASELINE.json north_star, normwise inf-relative (A18)
# SURVEY.md 8(c)'s per-row diagnostic ||y_v - yref_v|| / max(||yref_v||, 1e-3 ||yref||)
# is reported for every parity check and gated at ROW_GATE x the normwise bar
ROW_GATE = 10.0

# Every check() of the session: (test id, label, normwise err, per-row err, worst row, tol).
# tests/conftest.py writes them to $SAGA_PARITY_LOG (JSON) at the end of the session.
RECORDS: list = []
CURRENT_TEST = [""]


def check(y, ref, tol, label=""):
    """Parity gate: normwise inf-relative error <= tol (reading A18) and the
    per-row diagnostic <= ROW_GATE * tol.  Returns (normwise, per-row).
    (oracle is imported here, not at module level: bench.py's timed path uses
    this module's gpu_step and must not load the oracle.)"""
    import oracle
    yy = to_np(y) if isinstance(y, torch.Tensor) else np.asarray(y, dtype=np.float64)
    err = oracle.rel_err(yy, ref)
    rerr, row = oracle.row_err(yy, ref)
    RECORDS.append({"test": CURRENT_TEST[0], "label": label, "err": err, "row_err": rerr, "worst_row": row,
                    "tol": tol})
    assert err <= tol, f"{label}: normwise rel err {err:.3e} > {tol}"
    assert rerr <= ROW_GATE * tol, f"{label}: per-row err {rerr:.3e} (row {row}) > {ROW_GATE} x {tol}"
    return err, rerr


def dev_inputs(d, dev):
    return {k: (v.to(dev) if isinstance(v, torch.Tensor) else v) for k, v in d.items()}


def gpu_graph(saga, cfg, d):
    return saga.saga_graph_build(cfg.n, d["src"], d["dst"], d.get("etype"), cfg.num_etypes)


def gpu_step(saga, cfg, g, d, layers=None, outs=None):
    """Run the configured step; returns list of per-layer outputs (device).

    `outs` (the outputs of an earlier call) are reused as output buffers: no
    allocation, so the step can be captured in a CUDA graph."""
    o = (lambda i: outs[i]) if outs else (lambda i: None)
    act_relu = saga.SAGA_ACT_RELU
    dt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    if cfg.model == "gcn":
        lay = layers[0] if layers else saga.Layer("gcn", g, cfg.dims[0], cfg.dims[1], act_relu, dt,
                                                    fused=cfg.extra.get("fused", False))
        return [lay(d["X"], {"W": d["W"], "bias": d["b"]}, out=o(0))], [lay]
    if cfg.model == "sage":
        f0, f1, f2 = cfg.dims
        fz = cfg.extra.get("fused", False)   # NEXT-1: Gather + concat-GEMM in one kernel
        l1 = layers[0] if layers else saga.Layer("sage", g, f0, f1, act_relu, dt, fused=fz)
        l2 = layers[1] if layers else saga.Layer("sage", g, f1, f2, saga.SAGA_ACT_NONE, dt, fused=fz)
        h1 = l1(d["X"], {"W": d["W1"]}, out=o(0))
        return [h1, l2(h1, {"W": d["W2"]}, out=o(1))], [l1, l2]
    if cfg.model == "gat":
        fi, fo = cfg.dims
        lay = layers[0] if layers else saga.Layer("gat", g, fi, fo, saga.SAGA_ACT_ELU, dt, heads=cfg.heads,
                                                  head_dim=fo // cfg.heads, leaky_slope=0.2)
        return [lay(d["X"], {"W": d["W"], "attn_src": d["a_src"], "attn_dst": d["a_dst"]}, out=o(0))], [lay]
    if cfg.model == "gated":
        f = cfg.dims[0]
        lay = layers[0] if layers else saga.Layer("gated", g, f, f, saga.SAGA_ACT_NONE, dt)
        w = {k: d[k].contiguous() for k in ("W_type", "W_ih", "W_hh", "b_ih", "b_hh")}
        return [lay(d["H"], w, out=o(0))], [lay]
    if cfg.model == "sage_lstm":
        f, fo = cfg.dims
        lay = layers[0] if layers else saga.Layer("sage_lstm", g, f, fo, act_relu, dt)
        w = {k: d[k].contiguous() for k in ("W", "W_ih", "W_hh", "b_ih", "b_hh")}
        w["bias"] = d["b"]
        return [lay(d["X"], w, out=o(0))], [lay]
    if cfg.model == "ggnn":
        f = cfg.dims[0]
        lay = layers[0] if layers else saga.Layer("ggnn", g, f, f, act_relu, dt,
                                                  aggregator=cfg.extra.get("agg", "sum"))
        w = {k: d[k].contiguous() for k in ("W_ih", "W_hh", "b_ih", "b_hh")}
        w["W"], w["bias"] = d["W_e"].contiguous(), d["b_e"]
        return [lay(d["H"], w, out=o(0))], [lay]
    if cfg.model == "rgcn":
        f, fo = cfg.dims
        lay = layers[0] if layers else saga.Layer("rgcn", g, f, fo, act_relu, dt)
        return [lay(d["H"], {"W_type": d["W_type"].contiguous(), "W": d["W_self"], "bias": d["b"]}, out=o(0))], [lay]
    raise ValueError(cfg.model)


def oracle_graph(oracle, cfg, d):
    et = d.get("etype")
    return oracle.csr_build(cfg.n, d["src"].cpu(), d["dst"].cpu(), None if et is None else et.cpu(),
                            cfg.num_etypes)


def oracle_step(oracle, cfg, og, d, rows=None, layer_inputs=None):
    """fp64 reference of the configured step (list per layer).

    For SAGE, layer 2 takes `layer_inputs[1]` if given (the GPU's bf16 H1,
    per-layer parity, reading A19), else the oracle's own fp64 H1."""
    c = {k: (v.cpu() if isinstance(v, torch.Tensor) else v) for k, v in d.items()}
    if cfg.model == "gcn":
        return [oracle.gcn(og, c["X"], c["W"].float(), c["b"], act=1, rows=rows)]
    if cfg.model == "sage":
        h1 = oracle.sage_mean(og, c["X"], c["W1"].float(), act=1, rows=None)
        x2 = layer_inputs[1] if layer_inputs is not None else h1
        h2 = oracle.sage_mean(og, x2, c["W2"].float(), act=0, rows=rows)
        return [h1 if rows is None else h1[np.asarray(rows)], h2]
    if cfg.model == "gat":
        return [oracle.gat(og, c["X"], c["W"].float(), c["a_src"], c["a_dst"], 0.2, rows=rows)]
    if cfg.model == "gated":
        return [oracle.gated(og, c["H"], c["W_type"], c["W_ih"], c["W_hh"], c["b_ih"], c["b_hh"], rows=rows)]
    if cfg.model == "rgcn":
        return [oracle.rgcn(og, c["H"], c["W_type"], c["W_self"], c["b"], act=1, rows=rows)]
    if cfg.model == "ggnn":
        return [oracle.ggnn(og, c["H"], c["W_e"], c["b_e"], c["W_ih"], c["W_hh"], c["b_ih"], c["b_hh"], act=1,
                            agg=cfg.extra.get("agg", "sum"), rows=rows)]
    if cfg.model == "sage_lstm":
        return [oracle.sage_lstm(og, c["X"], c["W_ih"].float(), c["W_hh"].float(), c["b_ih"], c["b_hh"],
                                 c["W"].float(), c["b"], act=1, rows=rows)]
    raise ValueError(cfg.model)


def to_np(t):
    return t.detach().float().cpu().numpy().astype(np.float64)


def sample_rows(og, k, seed=0):
    """Sampled rows for full-size checks: the 16 highest in-degree rows (hubs,
    split across tasks), first/last rows, and k uniform rows."""
    n = og.n
    rng = np.random.default_rng(seed)
    hubs = np.argsort(-og.in_deg, kind="stable")[:16]
    rows = np.concatenate([hubs, [0, n - 1], rng.integers(0, n, k)]).astype(np.int64)
    return np.unique(rows)
