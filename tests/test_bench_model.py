"""bench.py's roofline model (CPU): per-launch algorithmic bytes/FLOPs and
the roofline object."""
import importlib.util
import os

import numpy as np

import pytest

import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_c5_aggregation_compulsory_bytes(bench):
    c = W.CONFIGS["C5"]
    a = bench.algorithmic(c)["agg_gcn_bf16"]
    n, e = 1 << 22, (1 << 26) + (1 << 22)
    # col_src once, row_ptr once, Y (bf16 256) once, dinv once, out (bf16 256) once
    assert a["bytes"] == 4 * e + 8 * (n + 1) + 512 * n + 4 * n + 512 * n
    assert a["peak"] == "hbm"
    g = bench.algorithmic(c)["gemm_bf16_tc"]
    assert g["flops"] == 2 * n * 256 * 256


def test_gat_view_bytes(bench):
    """GAT with the aggregation view (graph_build.cu step 8): the edge kernel's
    rows, edges and gathered sources only; the GEMM also writes the epilogue
    rows' outputs."""
    c = W.CONFIGS["C3"]
    n = c.n
    gs = {"n_epi": 100, "an": 900, "ae": 5000, "n_src": 700, "n_heavy": 0}
    a = bench.algorithmic(c, gs)["gat_edge"]
    assert a["bytes"] == 4 * 5000 + 8 * 901 + 4 * 900 + 32 * 900 + 700 * (128 + 32) + 900 * 128
    g = bench.algorithmic(c, gs)["gemm_bf16_tc_gat"]
    assert g["bytes"] == n * 512 + 256 * 64 * 2 + n * 128 + n * 64 + 100 * 128


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4", "C5", "C6", "C7", "C8"])
def test_every_profiled_kernel_has_a_model(bench, cfg):
    expected = {"C1": {"gcn_f32_fused"}, "C2": {"agg_mean_bf16", "gemm_bf16_tc"},
                "C3": {"gemm_bf16_tc_gat", "gat_edge"}, "C4": {"agg_typed_f32", "gated_apply_tf32x3"},
                "C5": {"gemm_bf16_tc", "agg_gcn_bf16"}, "C6": {"agg_typed_mean_f32", "rgcn_apply_tf32x3"},
                "C7": {"lstm_gather", "lstm_input_gemm", "gemm_bf16_tc"},
                "C8": {"ggnn_edge_i8x", "agg_edge_mlp_f32", "ggnn_gru_tf32x3"}}[cfg]
    alg = bench.algorithmic(W.CONFIGS[cfg])
    assert expected <= set(alg)
    for k in expected:
        assert alg[k]["bytes"] > 0 and alg[k]["flops"] > 0


def test_sage_model_is_per_launch(bench):
    """Two layers -> two launches per kernel per step: the model is the mean."""
    c = W.CONFIGS["C2"]
    n, e = c.n, c.num_edges
    a = bench.algorithmic(c)["agg_mean_bf16"]
    one = e * 4 + (n + 1) * 8 + n * 4 + 2 * n * 128 * 2   # width 128 both layers: X read + M written
    assert a["bytes"] == one


def test_roofline_object(bench):
    pk = {"hbm_gbs": 6500.0, "bf16_tflops": 1650.0, "bf16_tflops_sustained": 1390.0, "source": "measured"}
    r = bench.roofline_of("k", {"bytes": 6.5e9, "flops": 1, "peak": "hbm"}, 2e-3, pk, 1.0e10)
    assert r["bound"] == "hbm" and abs(r["achieved"] - 3250.0) < 1e-6 and abs(r["frac"] - 0.5) < 1e-12
    assert r["traffic"] == 1.0e10 and abs(r["dram_frac"] - 1.0e10 / 2e-3 / 6.5e12) < 1e-12
    t = bench.roofline_of("k", {"bytes": 1, "flops": 1e12, "peak": "tensor_tf32x3"}, 1e-2, pk, None)
    assert t["bound"] == "tensor" and abs(t["peak"] - 1650.0 * 1.1 / 2.25 / 3) < 1e-9
    assert abs(t["achieved"] - 100.0) < 1e-9


def test_hbm_bound_contraction_is_held_to_hbm(bench):
    """C5's pre-projection GEMM (128 FLOP/B) sits below the bf16 ridge."""
    pk = {"hbm_gbs": 6536.0, "bf16_tflops": 1653.2, "bf16_tflops_sustained": 1391.2, "source": "measured"}
    spec = bench.algorithmic(W.CONFIGS["C5"])["gemm_bf16_tc"]
    r = bench.roofline_of("gemm_bf16_tc", spec, 0.7e-3, pk, None)
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    c4 = bench.algorithmic(W.CONFIGS["C4"])["gated_apply_tf32x3"]
    assert bench.roofline_of("g", c4, 0.36e-3, pk, None)["bound"] == "tensor"


@pytest.mark.parametrize("cfg", sorted(W.CONFIGS))
def test_cpu_baseline_leg_runs_every_model(bench, cfg):
    """bench.py's cpu_baseline / --impl reference leg evaluates the oracle for
    every configured model (tiny scaled graph, CPU only)."""
    import oracle
    c = W.scaled(W.CONFIGS[cfg], 64, 256, cfg + "t")
    d = W.make_inputs(c, "cpu")
    og = oracle.csr_build(c.n, d["src"], d["dst"], None if d.get("etype") is None else d["etype"], c.num_etypes)
    rows = np.arange(0, c.n, 7, dtype=np.int64)
    out = bench.harness_step_rows(c, og, d, rows, oracle)
    assert np.all(np.isfinite(np.asarray(out)))


def test_lstm_gather_is_held_to_the_bf16_contraction_roofline(bench):
    """Round 2: the LSTM gather's recurrent GEMVs run on the tensor cores
    (mma.sync bf16) for the short sequences and on FHFMA across CTA pairs for
    the long ones, so it is held to the bf16 contraction roofline: 2 * 4f * f
    FLOPs per edge against a 1 KB P row per edge is 128 FLOP/B, below the
    measured ridge, so the HBM side of it applies."""
    a = bench.algorithmic(W.CONFIGS["C7"])["lstm_gather"]
    pk = bench.peaks()
    assert a["peak"] == "tensor_bf16" and a["flops"] / a["bytes"] < pk["bf16_tflops"] * 1e3 / pk["hbm_gbs"]
    r = bench.roofline_of("lstm_gather", a, 5.0e-3, pk, None)
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    assert r["achieved"] == pytest.approx(a["bytes"] / 5.0e-3 / 1e9)


def test_cpu_baseline_sample_grows_to_the_time_target(bench):
    """cpu_baseline sizing: a tiny first sample is grown (whole graph, then
    repeated runs) to about the requested CPU time; the value is updates/s of
    the oracle as it stands."""
    import oracle
    c = W.scaled(W.CONFIGS["C1"], 256, 1024, "C1t")
    d = W.make_inputs(c, "cpu")
    og = oracle.csr_build(c.n, d["src"], d["dst"])
    cpu = bench.sized_cpu_baseline(c, d, og, oracle, ref_edges=64, ref_seconds=0.2)
    assert cpu["kind"] == "oracle" and cpu["value"] > 0 and cpu["cores"] >= 1
    assert f"{c.n} random destination rows" in cpu["sample"] and " runs" in cpu["sample"]
    none = bench.sized_cpu_baseline(c, d, og, oracle, ref_edges=64, ref_seconds=0)
    assert " runs" not in none["sample"]


@pytest.mark.parametrize("cfg", sorted(W.CONFIGS))
def test_every_model_kernel_has_a_stage(bench, cfg):
    """The stage timeline tags every modelled launch with its SAGA stage."""
    c = W.CONFIGS[cfg]
    for k in bench.algorithmic(c):
        assert bench.stage_of(c, k) != "other", k


def test_stage_breakdown_and_timeline(bench, tmp_path):
    import json
    c = W.CONFIGS["C5"]
    trace = [("gemm_bf16_tc", 0.0, 0.7), ("agg_gcn_bf16", 0.7, 4.2), ("gemm_bf16_tc", 5.0, 5.8),
             ("agg_gcn_bf16", 5.8, 9.0)]
    st = bench.stage_breakdown(c, trace, 2)
    assert st["S2 pre-projection"]["ms_per_step"] == pytest.approx(0.75)
    assert st["S3+S4 Scatter/Gather (+S5 epilogue)"]["ms_per_step"] == pytest.approx(3.35)
    assert sum(v["share"] for v in st.values()) == pytest.approx(1.0)
    assert bench.stage_breakdown(c, [], 2) is None
    p = tmp_path / "t.json"
    bench.write_timeline(str(p), c, trace)
    ev = json.load(open(p))["traceEvents"]
    assert len(ev) == 4 and ev[1]["ts"] == pytest.approx(700.0) and ev[1]["dur"] == pytest.approx(3500.0)


def test_fused_gcn_model(bench):
    """--fused on C5 (NEXT-1, gcn_fused.cu): one kernel whose compulsory bytes are
    col_src, row_ptr, dinv, every X row once, W and the output."""
    c = W.scaled(W.CONFIGS["C5"], W.CONFIGS["C5"].n, W.CONFIGS["C5"].m, "C5")
    c.extra["fused"] = True
    alg = bench.algorithmic(c)
    assert set(alg) == {"gcn_fused_tc"}
    n, e = c.n, c.num_edges
    assert alg["gcn_fused_tc"]["bytes"] == e * 4 + (n + 1) * 8 + n * 4 + n * 256 * 2 + 256 * 256 * 2 + n * 256 * 2
    assert alg["gcn_fused_tc"]["flops"] == 2 * e * 256 + 2 * n * 256 * 256
    assert bench.stage_of(c, "gcn_fused_tc").startswith("S3+S4+S5")
