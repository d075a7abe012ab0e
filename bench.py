#!/usr/bin/env python
"""bench.py -- one SAGA-NN layer at inference on B200 (arXiv 2009.00804).

Metric (BASELINE.json): ms/layer and edge-feature updates/s per SAGA-NN layer;
% of HBM roofline.  A "step" is one pass of the whole hot path over one batch
(SURVEY.md 8(a) rows S1-S6 on a pre-built graph: pre-projection GEMM, fused
Scatter/ApplyEdge/Gather, ApplyVertex epilogue).  S0 (graph build) runs once
per graph and is reported separately (and inside the `e2e` figure).

Default workload: config C5 (GCN at scale, R-MAT 2^22 vertices, 2^26 edges +
self-loops, 256 -> 256 bf16), the largest configuration (BASELINE.json
configs[4]); C1-C4 are parity-test cases (`--config` runs them too).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl saga|reference]

N > 1 (torchrun): one independent replica per GPU ("replicas only": the
north star fixes one GPU with no sharding), value = total updates / max time.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
UNIT = "edge-feature updates/s"


def ncu_traffic(cfg_name, kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu capture
    (profiles/ncu_traffic.json, written by scripts/make_profiles.py), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        return json.load(open(p))[cfg_name][kernel]
    except Exception:
        return None


def ncu_traffic_source():
    """Where `traffic` comes from: the capture file and the commit it was taken at."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        j = json.load(open(p))
        return f"profiles/ncu_traffic.json (ncu --set full, commit {j.get('_commit', 'unknown')}, {j.get('_when', '')})"
    except Exception:
        return None


def measured_tensor_peaks(dev):
    """TF32 and INT8 dense tensor-core throughput measured in this run (torch /
    cuBLAS, 8192^3, best of 5): the roofline peaks of the split-TF32 and the
    int8-sliced GEMMs (MEASURED_PEAKS.json has bf16 only)."""
    out = {}
    try:
        n = 8192
        a = torch.randn(n, n, device=dev)
        b = torch.randn(n, n, device=dev)
        old = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = True
        out["tf32_tflops"] = _best_tflops(lambda: a @ b, 2.0 * n ** 3)
        torch.backends.cuda.matmul.allow_tf32 = old
        ai = torch.randint(-64, 64, (n, n), device=dev, dtype=torch.int8)
        bi = torch.randint(-64, 64, (n, n), device=dev, dtype=torch.int8).t()
        out["int8_tops"] = _best_tflops(lambda: torch._int_mm(ai, bi), 2.0 * n ** 3)
        del a, b, ai, bi
    except Exception as e:  # pragma: no cover
        out["error"] = str(e)[:120]
    return out


def _best_tflops(fn, flops, reps=5):
    fn()
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        t = s.elapsed_time(e) / 1e3
        best = t if best is None else min(best, t)
    return flops / best / 1e12


def graph_stats(cfg, d):
    """Sizes of the graph's aggregation view (graph_build.cu step 8) for the
    byte model: rows whose in-edges are one self-loop or none are finished by
    the GEMM epilogue; the gather runs over the other rows' edges and reads
    each distinct source row once at least."""
    src, dst = d["src"].long(), d["dst"].long()
    n = cfg.n
    indeg = torch.bincount(dst, minlength=n)
    loops = torch.bincount(dst[src == dst], minlength=n)
    epi = (indeg == 0) | ((indeg == 1) & (loops == 1))
    keep = ~epi[dst]
    srcs = torch.unique(src[keep])
    return {"n_epi": int(epi.sum()), "an": int((~epi).sum()), "ae": int(keep.sum()), "n_src": int(srcs.numel()),
            "n_heavy": int((indeg >= 256).sum())}  # kHeavyInDeg: the fp64 ApplyVertex rows (gru_f64.cu)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return {"hbm_gbs": j["hbm_gbs"], "bf16_tflops": j["bf16_tflops"],
                "bf16_tflops_sustained": j.get("bf16_tflops_sustained", j["bf16_tflops"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


# ---------------------------------------------------------------- clocks ----
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index):
        self.index, self.proc, self.lines = index, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------- byte model ----
def algorithmic(cfg, gs=None):
    """Algorithmic (compulsory) bytes and FLOPs PER LAUNCH of each kernel
    (DESIGN.md section 5): every array the kernel must touch, once; FLOPs are
    the layer's own arithmetic counted once.  `peak` names the roofline the
    kernel is held to: "hbm", or "tensor_bf16" / "tensor_tf32x3" (3xTF32: the
    fp32-accurate product costs three TF32 MMAs, so its peak is TF32 / 3).
    `gs` (graph_stats): the aggregation view's sizes (GAT) and the heavy rows
    (gated, GGNN)."""
    n, e = cfg.n, cfg.num_edges
    out = {}
    if cfg.model == "gcn" and cfg.dtype == "bf16" and cfg.extra.get("fused"):
        fi, fo = cfg.dims   # NEXT-1: col_src, row_ptr, dinv, every X row once, W, out
        out["gcn_fused_tc"] = {"bytes": e * 4 + (n + 1) * 8 + n * 4 + n * fi * 2 + fi * fo * 2 + n * fo * 2,
                               "flops": 2 * e * fi + 2 * n * fi * fo, "peak": "hbm"}
    elif cfg.model == "gcn" and cfg.dtype == "bf16":
        fi, fo = cfg.dims
        out["gemm_bf16_tc"] = {"bytes": n * fi * 2 + fi * fo * 2 + n * 4 + n * fo * 2, "flops": 2 * n * fi * fo,
                               "peak": "tensor_bf16"}
        out["agg_gcn_bf16"] = {"bytes": e * 4 + (n + 1) * 8 + n * fo * 2 + n * 4 + n * fo * 2, "flops": e * fo,
                               "peak": "hbm"}
    elif cfg.model == "gcn":
        fi, fo = cfg.dims
        out["gcn_f32_fused"] = {"bytes": e * 4 + (n + 1) * 8 + n * fi * 4 + n * 4 + n * fo * 4,
                                "flops": 2 * e * fi + 2 * n * fi * fo, "peak": "hbm"}
    elif cfg.model == "sage" and cfg.extra.get("fused"):
        f0, f1, f2 = cfg.dims   # NEXT-1: per launch x rows + gathered rows + out (mean of the two layers)
        out["sage_fused_tc"] = {"bytes": (e * 4 + (n + 1) * 8 + n * 4 + n * (f0 + f1) * 2 + n * (f1 + f2) * 2) // 2,
                                "flops": (e * (f0 + f1) + 2 * n * (2 * f0 * f1 + 2 * f1 * f2)) // 2, "peak": "hbm"}
    elif cfg.model == "sage":
        f0, f1, f2 = cfg.dims   # two layers: agg widths f0, f1; GEMMs 2f0 -> f1, 2f1 -> f2 (mean of the two launches)
        out["agg_mean_bf16"] = {"bytes": e * 4 + (n + 1) * 8 + n * 4 + n * (f0 + f1) * 2 * 2 // 2,
                                "flops": e * (f0 + f1) // 2, "peak": "hbm"}
        out["gemm_bf16_tc"] = {"bytes": n * 2 * (2 * f0 + f1 + 2 * f1 + f2) // 2,
                               "flops": 2 * n * (2 * f0 * f1 + 2 * f1 * f2) // 2, "peak": "tensor_bf16"}
    elif cfg.model == "gat":
        fi, fo = cfg.dims
        if gs is None:
            gs = {"n_epi": 0, "an": n, "ae": e, "n_src": n}
        an, ae = gs["an"], gs["ae"]
        # GEMM: X, W read; z and el / er of every row written, the epilogue rows' outputs
        out["gemm_bf16_tc_gat"] = {"bytes": n * fi * 2 + fi * fo * 2 + n * fo * 2 + n * 64 + gs["n_epi"] * fo * 2,
                                   "flops": 2 * n * fi * fo, "peak": "tensor_bf16"}
        # view gather: col_src, row_ptr, row map, er of its rows; z and el of each gathered source once; outputs
        out["gat_edge"] = {"bytes": ae * 4 + (an + 1) * 8 + an * 4 + an * 32 + gs["n_src"] * (fo * 2 + 32)
                           + an * fo * 2, "flops": 10 * ae * fo, "peak": "hbm"}
    elif cfg.model == "gated":
        f, T = cfg.dims[0], cfg.num_etypes
        # typed view (rows (v, t)): col_src, row_ptr of n*T rows, H once, S [n][T][f]
        out["agg_typed_f32"] = {"bytes": e * 4 + (n * T + 1) * 8 + n * f * 4 + n * T * f * 4, "flops": e * f,
                                "peak": "hbm"}
        # S read, m written + read, h read twice (GEMM A operand, GRU epilogue), h' written
        out["gated_apply_tf32x3"] = {"bytes": n * T * f * 4 + n * f * 4 * 5, "flops": 2 * n * (T * f * f + 6 * f * f),
                                     "peak": "tensor_tf32x3"}
        if gs:  # heavy rows: fp64 message GEMM + GRU from the fp64 sums (gru_f64.cu)
            nh = gs["n_heavy"]
            out["gru_heavy_f64"] = {"bytes": nh * (T * f * 8 + f * 4 * 2 + 4) + (T + 6) * f * f * 8,
                                    "flops": 2 * nh * (T * f * f + 6 * f * f), "peak": "fp64_pipe"}
    elif cfg.model == "sage_lstm":
        f, fo = cfg.dims
        # per edge: gather a 1 KB row of P (4 gates bf16); recurrent GEMV 2 * 4f * f FLOPs.  Round 2:
        # the short sequences' GEMVs run on the tensor cores (mma.sync bf16), the long ones' on FHFMA
        # across CTA pairs, so the bf16 tensor peak is the machine's bound for the contraction; the
        # kernel's real bound is the hub's chain of dependent steps (DESIGN.md NEXT-2)
        out["lstm_gather"] = {"bytes": e * 4 + (n + 1) * 8 + e * 4 * f * 2 + n * f * 2 + 4 * f * f * 2,
                              "flops": e * 2 * 4 * f * f, "peak": "tensor_bf16"}
        out["lstm_input_gemm"] = {"bytes": n * f * 2 + f * f * 2 + n * f * 2, "flops": 2 * n * f * f,
                                  "peak": "tensor_bf16"}
        out["gemm_bf16_tc"] = {"bytes": n * 2 * (2 * f + fo), "flops": 2 * n * 2 * f * fo, "peak": "tensor_bf16"}
    elif cfg.model == "rgcn":
        f, fo = cfg.dims
        T = cfg.num_etypes
        out["agg_typed_mean_f32"] = {"bytes": e * 4 + (n * T + 1) * 8 + n * T * 4 + n * f * 4 + n * T * f * 4,
                                     "flops": e * f, "peak": "hbm"}
        # S read, H read, out written
        out["rgcn_apply_tf32x3"] = {"bytes": n * T * f * 4 + n * f * 4 + n * fo * 4, "flops": 2 * n * (T + 1) * f * fo,
                                    "peak": "tensor_tf32x3"}
    elif cfg.model == "ggnn":
        f = cfg.dims[0]
        # AB = H . [W_a | W_b] + [0 | b_e] on the int8 tensor cores (exact accumulation):
        # H read, AB written (K = f, N = 2f); 8 int8 MMAs per product
        out["ggnn_edge_i8x"] = {"bytes": n * f * 4 + n * 2 * f * 4, "flops": 2 * n * f * 2 * f,
                                "peak": "tensor_i8x8"}
        # compulsory: col_src, row_ptr, AB read once (A and B halves), m written
        # (the per-edge A-row gathers, 512 B each, are L2 traffic, as for the
        # other gathers)
        out["agg_edge_mlp_f32"] = {"bytes": e * 4 + (n + 1) * 8 + n * 2 * f * 4 + n * f * 4,
                                   "flops": 3 * e * f, "peak": "hbm"}
        # GRU over [m || h]: m, h read (h twice), h' written
        out["ggnn_gru_tf32x3"] = {"bytes": n * f * 4 * 4, "flops": 2 * n * 6 * f * f, "peak": "tensor_tf32x3"}
        if gs:  # heavy rows in fp64: their B before the gather, the GRU after it (gru_f64.cu)
            nh = gs["n_heavy"]
            out["ggnn_heavy_b_f64"] = {"bytes": nh * (f * 4 + f * 8) + f * f * 8, "flops": 2 * nh * f * f,
                                       "peak": "fp64_pipe"}
            out["gru_heavy_f64"] = {"bytes": nh * (f * 8 + f * 4 * 2 + 4) + 6 * f * f * 8,
                                    "flops": 2 * nh * 6 * f * f, "peak": "fp64_pipe"}
    return out


FP64_PIPE_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12


def roofline_of(name, spec, avg_s, pk, traffic):
    """roofline object of the bench line for kernel `name`."""
    base = {"kernel": name, "kernel_ms": avg_s * 1e3, "traffic": traffic,
            "algorithmic_bytes": spec["bytes"], "algorithmic_flops": spec["flops"], "peak_source": pk["source"]}
    if spec["peak"] == "hbm":
        ach = spec["bytes"] / avg_s / 1e9
        r = dict(base, bound="hbm", achieved=ach, peak=pk["hbm_gbs"], unit="GB/s", frac=ach / pk["hbm_gbs"])
        if traffic:  # DRAM-throughput fraction: the ncu bytes this kernel really moves, at this launch time
            r["dram_frac"] = traffic / avg_s / 1e9 / pk["hbm_gbs"]
        return r
    if spec["peak"] == "fp64_pipe":
        peak = FP64_PIPE_TFLOPS
        ach = spec["flops"] / avg_s / 1e12
        return dict(base, bound="alu", achieved=ach, peak=peak, unit="TFLOP/s", frac=ach / peak,
                    peak_note="derived: 148 SM x 64 fp64 FMA/clk x 2 FLOP x 1.965 GHz (the DMMA tensor path and "
                              "DFMA share it: ncu sm__ops_path_tensor_src_fp64 peak 128 ops/clk/SM)")
    # tensor: bf16 measured burst peak (MEASURED_PEAKS.json); TF32 and INT8 measured
    # in this run (cuBLAS 8192^3, measured_tensor_peaks), else the nominal ratios
    peak = pk["bf16_tflops"]
    note = "measured bf16 burst"
    if spec["peak"] == "tensor_tf32x3":
        if pk.get("tf32_tflops"):
            peak, note = pk["tf32_tflops"] / 3.0, "TF32 measured in this run / 3 (3xTF32)"
        else:
            peak, note = pk["bf16_tflops"] * (1.1 / 2.25) / 3.0, "bf16 x nominal tf32/bf16 (1.1/2.25) / 3 (3xTF32)"
    elif spec["peak"] == "tensor_i8x8":
        if pk.get("int8_tops"):
            peak, note = pk["int8_tops"] / 8.0, "INT8 measured in this run / 8 (8 digit-pair MMAs per product)"
        else:
            peak, note = pk["bf16_tflops"] * 2.0 / 8.0, "bf16 x nominal int8/bf16 (2) / 8 (digit-pair MMAs)"
    # a contraction whose bytes take longer than its FLOPs is HBM-bound
    if spec["bytes"] / (pk["hbm_gbs"] * 1e9) > spec["flops"] / (peak * 1e12):
        ach = spec["bytes"] / avg_s / 1e9
        return dict(base, bound="hbm", achieved=ach, peak=pk["hbm_gbs"], unit="GB/s", frac=ach / pk["hbm_gbs"],
                    peak_note="arithmetic intensity below the ridge of " + note)
    ach = spec["flops"] / avg_s / 1e12
    return dict(base, bound="tensor", achieved=ach, peak=peak, unit="TFLOP/s", frac=ach / peak, peak_note=note)


# --------------------------------------------------------------- helpers ----
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def max_over_ranks(x: float, device) -> float:
    """Max of a per-rank scalar over all ranks (1 rank: itself).  Timing rule:
    multi-GPU numbers are the slowest rank's device time."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_value(units_per_step: int, steps: int, world_size: int, max_ms: float) -> float:
    """Whole-job throughput: the units every rank processed (weak scaling: each
    replica does a full step) over the slowest rank's time."""
    return units_per_step * steps * world_size / (max_ms / 1e3)


def emit(obj, rank):
    if rank == 0:
        print(json.dumps(obj), flush=True)


def l2_flush_buffer(dev):
    return torch.empty(512 << 20, dtype=torch.uint8, device=dev)


def cpu_baseline(cfg, d_cpu, og, sample_rows, oracle, reps=1):
    """Time the oracle (as it stands) on a bounded row sample on host cores
    (`reps` back-to-back runs of it)."""
    t0 = time.perf_counter()
    for _ in range(reps):
        harness_step_rows(cfg, og, d_cpu, sample_rows, oracle)
    dt = time.perf_counter() - t0
    upd = sample_updates(cfg, og, sample_rows) * reps
    return upd / dt, dt, upd


def sized_cpu_baseline(cfg, c, og, oracle, ref_edges, ref_seconds):
    """The cpu_baseline object: the oracle timed on a row sample of about
    ref_edges in-edges, grown to about ref_seconds of CPU work (more rows, up
    to the whole graph, then back-to-back repeated runs of it)."""
    rows = pick_sample(og, ref_edges)
    v_cpu, dt, upd = cpu_baseline(cfg, c, og, rows, oracle)
    reps = 1
    if ref_seconds > 0 and dt < 0.5 * ref_seconds:
        e_all = int(og.in_deg.sum())
        want = int(upd / cfg.f_canon * ref_seconds / max(dt, 1e-4))
        if cfg.model != "sage" and want > 1.5 * upd / cfg.f_canon and len(rows) < og.n:
            rows = pick_sample(og, min(want, e_all))
            v_cpu, dt, upd = cpu_baseline(cfg, c, og, rows, oracle)
        if dt < 0.5 * ref_seconds:
            reps = int(min(100000, max(1, ref_seconds / max(dt, 1e-5))))
            v_cpu, dt, upd = cpu_baseline(cfg, c, og, rows, oracle, reps)
    per = upd // reps // cfg.f_canon
    return {"value": v_cpu, "unit": UNIT, "cores": oracle_threads(), "kind": "oracle",
            "sample": f"{len(rows)} random destination rows of {cfg.name} ({per} in-edges)"
                      + (f" x {reps} runs" if reps > 1 else "") + f", fp64 C oracle, {dt:.1f} s"}


def harness_step_rows(cfg, og, c, rows, oracle):
    """The oracle's configured step restricted to destination `rows`
    (SAGE: both layers over all rows -- layer 2 needs H1 of every neighbour)."""
    if cfg.model == "gcn":
        return oracle.gcn(og, c["X"], c["W"].float(), c["b"], act=1, rows=rows)
    if cfg.model == "sage":
        h1 = oracle.sage_mean(og, c["X"], c["W1"].float(), act=1)
        return oracle.sage_mean(og, h1, c["W2"].float(), act=0)
    if cfg.model == "gat":
        return oracle.gat(og, c["X"], c["W"].float(), c["a_src"], c["a_dst"], 0.2, rows=rows)
    if cfg.model == "rgcn":
        return oracle.rgcn(og, c["H"], c["W_type"], c["W_self"], c["b"], act=1, rows=rows)
    if cfg.model == "sage_lstm":
        return oracle.sage_lstm(og, c["X"], c["W_ih"].float(), c["W_hh"].float(), c["b_ih"], c["b_hh"],
                                c["W"].float(), c["b"], act=1, rows=rows)
    if cfg.model == "ggnn":
        return oracle.ggnn(og, c["H"], c["W_e"], c["b_e"], c["W_ih"], c["W_hh"], c["b_ih"], c["b_hh"], act=1,
                           agg=cfg.extra.get("agg", "sum"), rows=rows)
    if cfg.model == "gated":
        return oracle.gated(og, c["H"], c["W_type"], c["W_ih"], c["W_hh"], c["b_ih"], c["b_hh"], rows=rows)
    raise ValueError(cfg.model)


def sample_updates(cfg, og, rows):
    if cfg.model == "sage":
        return cfg.layer_updates()
    deg = og.in_deg[np.asarray(rows)].astype(np.int64).sum()
    return int(deg) * cfg.f_canon


def pick_sample(og, target_edges, seed=1):
    rng = np.random.default_rng(seed)
    rows = rng.permutation(og.n)
    cum = np.cumsum(og.in_deg[rows].astype(np.int64))
    k = int(np.searchsorted(cum, target_edges)) + 1
    return np.sort(rows[:k]).astype(np.int64)


def oracle_threads():
    n = os.environ.get("OMP_NUM_THREADS")
    return int(n) if n else (len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count())


# ------------------------------------------------------------ reference ----
def run_reference(args, cfg):
    """--impl reference: the fp64 oracle as it stands on the host cores."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    d = W.make_inputs(cfg, dev)
    c = {k: (v.cpu() if isinstance(v, torch.Tensor) else v) for k, v in d.items()}
    og = oracle.csr_build(cfg.n, c["src"], c["dst"], c.get("etype"), cfg.num_etypes)
    rows = pick_sample(og, args.ref_edges)
    for _ in range(args.warmup):
        harness_step_rows(cfg, og, c, rows[: max(1, len(rows) // 8)], oracle)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        harness_step_rows(cfg, og, c, rows, oracle)
        times.append(time.perf_counter() - t0)
    upd = sample_updates(cfg, og, rows)
    tot = sum(times)
    val = upd * args.steps / tot
    cores = oracle_threads()
    sample = f"{len(rows)} destination rows ({upd // cfg.f_canon} in-edges) of {cfg.name} per step, fp64 C oracle"
    emit({"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
          "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
          "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
          "config": workload_config(cfg),
          "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
          "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}, 0)


def workload_config(cfg):
    desc = {"C1": "GCN fp32, ER N=2048 E=10240+self-loops, 64->16",
            "C2": "GraphSAGE-mean x2 bf16, R-MAT N=2^16 E=2^20 distinct, 128->128->64",
            "C3": "GAT 8x8 heads bf16, R-MAT N=2^18 E=2^22+self-loops, 256->64",
            "C4": "gated GRU fp32, R-MAT N=2^17 E=2^21, 4 edge types, 128",
            "C5": "GCN at scale bf16, R-MAT N=2^22 E=2^26+self-loops, 256->256",
            "C6": "R-GCN fp32 (NEXT-3), R-MAT N=2^17 E=2^21, 4 relation types, 128->128",
            "C7": "GraphSAGE-LSTM bf16 (NEXT-2), R-MAT N=2^16 E=2^20 distinct, 128->128",
            "C8": "paper-form GGNN fp32 (NEXT-4: edge MLP on [h_src||h_dst] + ReLU, sum, GRU), R-MAT N=2^17 E=2^21, 128"}
    w = desc.get(cfg.name, cfg.name) + (" [NEXT-1 fused Gather + ApplyVertex GEMM, one kernel]" if cfg.extra.get("fused") else "")
    return {"workload": f"{cfg.name}: {w}", "vertices": cfg.n, "edges": cfg.num_edges,
            "model": cfg.model, "global_batch": cfg.n, "parallelism": "replicas"}


# ----------------------------------------------------------------- main ----
def run_saga(args, cfg):
    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_2009_00804_b200 as saga
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from tests import harness as H

    d = W.make_inputs(cfg, dev)
    torch.cuda.synchronize()
    # S0 graph build (once per graph; timed separately, after one warm-up
    # build that fills the stream-ordered pool)
    H.gpu_graph(saga, cfg, d).close()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    g = H.gpu_graph(saga, cfg, d)
    t1.record()
    torch.cuda.synchronize()
    build_ms = t0.elapsed_time(t1)

    outs, layers = H.gpu_step(saga, cfg, g, d)
    big = cfg.n * max(cfg.dims) * (2 if cfg.dtype == "bf16" else 4) > (256 << 20)
    flush = None if big else l2_flush_buffer(dev)
    for _ in range(args.warmup):
        H.gpu_step(saga, cfg, g, d, layers, outs)
    torch.cuda.synchronize()

    # Timed regions of the same K steps (each step: L2 flush if the inputs fit
    # in L2, start event, the layer step, end event), each captured ONCE into a
    # CUDA graph and replayed once, so host launch overhead is out of the timed
    # steps (--eager launches them directly).
    #   1. only the step events: `value`, `ms_per_step` (mean), median / min;
    #   2. per-kernel event pairs around EVERY kernel (saga_profile): the
    #      `per_kernel` table; the pairs serialise the kernels and turn off
    #      programmatic launch, so these durations are upper bounds
    #      (`ms_per_step_profiled` is that region's step time);
    #   3. event pairs around the dominant kernel ONLY (saga_profile_filter),
    #      every other kernel launched exactly as in region 1 (PDL on): the
    #      roofline's kernel time;
    #   4. C1-C4, C6-C8 (inputs fit in L2): region 1 without the L2 flush --
    #      steady-state inference with a warm L2 (`warm_l2`).
    stream = torch.cuda.current_stream()
    ext = {} if args.eager else {"external": True}

    trace_box = []  # region 2's launch spans (saga_profile_trace)

    def region(profiled, only=None, do_flush=True):
        starts = [torch.cuda.Event(enable_timing=True, **ext) for _ in range(args.steps)]
        ends = [torch.cuda.Event(enable_timing=True, **ext) for _ in range(args.steps)]

        def timed_steps():
            for i in range(args.steps):
                if flush is not None and do_flush:
                    flush.zero_()
                starts[i].record()
                H.gpu_step(saga, cfg, g, d, layers, outs)
                ends[i].record()

        graph = None
        saga.saga_profile_filter(only)
        saga.saga_profile_enable(profiled and not args.no_kernel_events)
        if not args.eager:
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                timed_steps()
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        if graph is not None:
            graph.replay()
        else:
            timed_steps()
        torch.cuda.synchronize()
        prof = saga.saga_profile_read()
        if profiled and not only:
            trace_box[:] = saga.saga_profile_trace()
        saga.saga_profile_enable(False)
        saga.saga_profile_filter(None)
        if ws > 1:
            torch.distributed.barrier()
        return [s_.elapsed_time(e_) for s_, e_ in zip(starts, ends)], prof

    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.15)
    step_ms, _ = region(False)
    tot_ms = max_over_ranks(sum(step_ms), dev)
    prof_ms, prof = region(True)
    tot_prof_ms = max_over_ranks(sum(prof_ms), dev)
    dom = max(prof.items(), key=lambda kv: kv[1][1])[0] if prof else None
    dom_prof = region(True, only=dom)[1] if dom and not args.no_kernel_events else {}
    warm_ms = region(False, do_flush=False)[0] if flush is not None else None
    clocks = clk.stop()
    upd_step = cfg.layer_updates()
    value = job_value(upd_step, args.steps, ws, tot_ms)
    launches = sum(n for n, _ in prof.values())

    # roofline of the dominant kernel (largest share of the step), timed in region 3
    gs = graph_stats(cfg, d) if cfg.model in ("gat", "gated", "ggnn") else None
    alg = algorithmic(cfg, gs)
    pk = dict(peaks(), **measured_tensor_peaks(dev))
    roof = None
    if dom and dom in alg:
        n_l, ms_l = dom_prof.get(dom, prof[dom])
        traffic = args.traffic if args.traffic is not None else ncu_traffic(cfg.name, dom)
        roof = roofline_of(dom, alg[dom], ms_l / n_l / 1e3, pk, traffic)
        roof["kernel_ms_serialised"] = prof[dom][1] / prof[dom][0]
        roof["kernel_time"] = ("region 3: CUDA events around this kernel only, every other kernel as in the "
                               "timed step (programmatic launch on)")
        roof["traffic_source"] = ncu_traffic_source() if traffic is not None else None
    kernels = {}
    for k, (n_l, ms_l) in prof.items():
        a = alg.get(k, {"bytes": 0, "flops": 0})
        avg = ms_l / n_l
        kernels[k] = {"launches": n_l, "avg_ms": avg, "share": ms_l / tot_prof_ms if ws == 1 else None,
                      "alg_GBps": a["bytes"] / (avg / 1e3) / 1e9, "alg_TFLOPs": a["flops"] / (avg / 1e3) / 1e12}
        if k in alg:
            r = roofline_of(k, alg[k], avg / 1e3, pk, ncu_traffic(cfg.name, k))
            kernels[k].update({"bound": r["bound"], "frac": r["frac"], "traffic": r["traffic"]})

    # end to end through the public API with host buffers
    e2e = run_e2e(args, cfg, saga, H, d, dev, ws) if args.e2e_steps > 0 else None

    # CPU baseline: the oracle on a bounded sample (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        import oracle
        c = {k: (v.cpu() if isinstance(v, torch.Tensor) else v) for k, v in d.items()}
        og = oracle.csr_build(cfg.n, c["src"], c["dst"], c.get("etype"), cfg.num_etypes)
        cpu = sized_cpu_baseline(cfg, c, og, oracle, args.ref_edges, args.ref_seconds)

    conf = workload_config(cfg)
    conf.update({"l2": "inputs larger than L2 (no flush)" if big else "512 MiB L2 flush between steps (untimed)",
                 "graph_build_ms": build_ms, "per_kernel": kernels,
                 "step_ms": {"mean": tot_ms / args.steps, "median": statistics.median(step_ms), "min": min(step_ms),
                             "max": max(step_ms)},
                 "warm_l2": None if warm_ms is None else {
                     "what": "the same K steps without the L2 flush (steady-state, inputs L2-resident)",
                     "mean_ms": sum(warm_ms) / len(warm_ms), "median_ms": statistics.median(warm_ms),
                     "min_ms": min(warm_ms),
                     "value": job_value(upd_step, args.steps, ws, max_over_ranks(sum(warm_ms), dev))},
                 "graph_view": gs, "peaks": pk, "stages": stage_breakdown(cfg, trace_box, args.steps),
                 "ms_per_step_profiled": tot_prof_ms / args.steps,
                 "launch": "eager" if args.eager else "CUDA graph: the K timed steps captured once, replayed once"})
    res = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "bf16" if cfg.dtype == "bf16" else "f32",
           "data": "synthetic (seeded counter-based generator, workloads/)", "config": conf,
           "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks}
    emit(res, rank)
    if args.timeline and rank == 0:
        write_timeline(args.timeline, cfg, trace_box)
    if ws > 1:
        torch.distributed.destroy_process_group()


# SAGA-NN stage of each bracketed launch (SURVEY 8(a)
# S2-S5): the B200 analogue of the paper's per-stage breakdown (Fig. 5,
# lines 289, 309-310).  Fused kernels carry every stage they run.
STAGES = {
    "gcn_f32_fused": "S3+S4+S5 Scatter/Gather/ApplyVertex (fused)",
    "agg_gcn_bf16": "S3+S4 Scatter/Gather (+S5 epilogue)",
    "agg_mean_bf16": "S3+S4 Scatter/Gather",
    "agg_typed_f32": "S3+S4 Scatter/Gather",
    "agg_typed_mean_f32": "S3+S4 Scatter/Gather",
    "gat_edge": "S3+S4 Scatter/ApplyEdge/Gather (+S5 epilogue)",
    "agg_edge_mlp_f32": "S3+S4 Scatter/ApplyEdge/Gather",
    "gemm_bf16_tc_gat": "S2 pre-projection + ApplyEdge scores",
    "ggnn_edge_i8x": "S2 pre-projection (edge MLP)",
    "ggnn_heavy_b_f64": "S2 pre-projection (edge MLP, heavy rows)",
    "ggnn_split_weights": "S5 ApplyVertex (weight split)",
    "lstm_input_gemm": "S2 pre-projection (LSTM input)",
    "lstm_gather": "S4 Gather (LSTM)",
    "gated_apply_tf32x3": "S5 ApplyVertex",
    "rgcn_apply_tf32x3": "S5 ApplyVertex",
    "ggnn_gru_tf32x3": "S5 ApplyVertex",
    "gru_heavy_f64": "S5 ApplyVertex (heavy rows)",
    "sage_fused_tc": "S3+S4+S5 Scatter/Gather/ApplyVertex (fused)",
    "gcn_fused_tc": "S3+S4+S5 Scatter/Gather/ApplyVertex (fused)",
}


def stage_of(cfg, label):
    if label == "gemm_bf16_tc":  # GCN: the weight moved ahead of Scatter; SAGE/LSTM: ApplyVertex
        return "S2 pre-projection" if cfg.model == "gcn" else "S5 ApplyVertex"
    return STAGES.get(label, "other")


def stage_breakdown(cfg, trace, steps):
    """{stage: {"ms_per_step", "share"}} from region 2's spans (serialised
    launches: the stage times are upper bounds, their shares the breakdown)."""
    if not trace:
        return None
    per = {}
    for label, t0, t1 in trace:
        st = stage_of(cfg, label)
        per[st] = per.get(st, 0.0) + (t1 - t0)
    tot = sum(per.values())
    return {k: {"ms_per_step": v / steps, "share": v / tot if tot > 0 else None} for k, v in per.items()}


def write_timeline(path, cfg, trace):
    """Chrome trace-event JSON: one complete event per launch (ts/dur in us)."""
    ev = [{"name": label, "cat": stage_of(cfg, label), "ph": "X", "ts": t0 * 1e3, "dur": (t1 - t0) * 1e3,
           "pid": cfg.name, "tid": stage_of(cfg, label), "args": {"stage": stage_of(cfg, label)}}
          for label, t0, t1 in trace]
    with open(path, "w") as f:
        json.dump({"traceEvents": ev, "displayTimeUnit": "ms",
                   "otherData": {"workload": cfg.name, "source": "bench.py region 2: CUDA event pair per launch "
                                 "(saga_profile_trace), serialised launches"}}, f)


def run_e2e(args, cfg, saga, H, d, dev, ws):
    """Same metric through the public API with HOST inputs.  Every step: H2D of
    its COO + features from pinned memory, saga_graph_build, the layer step,
    D2H of its output -- a serving loop over K steps, pipelined on three
    streams so the copy-in of step i+1 and the copy-out of step i-1 overlap
    step i (double-buffered device inputs and outputs).  The timed region runs
    from the first copy-in to the last copy-out."""
    feats = [k for k in ("X", "H") if k in d]
    keys = [k for k in ("src", "dst", "etype") + tuple(feats) if isinstance(d.get(k), torch.Tensor)]
    host = {k: d[k].cpu().pin_memory() for k in keys}
    h2d = sum(host[k].numel() * host[k].element_size() for k in keys)
    weights_dev = {k: v for k, v in d.items() if k not in ("src", "dst", "etype", "X", "H")}
    main = torch.cuda.current_stream(dev)
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    inb = [{k: torch.empty_like(host[k], device=dev) for k in keys} for _ in range(2)]
    for k in keys:
        inb[0][k].copy_(host[k])
    dd0 = dict(weights_dev, **inb[0])
    dd0.setdefault("etype", None)
    g0 = H.gpu_graph(saga, cfg, dd0)
    outb = [H.gpu_step(saga, cfg, g0, dd0)[0] for _ in range(2)]   # per-slot output buffers (+ warm-up)
    g0.close()
    host_out = [torch.empty(outb[0][-1].shape, dtype=outb[0][-1].dtype, pin_memory=True) for _ in range(2)]
    in_ready = [torch.cuda.Event() for _ in range(2)]
    done = [None, None]        # main finished step i (its inputs and output slot)
    out_free = [None, None]    # the copy-out of the step that last used the slot finished
    K = max(1, args.e2e_steps)

    def copy_in(i):
        sl = i % 2
        with torch.cuda.stream(s_in):
            if done[sl] is not None:
                s_in.wait_event(done[sl])
            for k in keys:
                inb[sl][k].copy_(host[k], non_blocking=True)
            in_ready[sl].record(s_in)

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    copy_in(0)
    for i in range(K):
        sl = i % 2
        if i + 1 < K:
            copy_in(i + 1)
        main.wait_event(in_ready[sl])
        dd = dict(weights_dev, **inb[sl])
        dd.setdefault("etype", None)
        g = H.gpu_graph(saga, cfg, dd)
        if out_free[sl] is not None:
            main.wait_event(out_free[sl])
        H.gpu_step(saga, cfg, g, dd, None, outb[sl])
        ev = torch.cuda.Event()
        ev.record(main)
        done[sl] = ev
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev)
            host_out[sl].copy_(outb[sl][-1], non_blocking=True)
            fe = torch.cuda.Event()
            fe.record(s_out)
            out_free[sl] = fe
        g.close(sync=False)  # built and used on `main` only: a stream-ordered free, no host wait
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    d2h = host_out[0].numel() * host_out[0].element_size()
    tmax = max_over_ranks(dt, dev)
    return {"value": job_value(cfg.layer_updates(), K, ws, tmax * 1e3), "unit": UNIT,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": 1e3 * tmax / K, "steps": K,
            "includes": "per step: H2D COO+features (pinned), saga_graph_build, layer, D2H output; "
                        "K steps pipelined on 3 streams (copy-in i+1 | step i | copy-out i-1)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C5", choices=sorted(W.CONFIGS))
    ap.add_argument("--impl", default="saga", choices=["saga", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=12)
    ap.add_argument("--eager", action="store_true", help="launch the timed steps directly (no CUDA graph)")
    ap.add_argument("--fused", "--sage-fused", dest="sage_fused", action="store_true",
                    help="NEXT-1: Gather fused with the ApplyVertex tcgen05 GEMM in one kernel "
                         "(C2: the concat-GEMM; C5: aggregate-first GCN)")
    ap.add_argument("--ref-edges", type=int, default=2_000_000,
                    help="in-edges per oracle sample (bounded CPU work)")
    ap.add_argument("--ref-seconds", type=float, default=10.0,
                    help="cpu_baseline: grow the oracle's row sample to about this much CPU time")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-kernel-events", action="store_true",
                    help="diagnostic: no per-kernel event pairs in the timed graph (no roofline)")
    ap.add_argument("--timeline", default=None,
                    help="write region 2's per-launch spans, tagged with their SAGA stage, as a Chrome trace "
                         "(chrome://tracing / Perfetto) to this path")
    ap.add_argument("--traffic", type=float, default=None,
                    help="override: ncu dram bytes per launch of the dominant kernel "
                         "(default: profiles/ncu_traffic.json)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3   # timing rule: >= 3 warm-up steps
    cfg = W.CONFIGS[args.config]
    if args.sage_fused:
        if cfg.name not in ("C2", "C5"):
            raise SystemExit("--fused applies to the SAGE config (C2) and the GCN-at-scale config (C5)")
        cfg = W.scaled(cfg, cfg.n, cfg.m, cfg.name)
        cfg.extra["fused"] = True
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_saga(args, cfg)


if __name__ == "__main__":
    main()
