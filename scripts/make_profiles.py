"""Summarise a gpurun measurement pass (scripts/gpu_full.sh) into profiles/.

  python scripts/make_profiles.py <tag> [<commit>]

Writes profiles/<tag>_ncu_summary.md (per config and kernel: duration, DRAM
read/write bytes, L2 hit rate, occupancy, issue activity, top stall reasons),
profiles/<tag>_launches_C5.csv (+ kernel shares), the bench JSON lines, and
profiles/ncu_traffic.json (DRAM bytes per launch per config/kernel label, read
by bench.py for roofline.traffic).
"""
import csv
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LABELS = {  # config -> [(substring of the ncu kernel name, bench/profile label)]
    "C1": [("GcnF32FusedOp", "gcn_f32_fused")],
    "C2": [("SumBf16Op", "agg_mean_bf16"), ("k_gemm_bf16_tc", "gemm_bf16_tc")],
    "C3": [("GatShiftOp", "gat_edge"), ("k_gat_maxel", "gat_edge"), ("k_gemm_bf16_tc", "gemm_bf16_tc_gat")],
    "C4": [("SumF32Op", "agg_typed_f32"), ("k_gemm_tf32split", "gated_apply_tf32x3"), ("k_split_weights", "gated_apply_tf32x3"),
           ("k_gru_heavy_f64", "gru_heavy_f64")],
    "C5": [("SumBf16Op", "agg_gcn_bf16"), ("k_gcn_epi_rows", "agg_gcn_bf16"), ("k_gemm_bf16_tc", "gemm_bf16_tc")],
    "C6": [("SumF32Op", "agg_typed_mean_f32"), ("k_gemm_tf32split", "rgcn_apply_tf32x3"), ("k_split_rgcn", "rgcn_apply_tf32x3")],
    "C7": [("k_lstm_cluster", "lstm_gather"), ("k_lstm_mma", "lstm_gather"), ("k_stage_whh", "lstm_gather"),
           ("k_gemm_bf16_tc", "gemm_bf16_tc")],
    "C5_fused": [("k_gcn_fused", "gcn_fused_tc")],
    "C8": [("EdgeMlpOp", "agg_edge_mlp_f32"), ("k_gemm_tf32split<256", "ggnn_gru_tf32x3"),
           ("k_gemm_i8x", "ggnn_edge_i8x"), ("k_slice_rows", "ggnn_edge_i8x"), ("k_slice_wt_ggnn", "ggnn_edge_i8x"),
           ("k_split_ggnn", "ggnn_split_weights"), ("k_ggnn_heavy_b", "ggnn_heavy_b_f64"),
           ("k_gru_heavy_f64", "gru_heavy_f64")],
}
WANT = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "dram_read"),
        ("dram__bytes_write.sum", "dram_write"), ("lts__t_sector_hit_rate.pct", "L2_hit_%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_%"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_throughput_%"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_pipe_%"),
        ("launch__registers_per_thread", "regs"), ("smsp__inst_executed.sum", "warp_inst")]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}


def label_of(cfg, name):
    for sub, lab in LABELS[cfg]:
        if sub in name:
            return lab
    return None


def read_rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, units = r[0], r[1]
    rows = []
    for row in r[2:]:
        d = {"name": row[h.index("Kernel Name")]}
        for key, short in WANT:
            if key in h:
                i = h.index(key)
                try:
                    v = float(row[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if short.startswith("dram_r") or short.startswith("dram_w"):
                    v *= SCALE.get(u, 1)
                if short == "duration":
                    v *= SCALE.get(u, 1)  # -> ms
                d[short] = v
        stalls = []
        for i, a in enumerate(h):
            if a.startswith("smsp__pcsamp_warps_issue_stalled_") and not a.endswith("not_issued"):
                try:
                    stalls.append((float(row[i].replace(",", "")), a.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1
        d["stalls"] = ", ".join(f"{n} {100 * s / tot:.0f}%" for s, n in sorted(stalls, reverse=True)[:4])
        rows.append(d)
    return rows


def stall_lines(rep, out_path, top=30):
    """The SASS instructions holding the most warp-stall samples (ncu source page)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = next((i for i, r in enumerate(rows) if r and r[0] == "Address"), None)
    if hdr is None:
        return
    body = [r for r in rows[hdr + 1:] if len(r) > 5]
    tot = sum(int(r[2]) for r in body) or 1
    idx = sorted(range(len(body)), key=lambda i: -int(body[i][2]))[:top]
    lines = [f"# {os.path.basename(rep)}: SASS lines by warp-stall samples (all samples {tot}); index, instruction, "
             "samples, share, warp-level executions"]
    for i in sorted(idx):
        r = body[i]
        lines.append(f"{i:5d}  {r[1].strip()[:90]:90s} {r[2]:>8s} {100 * int(r[2]) / tot:5.1f}%  exec {r[5]}")
    open(out_path, "w").write("\n".join(lines) + "\n")


def main(tag, commit="unknown"):
    src = os.path.join(ROOT, "gpurun_out", tag)
    dst = os.path.join(ROOT, "profiles")
    os.makedirs(dst, exist_ok=True)
    traffic_path = os.path.join(dst, "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    md = [f"# ncu summary `{tag}` (ncu --set full --clock-control none; cold-cache replays)\n"]
    for cfg in ["C1", "C2", "C3", "C4", "C5", "C6", "C7", "C8", "C5_fused"]:
        rep = os.path.join(src, f"full_{cfg}.ncu-rep")
        if not os.path.exists(rep):
            continue
        md.append(f"\n## {cfg}\n")
        md.append("| kernel | label | ms | DRAM read GB | DRAM write GB | L2 hit % | DRAM thr % | tensor % | warps act % | issue % | regs | top stalls |")
        md.append("|---|---|---|---|---|---|---|---|---|---|---|---|")
        per = defaultdict(lambda: defaultdict(list))  # label -> kernel name -> DRAM bytes per launch
        for d in read_rep(rep):
            lab = label_of(cfg, d["name"])
            short = d["name"].split("(")[0][:60]
            md.append(f"| `{short}` | {lab} | {d.get('duration', 0):.4f} | {d.get('dram_read', 0) / 1e9:.3f} | "
                      f"{d.get('dram_write', 0) / 1e9:.3f} | {d.get('L2_hit_%', 0):.1f} | {d.get('dram_throughput_%', 0):.1f} | "
                      f"{d.get('tensor_pipe_%', 0):.1f} | {d.get('warps_active_%', 0):.1f} | {d.get('issue_active_%', 0):.1f} | "
                      f"{d.get('regs', 0):.0f} | {d['stalls']} |")
            if lab:
                per[lab][d["name"].split("(")[0]].append(d.get("dram_read", 0) + d.get("dram_write", 0))
        # a label's traffic per call: the mean of each of its kernels, summed over its kernels
        t = {lab: sum(sum(v) / len(v) for v in ks.values()) for lab, ks in per.items()}
        base = cfg.split("_")[0]  # "C5_fused" (the opt-in NEXT-1 kernel) files under C5
        if base == cfg:
            traffic[cfg] = t
        else:
            traffic.setdefault(base, {}).update(t)
        if cfg == "C5_fused":
            stall_lines(rep, os.path.join(dst, f"{tag}_gcn_fused_stalls.txt"))
    traffic["_commit"] = commit
    traffic["_when"] = tag
    open(os.path.join(dst, f"{tag}_ncu_summary.md"), "w").write("\n".join(md) + "\n")
    json.dump(traffic, open(traffic_path, "w"), indent=1)
    # launch list of the default bench command: shares per kernel
    lc = os.path.join(src, "launches_C5.csv")
    if os.path.exists(lc):
        shutil.copy(lc, os.path.join(dst, f"{tag}_launches_C5.csv"))
        rows = list(csv.reader(open(lc)))
        hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
        h = rows[hdr]
        agg = defaultdict(lambda: [0, 0.0])
        for r in rows[hdr + 1:]:
            d = dict(zip(h, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                k = d["Kernel Name"].split("(")[0]
                agg[k][0] += 1
                agg[k][1] += float(d["Metric Value"].replace(",", "")) / 1e6
        ours = {k: v for k, v in agg.items() if "saga" in k}
        tot = sum(v[1] for v in ours.values())
        lines = [f"# launch list of `python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0` ({tag})",
                 "# libsaga kernels only (torch's input-generation kernels omitted); ncu per-launch times are",
                 "# cold-cache and serialised: compare shares, not absolutes", "kernel,launches,total_ms,share"]
        for k, (n, t) in sorted(ours.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"{k},{n},{t:.4f},{t / tot:.4f}")
        open(os.path.join(dst, f"{tag}_launch_shares_C5.csv"), "w").write("\n".join(lines) + "\n")
    for cfg in ["C1", "C2", "C3", "C4", "C5", "C6", "C7", "C8", "C5_fused", "C2_fused"]:
        b = os.path.join(src, f"bench_{cfg}.json")
        if os.path.exists(b):
            shutil.copy(b, os.path.join(dst, f"{tag}_bench_{cfg}.json"))
    for extra in ["bench_ref_C5.json", "pytest_gpu.log", "smoke.log", "parity.json"]:
        b = os.path.join(src, extra)
        if os.path.exists(b):
            shutil.copy(b, os.path.join(dst, f"{tag}_{extra}"))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "unknown")
