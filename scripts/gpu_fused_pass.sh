# NEXT-1 (C5) evidence pass for the fused GCN kernel alone: parity tests, bench line, ncu --set full summary + stall lines.
# Usage (on the GPU box): bash scripts/gpu_fused_pass.sh <tag> <commit>
TAG=${1:-r2f}; COMMIT=${2:-unknown}
mkdir -p gpurun_out/$TAG
SAGA_PARITY_LOG=gpurun_out/$TAG/parity.json timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/$TAG/pytest_gpu.log
tail -2 gpurun_out/$TAG/pytest_gpu.log
timeout 600 python bench.py --config C5 --fused --no-cpu --e2e-steps 0 > gpurun_out/$TAG/bench_C5_fused.json 2> gpurun_out/$TAG/bench_C5_fused.err
timeout 600 python bench.py --config C5 --no-cpu --e2e-steps 0 > gpurun_out/$TAG/bench_C5.json 2> gpurun_out/$TAG/bench_C5.err
timeout 300 python bench.py --config C5 --fused --steps 1 --warmup 3 --no-cpu --e2e-steps 0 --eager > gpurun_out/$TAG/plain_C5_fused.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gcn_fused -s 1 -c 1 -o gpurun_out/$TAG/full_C5_fused \
    python bench.py --config C5 --fused --steps 1 --warmup 3 --no-cpu --e2e-steps 0 --eager > gpurun_out/$TAG/ncu_full_C5_fused.log 2>&1
python - "$TAG" "$COMMIT" <<'PY'
import json, os, sys
sys.path.insert(0, "scripts")
import make_profiles as mp
tag, commit = sys.argv[1], sys.argv[2]
src = f"gpurun_out/{tag}"
rep = f"{src}/full_C5_fused.ncu-rep"
out = [f"# ncu summary `{tag}` (commit {commit}): the fused GCN kernel, ncu --set full --clock-control none\n"]
for d in mp.read_rep(rep):
    out.append(json.dumps({k: v for k, v in d.items()}, indent=1))
open(f"{src}/{tag}_ncu_gcn_fused.md", "w").write("\n".join(out) + "\n")
mp.stall_lines(rep, f"{src}/{tag}_gcn_fused_stalls.txt")
for c in ["C5", "C5_fused"]:
    j = json.load(open(f"{src}/bench_{c}.json"))
    print(c, round(j["ms_per_step"], 4), j["config"]["step_ms"], j["clocks"])
PY
rm -f gpurun_out/$TAG/*.ncu-rep
