# Full measurement pass: parity tests, bench lines for every config, ncu launch
# list of the default bench command and one --set full capture per hot kernel.
# Usage (on the GPU box): bash scripts/gpu_full.sh <tag>
TAG=${1:-r1}
mkdir -p gpurun_out/$TAG
SAGA_PARITY_LOG=gpurun_out/$TAG/parity.json timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/$TAG/pytest_gpu.log
tail -2 gpurun_out/$TAG/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$TAG/smoke.log 2>&1; tail -1 gpurun_out/$TAG/smoke.log
timeout 900 python bench.py > gpurun_out/$TAG/bench_C5.json 2> gpurun_out/$TAG/bench_C5.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/$TAG/bench_ref_C5.json 2> gpurun_out/$TAG/bench_ref_C5.err
for c in C1 C2 C3 C4 C6 C7 C8; do timeout 600 python bench.py --config $c > gpurun_out/$TAG/bench_$c.json 2> gpurun_out/$TAG/bench_$c.err; done
# NEXT-1 opt-in paths: the fused Gather + GEMM kernels (C5: gcn_fused.cu, C2: sage_fused.cu)
for c in C5 C2; do timeout 600 python bench.py --config $c --fused --no-cpu --e2e-steps 0 > gpurun_out/$TAG/bench_${c}_fused.json 2> gpurun_out/$TAG/bench_${c}_fused.err; done
for c in C1 C2 C3 C4 C5 C6 C7 C8; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --e2e-steps 0 --timeline gpurun_out/$TAG/timeline_$c.json > /dev/null 2>&1; done
for c in C1 C2 C3 C4 C5 C6 C7 C8; do python -c "import json;j=json.load(open('gpurun_out/$TAG/bench_$c.json'));print('$c', round(j['ms_per_step'],4), j['value'], {k:round(v['avg_ms'],4) for k,v in j['config']['per_kernel'].items()})"; done
# ncu: launch list of the default bench command (plain run first)
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/$TAG/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$TAG/launches_C5.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/$TAG/ncu_launch.log 2>&1
for c in C5 C3 C4 C2 C1 C6 C7 C8; do
  KRE='k_segreduce|k_rowwise|k_gemm|k_lstm|k_slice|heavy|k_gcn_epi|k_split|k_gat_maxel'; NC=9
  [ $c = C7 ] && KRE='k_lstm|k_stage_whh' && NC=6  # the LSTM pair and its W_hh staging
  timeout 300 python bench.py --config $c --steps 1 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/$TAG/plain_$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 3 -c $NC \
      -o gpurun_out/$TAG/full_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/$TAG/ncu_full_$c.log 2>&1
done
# NEXT-1 (C5): the fused GCN kernel, one --set full capture and its per-instruction stall samples
timeout 300 python bench.py --config C5 --fused --steps 1 --warmup 3 --no-cpu --e2e-steps 0 --eager > gpurun_out/$TAG/plain_C5_fused.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gcn_fused -s 1 -c 1 -o gpurun_out/$TAG/full_C5_fused \
    python bench.py --config C5 --fused --steps 1 --warmup 3 --no-cpu --e2e-steps 0 --eager > gpurun_out/$TAG/ncu_full_C5_fused.log 2>&1
ls gpurun_out/$TAG
