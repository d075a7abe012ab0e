# Aggregation-engine variants on C5 + parity; usage: bash scripts/gpu_agg_variants.sh
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
for v in 0 1 2 3; do
  SAGA_AGG_VARIANT=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
  python -c "import json;j=json.load(open('gpurun_out/var_$v.json'));print('variant $v', j['ms_per_step'], {k:v['avg_ms'] for k,v in j['config']['per_kernel'].items()})"
done
for c in C1 C2 C3 C4; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/b_$c.json 2>&1;
  python -c "import json;j=json.load(open('gpurun_out/b_$c.json'));print('$c', j['ms_per_step'], {k:v['avg_ms'] for k,v in j['config']['per_kernel'].items()})"; done
