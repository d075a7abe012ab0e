timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log; tail -2 gpurun_out/pytest_gpu.log
for d in 0 1 3; do for v in 0 1 2; do
  SAGA_AGG_VARIANT=$v SAGA_AGG_DBG=$d timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/dbg_$d.json 2>/dev/null
  python -c "import json;j=json.load(open('gpurun_out/dbg_$d.json'));print('dbg $d var $v', j['config']['per_kernel']['agg_gcn_bf16']['avg_ms'])"
done; done
