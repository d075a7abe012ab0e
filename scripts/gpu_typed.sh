for v in 0 1 2 3; do SAGA_TYPED_VAR=$v timeout 300 python bench.py --config C4 --steps 20 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/t.json 2>/dev/null
  python -c "import json;j=json.load(open('gpurun_out/t.json'));print('typed var $v', {k:round(v['avg_ms'],4) for k,v in j['config']['per_kernel'].items()})"; done
