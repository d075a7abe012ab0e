for v in 0 1 2 3 4; do SAGA_AGG_VARIANT=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/t.json 2>/dev/null
  python -c "import json;j=json.load(open('gpurun_out/t.json'));print('C5 var $v', {k:round(v['avg_ms'],4) for k,v in j['config']['per_kernel'].items()})"; done
