for v in 0 10 11 12; do SAGA_AGG_VARIANT=$v timeout 300 python bench.py --config C3 --steps 20 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/t.json 2>/dev/null
  python -c "import json;j=json.load(open('gpurun_out/t.json'));print('C3 var $v', {k:round(v['avg_ms'],4) for k,v in j['config']['per_kernel'].items()})"; done
for v in 0 13 14 15; do SAGA_AGG_VARIANT=$v timeout 300 python bench.py --config C4 --steps 20 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/t.json 2>/dev/null
  python -c "import json;j=json.load(open('gpurun_out/t.json'));print('C4 var $v', {k:round(v['avg_ms'],4) for k,v in j['config']['per_kernel'].items()})"; done
