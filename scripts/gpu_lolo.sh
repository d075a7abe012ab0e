sed -n '/cat > \/tmp\/hub.py/,/^PY$/p' scripts/gpu_hub_err.sh | sed '1d;$d' > /tmp/hub.py
TAG=four SAGA_TF32_LOLO=1 timeout 300 python /tmp/hub.py
TAG=three SAGA_TF32_LOLO=0 timeout 300 python /tmp/hub.py
for v in 1 0; do SAGA_TF32_LOLO=$v timeout 300 python bench.py --config C4 --steps 20 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/t.json 2>/dev/null
  python -c "import json;j=json.load(open('gpurun_out/t.json'));print('lolo $v', {k:round(v['avg_ms'],4) for k,v in j['config']['per_kernel'].items()})"; done
SAGA_TF32_LOLO=0 timeout 300 python -m pytest tests -m gpu -q -k "gated or C4" 2>&1 | tail -1
