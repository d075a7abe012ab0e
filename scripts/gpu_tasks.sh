for t in 75776 37888 18944 9472; do for c in C5 C3 C2 C4; do
  SAGA_TASK_TARGET=$t timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/t.json 2>/dev/null
  python -c "import json;j=json.load(open('gpurun_out/t.json'));print('target $t $c', {k:round(v['avg_ms'],4) for k,v in j['config']['per_kernel'].items() if 'gemm' not in k and 'tf32' not in k})"
done; done
