# Quick check: GPU parity suite + a 20-step bench line per config (kernel times).
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log; tail -4 gpurun_out/pytest_gpu.log
for c in C1 C2 C3 C4 C5 C6 C7 C8; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/b_$c.json 2>&1;
  python -c "import json;j=json.load(open('gpurun_out/b_$c.json'));print('$c', round(j['ms_per_step'],4), {k:round(v['avg_ms'],4) for k,v in j['config']['per_kernel'].items()})"; done
