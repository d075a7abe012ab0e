timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 300 python bench.py --config C6 --steps 20 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/c6.json 2>gpurun_out/c6.err; tail -3 gpurun_out/c6.err
python -c "import json;j=json.load(open('gpurun_out/c6.json'));print('C6', round(j['ms_per_step'],4), {k:round(v['avg_ms'],4) for k,v in j['config']['per_kernel'].items()})"
