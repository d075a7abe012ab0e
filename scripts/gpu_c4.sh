timeout 600 python -m pytest tests -m gpu -x -q -k "gated or C4" > gpurun_out/pytest_c4.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_c4.log; tail -15 gpurun_out/pytest_c4.log
timeout 300 python bench.py --config C4 --steps 20 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/c4.json 2>gpurun_out/c4.err; tail -3 gpurun_out/c4.err
python -c "import json;j=json.load(open('gpurun_out/c4.json'));print('C4', round(j['ms_per_step'],4), {k:round(v['avg_ms'],4) for k,v in j['config']['per_kernel'].items()})"
