# A/B of development knobs (env VAR over values VALS), kernel times per config.
# EXTRA: extra bench.py arguments (e.g. --no-kernel-events).
for v in ${VALS:-0 1 2 3}; do for c in ${CONFIGS:-C5}; do env $VAR=$v timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --e2e-steps 0 $EXTRA > gpurun_out/b_$c.json 2>&1;
  python -c "import json;j=json.load(open('gpurun_out/b_$c.json'));print('$VAR=$v $c', round(j['ms_per_step'],4), {k:round(v['avg_ms'],4) for k,v in j['config']['per_kernel'].items()})"; done; done
