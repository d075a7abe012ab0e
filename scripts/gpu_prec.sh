# Precision round: gated/GGNN hub tests, zoo, configs, the workspace contract; C4/C8 step times.
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python scripts/tc_accum_probe.py 2>&1 | grep -A1 "library err"
SAGA_PARITY_LOG=gpurun_out/parity_prec.json timeout 1500 python -m pytest tests/test_gpu_parity.py -q \
  -k "ggnn_aggregators or hub70k or workspace or typed_view or config_full or scaled_ragged or (layer_zoo and (gated or ggnn or rgcn)) or (random_graphs and (gated or ggnn))" \
  2>&1 | tail -15
for c in C4 C8; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err;
  python -c "import json;j=json.load(open('gpurun_out/b_$c.json'));print('$c', round(j['ms_per_step'],4), {k:round(v['avg_ms'],4) for k,v in j['config']['per_kernel'].items()})"; done
