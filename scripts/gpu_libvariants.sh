# A/B of prebuilt library variants (scripts/variants/libsaga_<name>.so, made
# with SAGA_EXTRA_NVCC_FLAGS): bench step time per config for each variant.
for lib in ${LIBS}; do cp scripts/variants/libsaga_$lib.so paper_2009_00804_b200/libsaga.so; for c in ${CONFIGS:-C5}; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --e2e-steps 0 $EXTRA > gpurun_out/b_$c.json 2>&1;
  python -c "import json;j=json.load(open('gpurun_out/b_$c.json'));print('$lib $c', round(j['ms_per_step'],4), round(j['config']['ms_per_step_profiled'],4), {k:round(v['avg_ms'],4) for k,v in j['config']['per_kernel'].items()})"; done; done
