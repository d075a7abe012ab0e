for pf in 0 4 8 16 24 32; do for v in 0 1; do
  SAGA_AGG_PF=$pf SAGA_AGG_VARIANT=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/pf_${pf}_$v.json 2>/dev/null
  python -c "import json;j=json.load(open('gpurun_out/pf_${pf}_$v.json'));print('pf $pf variant $v', j['config']['per_kernel']['agg_gcn_bf16']['avg_ms'])"
done; done
