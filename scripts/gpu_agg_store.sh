for st in 0 1 2; do for v in 0 3; do
  SAGA_AGG_STORE=$st SAGA_AGG_VARIANT=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/st_${st}_$v.json 2>/dev/null
  python -c "import json;j=json.load(open('gpurun_out/st_${st}_$v.json'));print('store $st variant $v', {k:v['avg_ms'] for k,v in j['config']['per_kernel'].items()})"
done; done
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/plain.log 2>&1 && \
SAGA_AGG_VARIANT=3 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:segreduce -s 1 -c 1 -o gpurun_out/agg_c5_v3 python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ncu_agg.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o /tmp/gather_probe scripts/gather_probe.cu
python scripts/dump_colsrc.py C5 /tmp/c5_col.bin
ncu --set full --clock-control none -k regex:k_gather -s 5 -c 1 -o gpurun_out/probe_u8_pol1 /tmp/gather_probe /tmp/c5_col.bin 4194304 > gpurun_out/ncu_probe.log 2>&1
tail -3 gpurun_out/ncu_probe.log
