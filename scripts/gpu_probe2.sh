set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gather_probe scripts/gather_probe.cu
python scripts/dump_colsrc.py C5 /tmp/c5_col.bin
/tmp/gather_probe /tmp/c5_col.bin 4194304 > gpurun_out/probe2.txt 2>&1
for pol in 0 1 2 3; do for v in 0 2 1; do
  SAGA_AGG_LDPOL=$pol SAGA_AGG_VARIANT=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/pv_${pol}_$v.json 2>/dev/null
  echo "pol $pol var $v $(python -c "import json;j=json.load(open('gpurun_out/pv_${pol}_$v.json'));print(j['config']['per_kernel']['agg_gcn_bf16']['avg_ms'])")" >> gpurun_out/probe2.txt
done; done
for pol in 0 1 3; do SAGA_AGG_LDPOL=$pol timeout 300 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/c3_$pol.json 2>/dev/null
  echo "C3 pol $pol $(python -c "import json;j=json.load(open('gpurun_out/c3_$pol.json'));print(j['config']['per_kernel'])")" >> gpurun_out/probe2.txt; done
cat gpurun_out/probe2.txt
