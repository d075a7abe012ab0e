# NEXT-1 (C5): parity of the fused GCN kernel, then C5 bench lines with and without it.
mkdir -p gpurun_out/gf
timeout 900 python -m pytest tests -q -m gpu -x -k "gcn_fused" > gpurun_out/gf/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/gf/pytest.log; tail -6 gpurun_out/gf/pytest.log
for v in base fused; do
  fl=""; [ $v = fused ] && fl="--fused"
  timeout 400 python bench.py --config C5 --steps 20 --warmup 3 --no-cpu --e2e-steps 0 $fl > gpurun_out/gf/b_$v.json 2>gpurun_out/gf/b_$v.err
  python -c "import json;j=json.load(open('gpurun_out/gf/b_$v.json'));print('$v', round(j['ms_per_step'],4), j['config']['step_ms'], {k:round(v['avg_ms'],4) for k,v in j['config']['per_kernel'].items()})" || tail -5 gpurun_out/gf/b_$v.err
done
