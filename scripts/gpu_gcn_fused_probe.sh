# Timing probes of the fused GCN kernel (results wrong by construction): GF_PROBE=1 no MMA / epilogue, 2 no row loads
for P in 0 1 2; do
  SAGA_EXTRA_NVCC_FLAGS="-DGF_PROBE=$P" python -c "import importlib.util as u,os;s=u.spec_from_file_location('b','paper_2009_00804_b200/build.py');m=u.module_from_spec(s);s.loader.exec_module(m);m.build(force=True)" > /dev/null 2>&1 || { echo build failed; continue; }
  timeout 400 python bench.py --config C5 --steps 20 --warmup 3 --no-cpu --e2e-steps 0 --fused > /tmp/b.json 2>/tmp/b.err
  python -c "import json;j=json.load(open('/tmp/b.json'));print('probe $P:', round(j['ms_per_step'],4))" || tail -3 /tmp/b.err
done
