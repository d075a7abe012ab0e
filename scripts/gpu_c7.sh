timeout 1200 python -m pytest tests -m gpu -q -x -k "sage_lstm or C7" 2>&1 | tail -5
timeout 300 python bench.py --config C7 --steps 5 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/c7.json 2>gpurun_out/c7.err; tail -3 gpurun_out/c7.err
python -c "import json;j=json.load(open('gpurun_out/c7.json'));print('C7', round(j['ms_per_step'],4), {k:round(v['avg_ms'],4) for k,v in j['config']['per_kernel'].items()})"
python - <<'PY'
import sys; sys.path.insert(0, '.')
import workloads as W, torch
c = W.CONFIGS['C7']; s, d, _ = W.make_graph(c, 'cuda')
deg = torch.bincount(d.long(), minlength=c.n)
print('C7 max in-degree', int(deg.max()), 'edges', d.numel(), 'distinct degrees', int(torch.unique(deg).numel()))
PY
