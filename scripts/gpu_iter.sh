# Iteration helper: build, a pytest -k subset, bench lines and an ncu launch list.
# usage: bash scripts/gpu_iter.sh "<pytest -k expr or ''>" "<configs>" "<ncu config or ''>"
python -c "import __graft_entry__ as g; g.build()" || exit 1
if [ -n "$1" ]; then
  SAGA_PARITY_LOG=gpurun_out/parity_iter.json timeout 2400 python -m pytest tests -q -m gpu -k "$1" 2>&1 | tail -8
fi
for c in $2; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err;
  python -c "import json;j=json.load(open('gpurun_out/b_$c.json'));print('$c', round(j['ms_per_step'],4), {k:round(v['avg_ms'],4) for k,v in j['config']['per_kernel'].items()})" || tail -5 gpurun_out/b_$c.err; done
if [ -n "$3" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 40 --csv --log-file gpurun_out/launches_$3.csv \
    python bench.py --config $3 --steps 2 --warmup 3 --no-cpu --e2e-steps 0 --no-kernel-events > /dev/null 2>&1
  python - "$3" <<'PY'
import csv, sys, collections
rows = list(csv.reader(l for l in open(f"gpurun_out/launches_{sys.argv[1]}.csv") if not l.startswith("==")))
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[1:]:
    if len(r) <= vi: continue
    k = r[ki][:90]; agg.setdefault(k, []).append(float(r[vi].replace(",", "")) / 1000)
for k, v in agg.items(): print(f"{sum(v)/len(v):9.1f} us x{len(v):3d}  {k}")
PY
fi
