# A/B of the fused GCN kernel's shape constants, built on the box: "warps rows-per-batch prefetch-distance" ...
# usage: bash scripts/gpu_gcn_fused_variants.sh "24 8 0" "24 8 2" ...
F=paper_2009_00804_b200/csrc/gcn_fused.cu
cp $F /tmp/gcn_fused.cu.orig
for cfg in "$@"; do
  set -- $cfg
  sed -i "s/^constexpr int kWarps = [0-9]*; /constexpr int kWarps = $1; /; s/^constexpr int kU = [0-9]*; /constexpr int kU = $2; /; s/^constexpr int kAhead = [0-9]*; /constexpr int kAhead = $3; /" $F
  python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo "build failed $cfg"; continue; }
  timeout 300 python -m pytest tests -q -m gpu -x -k "gcn_fused_next1 or gcn_fused_random" 2>&1 | tail -1
  timeout 400 python bench.py --config C5 --steps 20 --warmup 3 --no-cpu --e2e-steps 0 --fused > /tmp/b.json 2>/tmp/b.err
  python -c "import json;j=json.load(open('/tmp/b.json'));print('variant $cfg:', round(j['ms_per_step'],4), 'median', round(j['config']['step_ms']['median'],4))" || tail -3 /tmp/b.err
done
cp /tmp/gcn_fused.cu.orig $F
