python -c "import __graft_entry__ as g; g.build()"
timeout 600 python scripts/tc_accum_probe.py 2>&1 | tee gpurun_out/tc_probe.txt
timeout 300 bash scripts/gpu_hub_err.sh 2>&1 | tee gpurun_out/hub_err.txt
