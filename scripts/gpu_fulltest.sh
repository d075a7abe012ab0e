# Full GPU parity suite with the per-check error log, plus the precision probe.
python -c "import __graft_entry__ as g; g.build()" || exit 1
SAGA_PARITY_LOG=gpurun_out/parity_full.json timeout 3000 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 | tee gpurun_out/pytest_full.txt
timeout 600 python scripts/tc_accum_probe.py > gpurun_out/tc_probe.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
