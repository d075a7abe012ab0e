SAGA_AGG_DBG=3 timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/plain.log 2>&1 || exit 1
SAGA_AGG_DBG=3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:segreduce -s 1 -c 1 -o gpurun_out/agg_dbg3 python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ncu_dbg.log 2>&1
