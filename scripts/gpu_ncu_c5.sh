# ncu --set full of the C5 aggregation kernel (default variant) + GAT (C3)
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:segreduce -s 1 -c 1 -o gpurun_out/agg_c5_cur python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ncu_c5.log 2>&1
