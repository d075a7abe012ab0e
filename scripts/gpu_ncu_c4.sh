timeout 300 python bench.py --config C4 --steps 1 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/plain_c4.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tf32split -s 2 -c 2 -o gpurun_out/c4_gemm python bench.py --config C4 --steps 1 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ncu_c4.log 2>&1
tail -1 gpurun_out/ncu_c4.log
