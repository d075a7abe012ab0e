# ncu --set full of the NEXT-1 fused SAGE kernel (C2, --sage-fused)
timeout 300 python bench.py --config C2 --sage-fused --steps 1 --warmup 3 --no-cpu --e2e-steps 0 --eager > gpurun_out/plain_fused.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sage_fused -s 1 -c 1 -o gpurun_out/sage_fused python bench.py --config C2 --sage-fused --steps 1 --warmup 3 --no-cpu --e2e-steps 0 --eager > gpurun_out/ncu_fused.log 2>&1
tail -2 gpurun_out/ncu_fused.log
