timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/plain.log 2>&1 || exit 1
for v in 5 1; do
SAGA_AGG_VARIANT=$v timeout 900 ncu --set full --clock-control none --import-source on -k regex:segreduce -s 1 -c 1 -o gpurun_out/dense_v$v python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ncu_dense_$v.log 2>&1
done
timeout 300 python bench.py --config C3 --steps 1 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:segreduce -s 1 -c 1 -o gpurun_out/gat_c3 python bench.py --config C3 --steps 1 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ncu_gat.log 2>&1
ls gpurun_out
