set -x
python scripts/dump_colsrc.py C5 /tmp/c5_col.bin
./scripts/gather_probe /tmp/c5_col.bin 4194304 > gpurun_out/probe1.txt 2>&1
cat gpurun_out/probe1.txt
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:segreduce -s 1 -c 1 -o gpurun_out/agg_c5_v1 python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ncu_agg.log 2>&1
tail -5 gpurun_out/ncu_agg.log
