set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for c in C1 C2 C3 C4; do timeout 600 python bench.py --config $c --steps 50 --warmup 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 900 python bench.py > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
cat gpurun_out/bench_*.json
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C5.csv python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ncu_launch.log 2>&1
echo done
