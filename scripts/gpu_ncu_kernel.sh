# ncu --set full (with source) of one kernel of one config.
# Usage: CFG=C4 KREGEX=tf32split SKIP=1 COUNT=2 bash scripts/gpu_ncu_kernel.sh
CFG=${CFG:-C4}; KREGEX=${KREGEX:-tf32split}; SKIP=${SKIP:-0}; COUNT=${COUNT:-1}
timeout 300 python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu --e2e-steps 0 --eager > gpurun_out/plain_k.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s $SKIP -c $COUNT -o gpurun_out/k_$CFG python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu --e2e-steps 0 --eager > gpurun_out/ncu_k.log 2>&1
tail -2 gpurun_out/ncu_k.log
ls -la gpurun_out/k_$CFG.ncu-rep
