# usage: bash scripts/gpu_ncu_one.sh <config> <kernel-regex> <outname>
C=$1; K=$2; O=$3
timeout 300 python bench.py --config $C --steps 1 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/plain_$O.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/$O python bench.py --config $C --steps 1 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ncu_$O.log 2>&1
tail -2 gpurun_out/ncu_$O.log
