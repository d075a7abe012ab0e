# Raw row-gather throughput probe on C5's edge stream (scripts/gather_probe.cu):
# register loads (the engine's scheme) vs TMA bulk-copy staging in shared memory.
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gather_probe scripts/gather_probe.cu
python scripts/dump_colsrc.py C5 /tmp/c5_col.bin
/tmp/gather_probe /tmp/c5_col.bin 4194304 | tee gpurun_out/gather_probe_r2.txt
