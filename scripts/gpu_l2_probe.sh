# L2 persistence probe on C5's edge stream (scripts/l2_probe.cu).
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2_probe scripts/l2_probe.cu
python scripts/dump_colsrc.py C5 /tmp/c5_col.bin
timeout 600 /tmp/l2_probe /tmp/c5_col.bin 4194304 2>&1 | tee gpurun_out/l2_probe.txt
