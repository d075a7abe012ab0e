# ncu --set full of the NEXT-1 fused GCN kernel (C5, --fused); summary made on the box
mkdir -p gpurun_out/gf
timeout 300 python bench.py --config C5 --fused --steps 1 --warmup 3 --no-cpu --e2e-steps 0 --eager > gpurun_out/gf/plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gcn_fused -s 1 -c 1 -o gpurun_out/gf/gcn_fused python bench.py --config C5 --fused --steps 1 --warmup 3 --no-cpu --e2e-steps 0 --eager > gpurun_out/gf/ncu.log 2>&1
tail -2 gpurun_out/gf/ncu.log
python scripts/ncu_summary.py gpurun_out/gf/gcn_fused.ncu-rep > gpurun_out/gf/ncu_summary.txt 2>&1
cat gpurun_out/gf/ncu_summary.txt
ncu -i gpurun_out/gf/gcn_fused.ncu-rep --page source --csv > gpurun_out/gf/source.csv 2>/dev/null
ls -la gpurun_out/gf
