set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 2 -c 1 -o gpurun_out/r18_fused python tools/one_fused.py fused 8192 8192 2048 > gpurun_out/r18_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/r18_fused.ncu-rep --page raw --csv > gpurun_out/r18_fused_raw.csv 2>&1
ncu -i gpurun_out/r18_fused.ncu-rep --page source --csv > gpurun_out/r18_fused_source.csv 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 2 -c 1 -o gpurun_out/r18_plain python tools/one_fused.py gemm 8192 8192 2048 > gpurun_out/r18_ncu2.log 2>&1; echo "ncu2 rc=$?"
ncu -i gpurun_out/r18_plain.ncu-rep --page raw --csv > gpurun_out/r18_plain_raw.csv 2>&1
rm -f gpurun_out/*.ncu-rep
