# ncu --set full of C4's fused short-k GEMM (16384x512x512 + add), then the round-end evidence run (v5).
set -x
timeout 300 python tools/one_fused.py fused 16384 512 512 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -c 1 -o gpurun_out/r43_fused_shortk python tools/one_fused.py fused 16384 512 512 > gpurun_out/r43_ncu.log 2>&1; echo "ncu $?"
ncu -i gpurun_out/r43_fused_shortk.ncu-rep --page source --csv --print-source sass > gpurun_out/r43_source.csv 2>/dev/null; echo "src $?"
ncu -i gpurun_out/r43_fused_shortk.ncu-rep --page raw --csv > gpurun_out/r43_raw.csv 2>/dev/null
bash tools/gpu_round.sh v5
