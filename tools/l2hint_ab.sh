#!/bin/bash
# A/B of the GEMM operand L2 eviction hints (PLANC_B200_L2HINT 0/1/2) on the
# C2 k=8192 shapes: per-shape step time, ncu DRAM bytes, then the C2 bench.
out=gpurun_out/l2hint
mkdir -p $out
shapes=("8192 2048 8192 0 0" "8192 2048 8192 1 0" "8192 2048 8192 0 1" "2048 8192 8192 1 0" "8192 8192 2048 0 0")
for mode in 0 1 2; do
  for sh in "${shapes[@]}"; do
    PLANC_B200_L2HINT=$mode timeout 120 python tools/one_gemm.py $sh 1 20 >> $out/time_$mode.txt 2>&1
  done
  PLANC_B200_L2HINT=$mode timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:gemm_tc --csv python tools/one_gemm.py 8192 2048 8192 1 0 1 2 > $out/ncu_gw2w_$mode.csv 2>/dev/null
  PLANC_B200_L2HINT=$mode timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:gemm_tc --csv python tools/one_gemm.py 2048 8192 8192 1 0 1 2 > $out/ncu_gf1w_$mode.csv 2>/dev/null
  PLANC_B200_L2HINT=$mode timeout 300 python bench.py --no-cpu-baseline --steps 50 --sustain-s 1 > $out/bench_$mode.json 2>/dev/null
done
PLANC_B200_L2HINT=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:gemm_tc --csv python bench.py --no-cpu-baseline --steps 1 --warmup 3 --sustain-s 0 > $out/ncu_c2_launches_hint1.csv 2>/dev/null
