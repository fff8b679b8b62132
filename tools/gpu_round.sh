#!/bin/bash
# Round-end GPU evidence: full -m gpu suite, smoke, every bench config, C2 ncu launch list + GEMM DRAM traffic.
# Usage (on the GPU box): bash tools/gpu_round.sh v9   — outputs under gpurun_out/
V=${1:-latest}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -15 > gpurun_out/final_gpu_tests_${V}.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke_${V}.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_${V}.log
for c in c2 c2x c1l c4 c5 c3; do timeout 600 python bench.py --config $c > gpurun_out/bench_${c}_${V}.json 2> gpurun_out/bench_${c}_${V}.err; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_c2_tp1_${V}.csv python tools/run_plan_steps.py c2_tp1 1 > /dev/null 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_tc --csv --log-file gpurun_out/ncu_gemm_dram_c2_tp1_${V}.csv python tools/run_plan_steps.py c2_tp1 1 > /dev/null 2>&1
echo done
