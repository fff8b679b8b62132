# C4: short-k GEMM variants (16384x512x512 plain / fused: 2-3x off their HBM / tensor balance point in the launch list)
for r in 1 2; do for e in "X=1" "PLANC_B200_2SM=2" "PLANC_B200_OCC2=2" "PLANC_B200_EPI8=0" "PLANC_B200_GROUP_M=16" "PLANC_B200_L2HINT=0"; do env $e timeout 300 python tools/run_plan_steps.py c4_coshard4_dp8 40 | sed "s/^/$e /" | tee -a gpurun_out/r40_ab.txt; done; done
