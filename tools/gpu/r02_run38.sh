# C5 / C4 tile-width and variant sweep after shared split-K.
for r in 1 2; do for e in "X=1" "PLANC_B200_GEMM_BN=64" "PLANC_B200_GEMM_BN=128" "PLANC_B200_EPI8=2" "PLANC_B200_2SM=0" "PLANC_B200_GROUP_M=4" "PLANC_B200_STREAMS=3"; do for c in c5_3f1b_dap c4_coshard4_dp8; do env $e timeout 300 python tools/run_plan_steps.py $c 40 | sed "s/^/$e /" | tee -a gpurun_out/r38_ab.txt; done; done; done
