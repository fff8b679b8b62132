# Plain short-k GEMMs on 128-wide tiles (A/B): C4 / C5 / C2x / C3.
PLANC_B200_SHORTK_BN=128 timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x 2>&1 | tail -2
for r in 1 2; do for e in "X=1" "PLANC_B200_SHORTK_BN=128"; do for c in c4_coshard4_dp8 c5_3f1b_dap c2x_tp1 c1l_dp1; do env $e timeout 300 python tools/run_plan_steps.py $c 40 | sed "s/^/$e /" | tee -a gpurun_out/r46_ab.txt; done; done; done
