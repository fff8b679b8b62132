# Fused short-k GEMMs on eight epilogue warps (OCC 3): tests + C4 A/B + bench c4 + ncu C4 list.
set -x
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "fused or epi" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_ext_gpu.py -q -x 2>&1 | tail -3
timeout 900 python -m pytest tests/test_fullsize_gpu.py -q -x -k "c4 or c5 or c2_tp1" 2>&1 | tail -3
for r in 1 2; do for e in "PLANC_B200_EPI8_FUSED=0" "X=1"; do for c in c4_coshard4_dp8 c2_tp1 c2x_tp1; do env $e timeout 300 python tools/run_plan_steps.py $c 40 | sed "s/^/$e /" | tee -a gpurun_out/r41_ab.txt; done; done; done
timeout 600 python bench.py --config c4 > gpurun_out/r41_c4.json 2> gpurun_out/r41_c4.err; echo "c4 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r41_ncu_c4.csv python tools/run_plan_steps.py c4_coshard4_dp8 1 > /dev/null 2>&1; echo "ncu $?"
