# Shared-GPU split-K (>= 4 splits) default: tests + C5/C4 A/B + bench c5.
set -x
timeout 900 python -m pytest tests/test_fullsize_gpu.py -q -x -k "shared_gpu_split or c5 or c4" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "splitk" 2>&1 | tail -3
for r in 1 2; do for e in "PLANC_B200_SPLITK_SHARED=0" "X=1"; do for c in c5_3f1b_dap c4_coshard4_dp8; do env $e timeout 300 python tools/run_plan_steps.py $c 40 | sed "s/^/$e /" | tee -a gpurun_out/r37_ab.txt; done; done; done
timeout 600 python bench.py --config c5 > gpurun_out/r37_c5.json 2> gpurun_out/r37_c5.err; echo "c5 rc=$?"
