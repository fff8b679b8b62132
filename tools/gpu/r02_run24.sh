set -x
timeout 600 python tools/micro_mem.py > gpurun_out/r24_micro_mem.json 2> gpurun_out/r24_micro_mem.err; grep '^{' gpurun_out/r24_micro_mem.err | grep reduce | cut -c1-160
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -p no:cacheprovider -x -k reduce 2>&1 | tail -2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r24_ncu_c5.csv python tools/run_plan_steps.py c5_3f1b_dap 1 > gpurun_out/r24_c5_steps.log 2>&1; echo "ncu c5 $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r24_ncu_c4.csv python tools/run_plan_steps.py c4_coshard4_dp8 1 > gpurun_out/r24_c4_steps.log 2>&1; echo "ncu c4 $?"
ls -la gpurun_out/
