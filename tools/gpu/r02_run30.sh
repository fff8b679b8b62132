set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r30_ncu_c5_gather.csv python tools/run_plan_steps.py c5_3f1b_dap 1 > gpurun_out/r30_a.log 2>&1; echo "a $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r30_ncu_c5_nogather.csv python tools/run_plan_steps.py c5_3f1b_dap 1 0x2000 > gpurun_out/r30_b.log 2>&1; echo "b $?"
python tools/run_plan_steps.py c5_3f1b_dap 30; python tools/run_plan_steps.py c5_3f1b_dap 30 0x2000
