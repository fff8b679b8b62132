set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r31_ncu_c5_gather.csv python tools/run_plan_steps.py c5_3f1b_dap 1 > gpurun_out/r31_a.log 2>&1; echo "a $?"
python tools/run_plan_steps.py c5_3f1b_dap 30; python tools/run_plan_steps.py c5_3f1b_dap 30 0x2000
