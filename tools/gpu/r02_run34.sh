# Critical-path launch priorities: A/B (PLANC_B200_PRIORITY=0 vs default on), C5 / C4 / C2 / C2x / C3.
set -x
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x 2>&1 | tail -3
for r in 1 2; do
 for p in 0 1; do
  for c in c5_3f1b_dap c4_coshard4_dp8 c2_tp1 c2x_tp1; do
   PLANC_B200_PRIORITY=$p timeout 300 python tools/run_plan_steps.py $c 40 | sed "s/^/prio=$p /" | tee -a gpurun_out/r34_ab.jsonl
  done
 done
done
for p in 0 1; do PLANC_B200_PRIORITY=$p timeout 600 python tools/run_plan_steps.py c3_pp4dp2_l24 4 0x800 | sed "s/^/prio=$p /" | tee -a gpurun_out/r34_ab.jsonl; done
