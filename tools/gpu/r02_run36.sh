# C5 / C4: long-k small-output dW GEMMs (2-SM BN=128, 2-4 CTAs, 40-60 us each in the C5 launch list) — stream-K / split-K A/B.
for r in 1 2; do
 for e in "X=0" "PLANC_B200_STREAMK=2" "PLANC_B200_SPLITK=2" "PLANC_B200_SPLITK_SHARED=1" "PLANC_B200_STREAMK=2 PLANC_B200_SPLITK=0"; do
  for c in c5_3f1b_dap c4_coshard4_dp8; do
   env $e timeout 300 python tools/run_plan_steps.py $c 40 | sed "s/^/$e /" | tee -a gpurun_out/r36_ab.txt
  done
 done
done
