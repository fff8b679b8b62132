set -x
timeout 600 python -m pytest tests/test_gemm_x3_gpu.py tests/test_kernels_gpu.py -k "x3 or vectorised or reduce or embedding or simt" -q -p no:cacheprovider > gpurun_out/r02_new_tests.log 2>&1; echo "new rc=$?"
tail -15 gpurun_out/r02_new_tests.log
timeout 600 python tools/gemm_fp32.py > gpurun_out/r02_gemm_fp32.json 2> gpurun_out/r02_gemm_fp32.err; echo "fp32 rc=$?"
tail -3 gpurun_out/r02_gemm_fp32.err
timeout 600 python tools/micro_mem.py > gpurun_out/r02_micro_mem.json 2> gpurun_out/r02_micro_mem.err; echo "mem rc=$?"
tail -3 gpurun_out/r02_micro_mem.err
for p in c4_coshard4_dp8 c5_3f1b_dap; do timeout 300 python tools/timeline.py $p gpurun_out/r02_timeline_$p.json > gpurun_out/r02_timeline_$p.log 2>&1; echo "tl $p rc=$?"; done
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=60 > gpurun_out/r02_gputests_full.log 2>&1; echo "full rc=$?"
tail -80 gpurun_out/r02_gputests_full.log
