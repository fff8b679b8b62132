# Fused short-k: 128-wide tiles by default (64-wide excluded from the eight-warp variant). Tests + A/B + bench c4.
set -x
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x 2>&1 | tail -2
for w in 0 128; do PLANC_B200_FUSED_SHORTK_BN=$w timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "fused" 2>&1 | tail -2; done
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_ext_gpu.py -q -x 2>&1 | tail -2
timeout 900 python -m pytest tests/test_fullsize_gpu.py -q -x 2>&1 | tail -2
for r in 1 2; do for e in "PLANC_B200_FUSED_SHORTK_BN=0" "X=1"; do env $e timeout 300 python tools/run_plan_steps.py c4_coshard4_dp8 40 | sed "s/^/$e /" | tee -a gpurun_out/r45_ab.txt; done; done
timeout 600 python bench.py --config c4 > gpurun_out/r45_c4.json 2> gpurun_out/r45_c4.err; echo "c4 rc=$?"
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' 2>&1 | tail -1
