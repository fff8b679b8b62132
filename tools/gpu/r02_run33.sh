# Fused epilogue: operand prefetch two chunks ahead (one-slot ops). Parity + timing.
set -x
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "fused or two_sm" 2>&1 | tail -5
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x 2>&1 | tail -5
timeout 600 python tools/fuse_micro.py > gpurun_out/r33_fuse_micro.json 2> gpurun_out/r33_fuse_micro.err; tail -20 gpurun_out/r33_fuse_micro.json
for i in 1 2; do timeout 600 python bench.py --config c2 --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r33_c2_$i.json 2> gpurun_out/r33_c2_$i.err; python -c "import json,sys;d=json.loads(open('gpurun_out/r33_c2_$i.json').read().strip().splitlines()[-1]);print('c2', round(d['ms_per_step'],4), d['roofline']['frac'], d['clocks'])"; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm_tc --csv --log-file gpurun_out/r33_ncu_c2.csv python tools/run_plan_steps.py c2_tp1 1 > /dev/null 2>&1; echo ncu $?
