set -x
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_parity_gpu.py -q -p no:cacheprovider -rf -x > gpurun_out/r17_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r17_tests.log
for v in 148 0; do
  PLANC_B200_FUSE_MIN_TILES=$v timeout 600 python bench.py --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r17_bench_c2_mt$v.json 2> gpurun_out/r17_bench_c2_mt$v.err; echo "c2 mt=$v rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/r17_bench_c2_mt$v.json').read().strip().splitlines()[-1]);print('c2 mt=$v', round(d['ms_per_step'],4), d['kernel_families'], d['roofline']['frac'], d['roofline']['frac_tensor_only'])"
  PLANC_B200_FUSE_MIN_TILES=$v timeout 600 python bench.py --config c2x --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r17_bench_c2x_mt$v.json 2> gpurun_out/r17_bench_c2x_mt$v.err; echo "c2x mt=$v rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/r17_bench_c2x_mt$v.json').read().strip().splitlines()[-1]);print('c2x mt=$v', round(d['ms_per_step'],4))"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm_tc_kernel -s 60 -c 14 --csv --log-file gpurun_out/r17_ncu_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --sustain-s 0 > /dev/null 2>&1; echo "ncu rc=$?"
