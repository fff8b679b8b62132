set -x
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_parity_gpu.py tests/test_attention_gpu.py -q -p no:cacheprovider -rf -x > gpurun_out/r13_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r13_tests.log
for c in c2 c2x c1l c2sp c2a c4 c5; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r13_bench_$c.json 2> gpurun_out/r13_bench_$c.err; echo "$c rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/r13_bench_$c.json').read().strip().splitlines()[-1]);print('$c', round(d['ms_per_step'],4), 'plan', round(d['plan_roofline']['frac'],3), d['roofline']['kernel'], round(d['roofline']['frac'],3), round(d['roofline'].get('frac_tensor_only',0),3))"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm_tc_kernel -s 60 -c 14 --csv --log-file gpurun_out/r13_ncu_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --sustain-s 0 > /dev/null 2>&1; echo "ncu rc=$?"
