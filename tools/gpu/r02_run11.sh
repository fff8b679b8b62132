set -x
for v in 1 0; do
  PLANC_B200_L2HINT_STREAM=$v timeout 600 python bench.py --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r11_bench_c2_stream$v.json 2> gpurun_out/r11_bench_c2_stream$v.err; echo "c2 stream=$v rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/r11_bench_c2_stream$v.json').read().strip().splitlines()[-1]);print('c2 stream=$v', d['ms_per_step'], d['kernel_families']['gemm_tc'])"
  PLANC_B200_L2HINT_STREAM=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm_tc_kernel -s 60 -c 14 --csv --log-file gpurun_out/r11_ncu_c2_stream$v.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --sustain-s 0 > /dev/null 2>&1; echo "ncu rc=$?"
done
