set -x
timeout 300 python -m pytest tests/test_gemm_x3_gpu.py -q -p no:cacheprovider -rf > gpurun_out/r03_x3.log 2>&1; echo "x3 rc=$?"
tail -15 gpurun_out/r03_x3.log
timeout 600 python tools/gemm_fp32.py > gpurun_out/r03_gemm_fp32.json 2> gpurun_out/r03_gemm_fp32.err; echo "fp32 rc=$?"
grep '^{' gpurun_out/r03_gemm_fp32.err
for f in test_parity_gpu test_ext_gpu test_dropin_gpu test_kernels_gpu; do
  timeout 900 python -m pytest tests/$f.py -q -p no:cacheprovider -rf --durations=15 > gpurun_out/r03_$f.log 2>&1; echo "$f rc=$?"
  grep -E "^FAILED|passed|failed" gpurun_out/r03_$f.log | head -20
done
for c in c4 c5 c2; do
  for b in 1 0; do
    PLANC_B200_BATCH=$b timeout 600 python bench.py --config $c --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r03_bench_${c}_batch$b.json 2> gpurun_out/r03_bench_${c}_batch$b.err; echo "$c batch=$b rc=$?"
    python -c "import json;d=json.loads(open('gpurun_out/r03_bench_${c}_batch$b.json').read().strip().splitlines()[-1]);print('$c', $b, d['ms_per_step'], d['plan_roofline']['frac'], d['gpu_launches'])"
  done
done
