set -x
timeout 900 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k "batching or launch_modes or golden_plan_parity" > gpurun_out/r03_parity.log 2>&1; echo "parity rc=$?"
tail -5 gpurun_out/r03_parity.log
for c in c4 c5 c3 c2; do
  for b in 1 0; do
    PLANC_B200_BATCH=$b timeout 600 python bench.py --config $c --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r03_bench_${c}_batch$b.json 2> gpurun_out/r03_bench_${c}_batch$b.err; echo "$c batch=$b rc=$?"
    python -c "import json;d=json.loads(open('gpurun_out/r03_bench_${c}_batch$b.json').read().strip().splitlines()[-1]);print('$c', $b, d['ms_per_step'], d['plan_roofline']['frac'], d['gpu_launches'])"
  done
done
