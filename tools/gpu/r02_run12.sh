set -x
for c in c5 c4 c3; do
  for mc in 8 16 32; do
    CUDA_DEVICE_MAX_CONNECTIONS=$mc timeout 600 python bench.py --config $c --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r12_bench_${c}_mc$mc.json 2> gpurun_out/r12_bench_${c}_mc$mc.err; echo "$c mc=$mc rc=$?"
    python -c "import json;d=json.loads(open('gpurun_out/r12_bench_${c}_mc$mc.json').read().strip().splitlines()[-1]);print('$c mc=$mc', d['ms_per_step'], d['plan_roofline']['frac'])"
  done
done
