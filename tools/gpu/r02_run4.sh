set -x
timeout 900 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -rf -x > gpurun_out/r04_parity.log 2>&1; echo "parity rc=$?"
tail -15 gpurun_out/r04_parity.log
timeout 600 python bench.py --config c2sp --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r04_bench_c2sp.json 2> gpurun_out/r04_bench_c2sp.err; echo "c2sp rc=$?"
tail -3 gpurun_out/r04_bench_c2sp.err
python -c "import json;d=json.loads(open('gpurun_out/r04_bench_c2sp.json').read().strip().splitlines()[-1]);print('c2sp', d['ms_per_step'], d['plan_roofline']['frac'], d['gpu_launches'], d['roofline']['frac'])"
PLANC_B200_BENCH_FLAGS=0x2000 timeout 600 python bench.py --config c2sp --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r04_bench_c2sp_nogather.json 2> gpurun_out/r04_bench_c2sp_nogather.err; echo "c2sp nogather rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r04_bench_c2sp_nogather.json').read().strip().splitlines()[-1]);print('c2sp-nogather', d['ms_per_step'], d['plan_roofline']['frac'], d['gpu_launches'])"
for c in c4 c5; do
  PLANC_B200_BATCH=2 timeout 600 python bench.py --config $c --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r04_bench_${c}_batch2.json 2> gpurun_out/r04_bench_${c}_batch2.err; echo "$c batch=2 rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/r04_bench_${c}_batch2.json').read().strip().splitlines()[-1]);print('$c', 2, d['ms_per_step'], d['plan_roofline']['frac'], d['gpu_launches'])"
done
