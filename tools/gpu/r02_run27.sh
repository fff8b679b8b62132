set -x
export PLANC_B200_SKIP_SLOW=1
timeout 900 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -rf -x > gpurun_out/r27_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r27_tests.log
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --config $CFG --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r27_${CFG}_$tag.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/r27_${CFG}_$tag.json').read().strip().splitlines()[-1]);print('$CFG $tag', round(d['ms_per_step'],4), round(d['plan_roofline']['frac'],3), d['gpu_launches'], d['clocks'])"; }
for CFG in c5 c4; do
  export CFG
  run base PLANC_B200_X=0
  run nogather PLANC_B200_BENCH_FLAGS=0x2000
done
CFG=c2sp run base PLANC_B200_X=0
