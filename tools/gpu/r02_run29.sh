set -x
timeout 900 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -rf -x -k "full_size or gathered or box_elementwise or views" > gpurun_out/r29_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r29_tests.log
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --config $CFG --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r29_${CFG}_$tag.json 2>gpurun_out/r29_${CFG}_$tag.err; python -c "import json;d=json.loads(open('gpurun_out/r29_${CFG}_$tag.json').read().strip().splitlines()[-1]);print('$CFG $tag', round(d['ms_per_step'],4), round(d['plan_roofline']['frac'],3), d['gpu_launches'], d['clocks'])"; }
CFG=c5 run base PLANC_B200_X=0
CFG=c5 run nogather PLANC_B200_BENCH_FLAGS=0x2000
CFG=c2 run base PLANC_B200_X=0
CFG=c5 run base2 PLANC_B200_X=0
