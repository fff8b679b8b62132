set -x
timeout 600 python bench.py --config c5 --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r28_c5.json 2> gpurun_out/r28_c5.err; echo "c5 rc=$?"; tail -5 gpurun_out/r28_c5.err; tail -c 300 gpurun_out/r28_c5.json
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --config $CFG --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r28_${CFG}_$tag.json 2>gpurun_out/r28_${CFG}_$tag.err; python -c "import json;d=json.loads(open('gpurun_out/r28_${CFG}_$tag.json').read().strip().splitlines()[-1]);print('$CFG $tag', round(d['ms_per_step'],4), round(d['plan_roofline']['frac'],3), d['gpu_launches'], d['clocks'])"; }
CFG=c2 run base PLANC_B200_X=0
CFG=c2sp run base PLANC_B200_X=0
CFG=c2sp run nogather PLANC_B200_BENCH_FLAGS=0x2000
