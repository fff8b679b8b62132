set -x
timeout 300 python -m pytest tests/test_ext_gpu.py -q -p no:cacheprovider -rf -k attn > gpurun_out/r06_ext.log 2>&1; echo "ext rc=$?"; tail -3 gpurun_out/r06_ext.log
timeout 600 python tools/attn_bench.py > gpurun_out/r06_attn_bench.json 2> gpurun_out/r06_attn_bench.err; echo "attn bench rc=$?"; grep '^{' gpurun_out/r06_attn_bench.err; tail -3 gpurun_out/r06_attn_bench.err
timeout 600 python bench.py --config c2a > gpurun_out/r06_bench_c2a.json 2> gpurun_out/r06_bench_c2a.err; echo "c2a rc=$?"; tail -3 gpurun_out/r06_bench_c2a.err
python -c "import json;d=json.loads(open('gpurun_out/r06_bench_c2a.json').read().strip().splitlines()[-1]);print('c2a', d['ms_per_step'], d['plan_roofline']['frac'], d['roofline']['kernel'], d['roofline']['frac'], d['kernel_families'])"
