set -x
timeout 600 python -m pytest tests/test_ext_gpu.py -q -p no:cacheprovider -rf -k attn_block_train > gpurun_out/r15_ext.log 2>&1; echo "ext rc=$?"; grep -E "^FAILED|passed|failed" gpurun_out/r15_ext.log | head
for c in c2at c2a c2x; do
  timeout 600 python bench.py --config $c > gpurun_out/r15_bench_$c.json 2> gpurun_out/r15_bench_$c.err; echo "$c rc=$?"; tail -2 gpurun_out/r15_bench_$c.err
  python -c "import json;d=json.loads(open('gpurun_out/r15_bench_$c.json').read().strip().splitlines()[-1]);print('$c', round(d['ms_per_step'],4), 'plan', round(d['plan_roofline']['frac'],3), d['roofline']['kernel'], round(d['roofline']['frac'],3), d['kernel_families'])"
done
