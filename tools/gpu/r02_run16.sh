set -x
timeout 600 python -m pytest tests/test_ext_gpu.py tests/test_attention_gpu.py -q -p no:cacheprovider -rf > gpurun_out/r16_ext.log 2>&1; echo "ext rc=$?"; grep -E "^FAILED|passed|failed|^E " gpurun_out/r16_ext.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r16_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r16_smoke.log
timeout 600 python tools/attn_bench.py > gpurun_out/r16_attn_bench.json 2> gpurun_out/r16_attn_bench.err; echo "attn rc=$?"; grep '^{' gpurun_out/r16_attn_bench.err | head -4; tail -2 gpurun_out/r16_attn_bench.err
timeout 600 python bench.py --config c2at > gpurun_out/r16_bench_c2at.json 2> gpurun_out/r16_bench_c2at.err; echo "c2at rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r16_bench_c2at.json').read().strip().splitlines()[-1]);print('c2at', round(d['ms_per_step'],4), 'plan', round(d['plan_roofline']['frac'],3), d['roofline']['kernel'], round(d['roofline']['frac'],3), d['kernel_families'])"
