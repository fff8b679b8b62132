set -x
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_parity_gpu.py tests/test_attention_gpu.py tests/test_ext_gpu.py tests/test_gemm_x3_gpu.py -q -p no:cacheprovider -rf -x > gpurun_out/r21_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r21_tests.log
for c in c2 c5 c4 c2a c2at c2x c1l; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r21_bench_$c.json 2> gpurun_out/r21_bench_$c.err; echo "$c rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/r21_bench_$c.json').read().strip().splitlines()[-1]);print('$c', round(d['ms_per_step'],4), 'plan', round(d['plan_roofline']['frac'],3), d['roofline']['kernel'], round(d['roofline']['frac'],3))"
done
timeout 600 python tools/attn_bench.py > gpurun_out/r21_attn_bench.json 2> gpurun_out/r21_attn_bench.err; grep '^{' gpurun_out/r21_attn_bench.err | head -4
timeout 600 python tools/gemm_fp32.py > gpurun_out/r21_gemm_fp32.json 2> gpurun_out/r21_gemm_fp32.err; grep '^{' gpurun_out/r21_gemm_fp32.err | head -3
