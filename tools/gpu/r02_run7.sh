set -x
timeout 600 python -m pytest tests/test_attention_gpu.py tests/test_ext_gpu.py -q -p no:cacheprovider -rf -x > gpurun_out/r07_attn.log 2>&1; echo "attn rc=$?"; tail -3 gpurun_out/r07_attn.log
timeout 600 python tools/attn_bench.py > gpurun_out/r07_attn_bench.json 2> gpurun_out/r07_attn_bench.err; echo "attn bench rc=$?"; grep '^{' gpurun_out/r07_attn_bench.err | head -4
