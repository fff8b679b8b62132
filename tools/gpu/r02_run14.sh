set -x
timeout 600 python -m pytest tests/test_attention_gpu.py tests/test_ext_gpu.py -q -p no:cacheprovider -rf > gpurun_out/r14_attn.log 2>&1; echo "attn rc=$?"; grep -E "^FAILED|passed|failed|Error|assert" gpurun_out/r14_attn.log | head -30
