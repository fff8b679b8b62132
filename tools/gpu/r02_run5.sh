set -x
timeout 600 python -m pytest tests/test_attention_gpu.py tests/test_ext_gpu.py -q -p no:cacheprovider -rf > gpurun_out/r05_attn.log 2>&1; echo "attn rc=$?"
grep -E "^FAILED|passed|failed|Error" gpurun_out/r05_attn.log | head -30
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_kernels_gpu.py -q -p no:cacheprovider -rf > gpurun_out/r05_parity.log 2>&1; echo "parity rc=$?"
grep -E "^FAILED|passed|failed" gpurun_out/r05_parity.log | head -30
timeout 300 python tools/micro_mem.py > gpurun_out/r05_micro_mem.json 2> gpurun_out/r05_micro_mem.err; grep reduce gpurun_out/r05_micro_mem.err
