set -x
start=$(date +%s)
PLANC_B200_SLOW_TESTS=1 timeout 3000 python -m pytest tests -m "gpu and slow" -q -p no:cacheprovider -rf --durations=20 > gpurun_out/slow_tests.log 2>&1; echo "slow rc=$? secs=$(( $(date +%s) - start ))"
grep -E "^FAILED|passed|failed" gpurun_out/slow_tests.log | head -20
