set -x
start=$(date +%s)
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --durations=40 > gpurun_out/r09_gputests.log 2>&1; echo "suite rc=$? secs=$(( $(date +%s) - start ))"
grep -E "^FAILED|passed|failed" gpurun_out/r09_gputests.log | head -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r09_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r09_smoke.log
