set -x
nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_gputests.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r02_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err; echo "bench rc=$?"
cat gpurun_out/r02_bench_c2.json
for c in c1l c2x c3 c4 c5; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.err; echo "$c rc=$?"; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02_bench_ref.json 2>&1; echo "ref rc=$?"
