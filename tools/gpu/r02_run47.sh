# Final check at HEAD: full GPU suite, smoke, default bench (c2, with its reference arm), c4 / c5.
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/final_gpu_tests_v7.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke_v7.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_v7.log
timeout 600 python bench.py > gpurun_out/bench_default_v7.json 2> gpurun_out/bench_default_v7.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_v7.json 2> gpurun_out/bench_ref_v7.err; echo "ref rc=$?"
for c in c4 c5; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${c}_v7.json 2> gpurun_out/bench_${c}_v7.err; done
cat gpurun_out/final_gpu_tests_v7.log gpurun_out/smoke_v7.log
