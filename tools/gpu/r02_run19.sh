set -x
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_parity_gpu.py -q -p no:cacheprovider -rf -x -k "fused or golden or train or gelu" > gpurun_out/r19_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r19_tests.log
timeout 600 python bench.py --no-cpu-baseline --sustain-s 0.5 > gpurun_out/r19_bench_c2.json 2> gpurun_out/r19_bench_c2.err; echo "c2 rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r19_bench_c2.json').read().strip().splitlines()[-1]);print('c2', round(d['ms_per_step'],4), d['kernel_families']['gemm_tc'], d['roofline']['frac'], d['roofline']['frac_tensor_only'])"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm_tc_kernel -s 60 -c 14 --csv --log-file gpurun_out/r19_ncu_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --sustain-s 0 > /dev/null 2>&1; echo "ncu rc=$?"
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/r19_ncu_c2.csv')))
hdr=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hdr]; data=[dict(zip(h,r)) for r in rows[hdr+1:] if len(r)==len(h)]
by={}
for d in data: by.setdefault(d['ID'],{})[d['Metric Name']]=float(d['Metric Value'])
print('sum us', round(sum(x['gpu__time_duration.sum'] for x in by.values())/1e3,1), [round(x['gpu__time_duration.sum']/1e3,1) for x in by.values()])
PY
