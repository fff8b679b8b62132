# Profile with a host gate (per-instruction events without host launch latency): bench lines c2 / c5 / c4 + C5 launch list.
set -x
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "profile or timeline or e2e" 2>&1 | tail -3
for c in c2 c5 c4; do timeout 600 python bench.py --config $c --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r35_$c.json 2> gpurun_out/r35_$c.err; echo "$c rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r35_$c.json').read().strip().splitlines()[-1]);print('$c', round(d['ms_per_step'],4), json.dumps(d['roofline'])[:300]); print(json.dumps(d.get('kernel_families')))"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r35_ncu_c5.csv python tools/run_plan_steps.py c5_3f1b_dap 1 > gpurun_out/r35_ncu_c5.log 2>&1; echo "ncu $?"
