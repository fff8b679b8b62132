set -x
for i in 1 2; do python tools/run_plan_steps.py c5_3f1b_dap 30; python tools/run_plan_steps.py c5_3f1b_dap 30 0x2000; done
timeout 600 python bench.py --config c5 --no-cpu-baseline --sustain-s 0.3 > gpurun_out/r32_c5.json 2> gpurun_out/r32_c5.err; echo "c5 rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r32_c5.json').read().strip().splitlines()[-1]);print('c5', round(d['ms_per_step'],4), round(d['plan_roofline']['frac'],3), d['gpu_launches'], d['clocks'])"
