set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 1 -c 1 -o gpurun_out/r08_attn python tools/one_attn.py 8192 16 128 2048 0 1 > gpurun_out/r08_ncu.log 2>&1; echo "ncu rc=$?"
tail -5 gpurun_out/r08_ncu.log
ncu -i gpurun_out/r08_attn.ncu-rep --page raw --csv > gpurun_out/r08_attn_raw.csv 2>&1
ncu -i gpurun_out/r08_attn.ncu-rep --page source --csv > gpurun_out/r08_attn_source.csv 2>&1
ncu -i gpurun_out/r08_attn.ncu-rep --page details --csv > gpurun_out/r08_attn_details.csv 2>&1
ls -la gpurun_out/
