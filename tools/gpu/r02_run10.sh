set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 2 -c 1 -o gpurun_out/r10_fused python tools/one_fused.py fused 8192 8192 2048 > gpurun_out/r10_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/r10_fused.ncu-rep --page raw --csv > gpurun_out/r10_fused_raw.csv 2>&1
ncu -i gpurun_out/r10_fused.ncu-rep --page source --csv > gpurun_out/r10_fused_source.csv 2>&1
ncu -i gpurun_out/r10_fused.ncu-rep --page details --csv > gpurun_out/r10_fused_details.csv 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 1 -c 1 -o gpurun_out/r10_attn python tools/one_attn.py 8192 16 128 2048 0 1 > gpurun_out/r10_ncu_attn.log 2>&1; echo "ncu attn rc=$?"
ncu -i gpurun_out/r10_attn.ncu-rep --page details --csv > gpurun_out/r10_attn_details.csv 2>&1
ncu -i gpurun_out/r10_attn.ncu-rep --page raw --csv > gpurun_out/r10_attn_raw.csv 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_x3_kernel -s 1 -c 1 -o gpurun_out/r10_x3 python -c "
import sys; sys.path[:0]=['.','tests']
import numpy as np, paper_2301_08984_b200 as pb
from plan_builder import matmul_plan
plan, o = matmul_plan(4096, 4096, 4096, in_elem=4, out_elem=4)
rng = np.random.default_rng(0)
with pb.Executor(plan, lane_gpus=[0]) as ex:
    ex.set_inputs({0: rng.standard_normal((4096, 4096)), 1: rng.standard_normal((4096, 4096))})
    ex.run(2)
" > gpurun_out/r10_ncu_x3.log 2>&1; echo "ncu x3 rc=$?"
ncu -i gpurun_out/r10_x3.ncu-rep --page details --csv > gpurun_out/r10_x3_details.csv 2>&1
ncu -i gpurun_out/r10_x3.ncu-rep --page raw --csv > gpurun_out/r10_x3_raw.csv 2>&1
rm -f gpurun_out/*.ncu-rep
