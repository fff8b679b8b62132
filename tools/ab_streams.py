import sys, json
sys.path.insert(0, '.')
import bench, paper_2301_08984_b200 as pb
plan, meta = bench.load_plan('c2_tp1')
inp = bench.synthetic_inputs(plan)
for flags in (0, pb.SERIAL_LANES, 0, pb.SERIAL_LANES):
    with pb.Executor(plan, lane_gpus=[0], flags=flags) as ex:
        ex.set_inputs(inp); ex.run(5); ms = ex.run(30)
    print("flags", flags, "ms/step", round(ms, 4), "tokens/s", round(meta['samples_per_step'] / ms * 1e3))
