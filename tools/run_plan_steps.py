"""Runs a benchmark plan for a few graph-replayed steps (for ncu launch lists
and captures):  python tools/run_plan_steps.py c5_3f1b [steps] [flags]"""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2301_08984_b200 as pb  # noqa: E402

name = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
flags = int(sys.argv[3], 0) if len(sys.argv) > 3 else 0
plan, meta = bench.load_plan(name)
nl = len(json.loads(plan)["lanes"])
with pb.Executor(plan, lane_gpus=[0] * nl, flags=flags) as ex:
    ex.set_inputs(bench.synthetic_inputs(plan))
    ms = ex.run(steps)
    print(json.dumps({"plan": name, "ms_per_step": ms, "kernels_per_step": ex.stats()["kernels_per_step"]}))
